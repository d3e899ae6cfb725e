"""bench.py's driver contract, checked on the CPU box: the reference arm
(`--impl reference`: the unmodified reference run_moshpit on host cores)
prints one JSON line with the contract's keys; non-zero ranks of a torchrun
launch exit 0 without work; the GPU arm fails loudly without a device."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None, timeout=300):
    env = dict(os.environ, MOSHPIT_REF_TOTAL_S="2", **(env_extra or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          env=env, capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line(ref):
    r = _bench(["--impl", "reference", "--steps", "2", "--warmup", "3"],
               {"RANK": "0", "WORLD_SIZE": "1"})
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2")


def test_reference_arm_other_ranks_exit_quietly():
    r = _bench(["--impl", "reference", "--steps", "2", "--warmup", "3"],
               {"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_gpu_arm_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = _bench(["--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu"],
               {"RANK": "0", "WORLD_SIZE": "1"})
    assert r.returncode != 0
    assert r.stdout.strip() == ""


def test_both_arms_print_the_same_config(ref):
    """The driver compares the arms' `config` dicts: both come from
    bench.workload_config with no arm-specific keys."""
    sys.path.insert(0, ROOT)
    import bench
    r = _bench(["--impl", "reference", "--steps", "1", "--warmup", "3"],
               {"RANK": "0", "WORLD_SIZE": "1"})
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["config"] == bench.workload_config("C2")
    assert "parallelism" not in d["config"] and "kernel" not in d["config"]
