"""Build libmoshpit_b200.so in-tree for sm_100a (nvcc, static cudart).

    python -m paper_2103_03239_b200.build [--force]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false`` (no FMA
contraction: the averaging tree must round exactly like the reference) and
linked into ``paper_2103_03239_b200/libmoshpit_b200.so``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmoshpit_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-prec-div=true",
         "-prec-sqrt=true", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fno-fast-math", "-I" + os.path.join(ROOT, "include")]
# measurement builds only (e.g. "-DMB_PHILOX_ROUNDS=7" in a scratch copy)
FLAGS += os.environ.get("MOSHPIT_NVCC_EXTRA", "").split()


def _nvcc():
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def up_to_date():
    """The library is current when every object is fresh and the library is
    newer than every object."""
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if not _obj_fresh(src, obj) or os.path.getmtime(obj) > t:
            return False
    return True


def _includes(path, seen=None):
    """Local headers a source pulls in (#include "...", transitively)."""
    import re
    seen = set() if seen is None else seen
    try:
        text = open(path).read()
    except OSError:
        return seen
    for name in re.findall(r'^\s*#\s*include\s+"([^"]+)"', text, re.M):
        for d in (os.path.dirname(path), CSRC, os.path.join(ROOT, "include")):
            h = os.path.normpath(os.path.join(d, name))
            if os.path.exists(h):
                if h not in seen:
                    seen.add(h)
                    _includes(h, seen)
                break
    return seen


def _obj_fresh(src, obj):
    """An object is reused when it is newer than its .cu and every local
    header it includes."""
    if not os.path.exists(obj):
        return False
    t = os.path.getmtime(obj)
    return all(os.path.getmtime(d) <= t for d in [src, *_includes(src)])


def _compile(src, nvcc, force=False):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if not force and _obj_fresh(src, obj):
        return obj
    cmd = [nvcc, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force=False, verbose=False):
    """force=True recompiles every object; otherwise only stale objects are
    rebuilt (mean_kernel.cu alone takes minutes: 32 specialised trees x dtypes)."""
    if not force and up_to_date():
        return LIB
    nvcc = _nvcc()
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, nvcc, force), sources()))
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print("built", LIB)
    return LIB


def build_host_tools(verbose=False):
    """g++ of the host-side programs over the drop-in header: the drop-in
    bench (bench.py's e2e_dropin_f64) and, where the reference tree is present
    (the build container), the reference-harness bridge test binary -- both
    travel to the GPU box with the snapshot."""
    lib_dir = HERE
    out = []
    src = os.path.join(CSRC, "host", "bench_dropin.cpp")
    exe = os.path.join(HERE, "bench_dropin")
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", src, "-I", os.path.join(ROOT, "include"),
           "-L", lib_dir, "-lmoshpit_b200", "-Wl,-rpath,$ORIGIN", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, timeout=300)
    out.append(exe)
    ref_inc = "/root/reference/proj/include"
    json_inc = os.path.join(sys.prefix, "lib", "python3.12", "site-packages", "include",
                            "cudnn_frontend", "thirdparty", "nlohmann")
    if os.path.isdir(os.path.join(ref_inc, "moshpit")) and os.path.exists(
            os.path.join(json_inc, "json.hpp")):
        src = os.path.join(ROOT, "tests", "cpp", "test_harness_bridge.cpp")
        exe = os.path.join(ROOT, "tests", "cpp", "test_harness_bridge")
        cmd = ["g++", "-std=c++20", "-O2", src, "-I", os.path.join(ROOT, "include"), "-I",
               ref_inc, "-I", json_inc, "-L", lib_dir, "-lmoshpit_b200",
               "-Wl,-rpath,$ORIGIN/../../paper_2103_03239_b200", "-o", exe]
        subprocess.run(cmd, check=True, capture_output=True, timeout=300)
        out.append(exe)
    if verbose:
        print("built", *out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    build_host_tools(verbose=True)
