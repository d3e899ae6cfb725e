"""record_round diagnostics on the device at C2 size (1024 x 4 Mi): per-round
time of the Engine round + record (FAST fp32, EXACT fp64) and the host-buffer
run_moshpit e2e (FAST fp32, pinned).  `python profiles/diag_probe.py` prints
timings; `... ncu` runs a short sequence for an ncu launch list."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_03239_b200 as mb  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "time"
tag = os.environ.get("MOSHPIT_DIAG_PASS", "0")
if mode == "ncu":
    for f64, diag in ((False, "fast"), (True, "exact")):
        bench.measure_variant(mb, torch, "C2", 0, 2, 0, f64=f64, diag=diag)
    sys.exit(0)
out = {"MOSHPIT_DIAG_PASS": tag}
for name, kw in (("f32_fast", dict(diag="fast")), ("f64_exact", dict(f64=True, diag="exact")),
                 ("f32_none", {})):
    r = bench.measure_variant(mb, torch, "C2", 0, 10, 3, **kw)
    out[name] = r["ms_per_step"]
e = bench.measure_e2e(mb, "C2")
out["e2e_f32_fast_pinned_s"] = e["seconds"]
print(json.dumps(out), flush=True)
