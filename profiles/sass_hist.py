"""SASS instruction histogram per kernel of the built library (cuobjdump
-sass), for the hot kernels: kernel 1 (form_groups_kernel), kernel 2
(group_mean_register, group_mean_bulk), kernel 3 (group_mean_step_leaf), the
two-round SGD pass, the cross-round kernels (exact and partial-sum) and the
EXACT diagnostics.  Writes a text table.

    python profiles/sass_hist.py > profiles/r02/sass_hist.txt
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2103_03239_b200", "libmoshpit_b200.so")
PATTERNS = ["form_groups_kernel", "group_mean_register", "group_mean_bulk",
            "group_mean_step_leaf", "two_round_step_kernel", "cross_mean_kernel",
            "partial_sum_kernel", "partial_combine_kernel", "shard_pull_kernel",
            "dist_exact_tiled", "colmean_kernel"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if m and cur:
            funcs[cur][m.group(1).split(".")[0]] += 1
    print(f"library: {os.path.basename(LIB)} ({os.path.getsize(LIB) / 1e6:.1f} MB), "
          f"{len(funcs)} kernels, {sum(sum(c.values()) for c in funcs.values())} SASS instructions")
    tot = collections.Counter()
    for c in funcs.values():
        tot.update(c)
    print("whole library, top opcodes:", ", ".join(f"{k} {v}" for k, v in tot.most_common(12)))
    for k in ("UTMALDG", "UTMASTG", "UBLKCP", "HMMA", "UTCHMMA", "UTCQMMA", "LDTM", "STTM"):
        print(f"  {k}: {tot.get(k, 0)}")
    for pat in PATTERNS:
        names = [f for f in funcs if pat in f]
        for f in names:
            c = funcs[f]
            short = re.sub(r"_ZN5mb200\d*_GLOBAL__N__\w+?_\d+", "", f)[:90]
            print(f"\n{short}: {sum(c.values())} instructions")
            print("   " + ", ".join(f"{k} {v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    sys.exit(main())
