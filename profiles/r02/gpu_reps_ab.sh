for g in 0 1; do for w in 1 4 16; do
  echo "gather32=$g waves=$w $(MOSHPIT_REP_GATHER_F32=$g MOSHPIT_FAST_ROW_WAVES=$w timeout 300 python -c "
import sys,os; sys.path.insert(0,'.'); import json, bench, torch, paper_2103_03239_b200 as mb
print(min(bench.measure_variant(mb, torch, 'C2', 0, 20, 3, diag='fast')['ms_per_step'] for _ in range(2)))" 2>&1 | tail -1)"
done; done
