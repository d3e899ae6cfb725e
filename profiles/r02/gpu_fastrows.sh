#!/bin/bash
# FAST distortion partials: rows per block 8 (built) vs 16 vs 4, same box (diag_probe: ms per C2 round + record)
python profiles/diag_probe.py > gpurun_out/fr_8.txt 2>&1
for R in 16 4; do
  touch paper_2103_03239_b200/csrc/diag_kernel.cu
  MOSHPIT_NVCC_EXTRA="-DMB_FAST_ROWS=$R" python -c "from paper_2103_03239_b200 import build as b; b.build()" > gpurun_out/fr_build_$R.log 2>&1
  python profiles/diag_probe.py > gpurun_out/fr_$R.txt 2>&1
done
touch paper_2103_03239_b200/csrc/diag_kernel.cu
python -c "from paper_2103_03239_b200 import build as b; b.build()" > /dev/null 2>&1
python profiles/diag_probe.py > gpurun_out/fr_8b.txt 2>&1
tail -n1 gpurun_out/fr_*.txt
