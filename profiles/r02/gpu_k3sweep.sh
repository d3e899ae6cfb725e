# kernel-3 (noisy) occupancy / ILP variants, each built in a scratch copy
for v in "-DMB_K3_MINB=5" "-DMB_K3_MINB=6" "-DMB_K3_MINB=4" "-DMB_K3_MINB=6 -DMB_K3_ILP=2" "-DMB_K3_MINB=8 -DMB_K3_ILP=2"; do
  rm -rf /tmp/k3v && cp -r . /tmp/k3v && (cd /tmp/k3v && MOSHPIT_NVCC_EXTRA="$v" python -c "from paper_2103_03239_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 && MOSHPIT_NVCC_EXTRA="$v" timeout 300 python profiles/k3_rounds.py)
done > gpurun_out/k3_sweep.jsonl 2>&1
cat gpurun_out/k3_sweep.jsonl
