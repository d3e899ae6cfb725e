# kernel-3 prefetch variants (profiles/k3v/lib_*.so built from step_kernel.cu
# with -DMB_K3_PF=1 -DMB_K3_MINB=N, "head" = defaults): parity on the SGD GPU
# tests, then C4 sigma=1 / sigma=0 step time per variant, alternating.
L=paper_2103_03239_b200/libmoshpit_b200.so
cp $L /tmp/lib_keep.so
for v in pf1m4; do
  cp profiles/k3v/lib_$v.so $L; touch $L
  timeout 600 python -m pytest tests/test_gpu_sgd.py -q -x 2>&1 | tail -2 | sed "s/^/$v pytest: /"
done
for v in head pf1m4 pf1m5 head pf1m4 pf1m5; do
  cp profiles/k3v/lib_$v.so $L; touch $L
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-full 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['sgd_c4']; print('$v', s['ms_per_sgd_step'], s['sigma0']['ms_per_sgd_step'])"
done
cp /tmp/lib_keep.so $L
