# kernel-3 variants (profiles/k3v/lib_*.so, built from step_kernel.cu with
# -DMB_K3_ILP=N or HEAD's file): C4 sigma=1 / sigma=0 step time per variant
L=paper_2103_03239_b200/libmoshpit_b200.so
cp $L /tmp/lib_keep.so
for v in i4m5 i4m4 i4m5 i4m4; do
  cp profiles/k3v/lib_$v.so $L; touch $L
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-full 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['sgd_c4']; print('$v', s['ms_per_sgd_step'], s['sigma0']['ms_per_sgd_step'])"
done
cp /tmp/lib_keep.so $L
