# e2e of the C2 bench with HEAD's kernel 1 (fused narrow-round code, 1088-byte
# stack frame) against the same library with the pre-fusion kernel 1 (no stack)
L=paper_2103_03239_b200/libmoshpit_b200.so
cp $L profiles/k1v/lib_head.so
for v in head nofuse head nofuse; do
  cp profiles/k1v/lib_$v.so $L; touch $L
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-full 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v', e['value'], e['seconds_each'], e.get('frac_of_pcie_ceiling'), d['value'])"
done
cp profiles/k1v/lib_head.so $L
