# Kernel 2: register form (default) vs the leaf-streamed body (MOSHPIT_K2_LEAF=4|8)
for cfg in C1 C2 C3slab C5slab; do
  for v in "" 4 8; do
    MOSHPIT_K2_LEAF=$v python bench.py --config $cfg --steps 30 --no-e2e --no-cpu --no-sgd --no-full 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'leaf=${v:-reg}', d['ms_per_step'], d['roofline']['frac'])"
  done
done
