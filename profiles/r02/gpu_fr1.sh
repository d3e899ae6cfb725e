timeout 1200 python -m pytest tests/test_gpu_fused_rounds.py -x -q 2>&1 | tail -15
for f in 1 0; do echo "== MOSHPIT_SGD_FUSED_ROUNDS=$f"; MOSHPIT_SGD_FUSED_ROUNDS=$f timeout 600 python profiles/k3_rounds.py; done
