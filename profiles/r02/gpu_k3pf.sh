timeout 900 python -m pytest tests/test_gpu_sgd.py -x -q -k fused 2>&1 | tail -1
MOSHPIT_K3_L2PF=1 timeout 900 python -m pytest tests/test_gpu_sgd.py -x -q -k fused 2>&1 | tail -1
for i in 1 2; do for pf in 0 1; do echo "== pf=$pf"; MOSHPIT_K3_L2PF=$pf timeout 600 python profiles/k3_rounds.py; done; done
