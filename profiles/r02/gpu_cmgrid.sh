timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "column_means or f32_bit_exact or record" 2>&1 | tail -1
for g in 0 444 296 222 148 74; do echo "== MOSHPIT_CM_GRID=$g"; MOSHPIT_CM_GRID=$g timeout 600 python profiles/diag_probe.py 2>&1 | tail -1 | cut -c1-120; done
