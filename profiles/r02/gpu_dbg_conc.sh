for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "concurrent" 2>&1 | tail -30; done
