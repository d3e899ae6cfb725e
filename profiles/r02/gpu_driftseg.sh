timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q 2>&1 | tail -2
timeout 600 python profiles/diag_probe.py 2>&1 | tail -1 | cut -c1-150
