set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g; nproc; grep -m1 "model name" /proc/cpuinfo
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python profiles/e2e_modes.py > gpurun_out/e2e_modes.txt 2>&1
cat gpurun_out/e2e_modes.txt
