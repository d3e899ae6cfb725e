set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/dadd_chain profiles/dadd_chain.cu && ./profiles/dadd_chain > gpurun_out/dadd_chain.json; cat gpurun_out/dadd_chain.json
timeout 600 python profiles/diag_probe.py > gpurun_out/diag_time.json 2>&1; cat gpurun_out/diag_time.json
timeout 300 python profiles/k3_rounds.py > gpurun_out/k3_rounds7_default.json 2>&1; cat gpurun_out/k3_rounds7_default.json
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -c 300 gpurun_out/bench_n1.err
python profiles/nvlink_ncu.py C2 > gpurun_out/nvl_plain.log 2>&1 && timeout 900 ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"cross_mean|shard_pull" --csv --log-file gpurun_out/nvl_ncu_c2.csv python profiles/nvlink_ncu.py C2 > gpurun_out/nvl_ncu_c2.log 2>&1; tail -3 gpurun_out/nvl_plain.log
bash profiles/r02/gpu_pipe_sweep.sh 2>&1 | grep "G=" > gpurun_out/pipe_sweep_g2.txt; cat gpurun_out/pipe_sweep_g2.txt
