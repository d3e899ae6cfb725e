set -x
python - <<'PY' > gpurun_out/ctx_init.json
import time, ctypes
t=time.perf_counter(); import torch; torch.cuda.init(); x=torch.zeros(1,device="cuda"); torch.cuda.synchronize()
print('{"torch_cuda_context_s": %.4f}' % (time.perf_counter()-t))
PY
cat gpurun_out/ctx_init.json
MOSHPIT_LOGIT_TC=1 python profiles/logistic_tc_bench.py 1024 1024 4096 2 > gpurun_out/tc_plain.log 2>&1 && \
MOSHPIT_LOGIT_TC=1 timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_op_hmma.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"tc_gemm|split_kernel|logit_grad|logit_coeff" -c 12 --csv --log-file gpurun_out/tc_launches.csv python profiles/logistic_tc_bench.py 1024 1024 4096 2 > gpurun_out/tc_ncu.log 2>&1
MOSHPIT_LOGIT_TC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -c 2 -o gpurun_out/tc_full python profiles/logistic_tc_bench.py 1024 1024 4096 2 > gpurun_out/tc_ncu_full.log 2>&1
tail -3 gpurun_out/tc_ncu_full.log
