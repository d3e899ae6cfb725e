#!/bin/bash
# NVLink user bytes of the partial-sum cross round (probe mode) vs the model, 2 and 4 GPUs
for w in 2 4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum --clock-control none --csv -k regex:"partial|shard_pull" --log-file gpurun_out/p9_ncu_nvl_g${w}_partial.csv python profiles/partial_probe.py $w partial > gpurun_out/p9_model_g${w}.log 2>&1
done
grep world gpurun_out/p9_model_g*.log
