#!/bin/bash
# per-kernel ncu view of one rank's partial-sum cross round (probe mode, 4 GPUs mapped)
python profiles/partial_probe.py 4 partial > gpurun_out/p4_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv -k regex:"partial|shard_pull|move_rows|group_mean|cross_mean|barrier" --log-file gpurun_out/p4_ncu_g4_partial.csv python profiles/partial_probe.py 4 partial > gpurun_out/p4_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum --clock-control none --csv -k regex:"partial|shard_pull|move_rows|group_mean|cross_mean" --log-file gpurun_out/p4_ncu_g4_exact.csv python profiles/partial_probe.py 4 exact >> gpurun_out/p4_ncu.log 2>&1
tail -3 gpurun_out/p4_ncu.log
