#!/bin/bash
# rounds_record with the FAST row-partial cache: parity tests, then C2 round + FAST record per round
python -m pytest tests/test_gpu_parity.py -q -k "rounds_record or round_record or report or streamed" 2>&1 | tail -3 > gpurun_out/rrec_pytest.log; cat gpurun_out/rrec_pytest.log
python profiles/diag_probe.py > gpurun_out/rrec_new.txt 2>&1
MOSHPIT_BENCH_ROUND_RECORD=1 python profiles/diag_probe.py > gpurun_out/rrec_old.txt 2>&1
tail -n1 gpurun_out/rrec_new.txt gpurun_out/rrec_old.txt
python profiles/diag_probe.py ncu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/rrec_launches.csv python profiles/diag_probe.py ncu > /dev/null 2>&1
