#!/bin/bash
# drift finish staged in shared memory: FAST parity tests (all paths), timing, launch list
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_sgd.py -q -k "fast or rounds_record or round_record or report or streamed or rows_equals or concurrent" 2>&1 | tail -3 > gpurun_out/rrec2_pytest.log; cat gpurun_out/rrec2_pytest.log
python profiles/diag_probe.py > gpurun_out/rrec2_new.txt 2>&1; tail -n1 gpurun_out/rrec2_new.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"drift|fold|colmean|dist_rows" --log-file gpurun_out/rrec2_launches.csv python profiles/diag_probe.py ncu > /dev/null 2>&1
