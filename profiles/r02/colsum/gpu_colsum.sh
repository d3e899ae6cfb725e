#!/bin/bash
# exact-sum fp32 column means over the distinct rows: GPU suite, record timing with it on/off, launch list
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/cs_pytest.log; cat gpurun_out/cs_pytest.log
MOSHPIT_COLSUM_EXACT=0 python profiles/diag_probe.py 2>&1 | tail -n1 > gpurun_out/cs_off.txt; cat gpurun_out/cs_off.txt
python profiles/diag_probe.py 2>&1 | tail -n1 > gpurun_out/cs_on.txt; cat gpurun_out/cs_on.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"cs_|dist_rows|fold|drift" --log-file gpurun_out/cs_launches.csv python profiles/diag_probe.py ncu > /dev/null 2>&1
