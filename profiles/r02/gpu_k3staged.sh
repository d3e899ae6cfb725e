timeout 900 python -m pytest tests/test_gpu_sgd.py tests/test_gpu_logistic.py -x -q 2>&1 | tail -3
for form in regs staged; do echo "== $form"; MOSHPIT_K3_FORM=$form timeout 600 python profiles/k3_rounds.py; done
for form in regs staged; do echo "== $form"; MOSHPIT_K3_FORM=$form timeout 600 python profiles/k3_rounds.py; done
MOSHPIT_K3_FORM=staged timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:"group_mean_step|group_mean_reg" -c 6 --csv --log-file gpurun_out/k3_staged_ncu.csv python profiles/k3_rounds.py > /dev/null 2>&1
MOSHPIT_K3_FORM=regs timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:"group_mean_step|group_mean_reg" -c 6 --csv --log-file gpurun_out/k3_regs_ncu.csv python profiles/k3_rounds.py > /dev/null 2>&1
grep -h "gpu__time_duration" gpurun_out/k3_*_ncu.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-160
