for ca in 0 1; do echo "== CA=$ca"; MOSHPIT_CM_CA=$ca timeout 600 python profiles/diag_probe.py 2>&1 | tail -1; done
MOSHPIT_CM_CA=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__inst_issued.avg.pct_of_peak_sustained_active -k regex:colmean --clock-control none --csv --log-file gpurun_out/cm_ca.csv python profiles/diag_probe.py ncu > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time\|lts__t" gpurun_out/cm_ca.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-50,90-200
