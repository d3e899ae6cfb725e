for m in 0 2; do echo "== MOSHPIT_SGD_FUSED_HAT=$m"; MOSHPIT_SGD_FUSED_HAT=$m timeout 600 python profiles/r02/c4_diag.py; done
MOSHPIT_SGD_FUSED_HAT=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16 --csv --log-file gpurun_out/c4diag_unfused.csv python profiles/r02/c4_diag.py > /dev/null 2>&1; echo rc=$?
grep -h "gpu__time_duration" gpurun_out/c4diag_unfused.csv | awk -F'","' '{print $5, $NF}' | cut -c1-60,100-200
