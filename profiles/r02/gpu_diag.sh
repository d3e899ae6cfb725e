set -x
for m in 0 1; do MOSHPIT_DIAG_PASS=$m timeout 600 python profiles/diag_probe.py > gpurun_out/diag_time_$m.json 2> gpurun_out/diag_time_$m.err; cat gpurun_out/diag_time_$m.json; done
for m in 0 1; do MOSHPIT_DIAG_PASS=$m python profiles/diag_probe.py ncu > /dev/null 2>&1 && MOSHPIT_DIAG_PASS=$m timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/diag_launches_$m.csv python profiles/diag_probe.py ncu > gpurun_out/diag_ncu_$m.log 2>&1; done
cp -r . /tmp/v7 && cd /tmp/v7 && MOSHPIT_NVCC_EXTRA="-DMB_PHILOX_ROUNDS=7" python -c "from paper_2103_03239_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 && MOSHPIT_NVCC_EXTRA="-DMB_PHILOX_ROUNDS=7" timeout 300 python profiles/k3_rounds.py > $GRAFT_REPO_ROOT/gpurun_out/k3_rounds7.json 2>&1; cd $GRAFT_REPO_ROOT
timeout 300 python profiles/k3_rounds.py > gpurun_out/k3_rounds10.json 2>&1
cat gpurun_out/k3_rounds*.json
