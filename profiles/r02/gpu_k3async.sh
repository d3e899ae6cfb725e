MOSHPIT_K3_ASYNC=1 timeout 900 python -m pytest tests/test_gpu_sgd.py tests/test_gpu_fused_rounds.py -x -q 2>&1 | tail -1
for i in 1 2; do for a in 0 1; do echo "== async=$a"; MOSHPIT_K3_ASYNC=$a timeout 600 python profiles/k3_rounds.py | cut -c60-400; done; done
for a in 0 1; do MOSHPIT_K3_ASYNC=$a timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:step_leaf -c 3 --csv --log-file gpurun_out/k3a$a.csv python profiles/k3_rounds.py > /dev/null 2>&1; grep -h gpu__time gpurun_out/k3a$a.csv | awk -F'","' '{print "async='$a'", substr($5,1,50), $NF}'; done
