B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sgd --no-full --no-variants"
$B > gpurun_out/bench_small.json 2>&1; tail -c 200 gpurun_out/bench_small.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_n1.csv $B > /dev/null 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:group_mean_register -s 3 -c 1 -o gpurun_out/k2_full_c2 $B > /dev/null 2>&1; echo full rc=$?
ncu -i gpurun_out/k2_full_c2.ncu-rep --page raw --csv > gpurun_out/k2_full_c2_raw.csv 2>/dev/null; echo raw rc=$?
ncu -i gpurun_out/k2_full_c2.ncu-rep --page details --csv > gpurun_out/k2_full_c2_details.csv 2>/dev/null; echo details rc=$?
ls -la gpurun_out/k2_full_c2*
