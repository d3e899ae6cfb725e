# kernel 1 (form_groups) time per launch on C2 / C4 shapes
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:form_groups python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-sgd --no-full 2>/dev/null | grep form_groups | tail -3 | awk -F'","' '{print "C2 form_groups ns", $NF}'
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:form_groups python bench.py --config C1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-sgd --no-full 2>/dev/null | grep form_groups | tail -2 | awk -F'","' '{print "C1 form_groups ns", $NF}'
