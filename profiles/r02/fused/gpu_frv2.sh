#!/bin/bash
# fused rounds, leaf-row lane mapping: tests + bench for (teams, vectors) = (2, 4) default and (4, 2); ncu of the default
cp paper_2103_03239_b200/libmoshpit_b200.so /tmp/lib_orig.so
for v in t2_v4 t4_v2; do
  cp profiles/r02/frv/lib_$v.so paper_2103_03239_b200/libmoshpit_b200.so
  r=$(timeout 600 python -m pytest tests/test_gpu_fused_rounds.py -q -x 2>&1 | tail -1)
  b=$(timeout 300 python profiles/fused_rounds_bench.py 2>&1 | tail -1)
  echo "{\"variant\": \"rowmap_$v\", \"tests\": \"$r\", \"bench\": $b}" | tee -a gpurun_out/frv2.jsonl
done
cp /tmp/lib_orig.so paper_2103_03239_b200/libmoshpit_b200.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rounds_fused -c 1 -o gpurun_out/frv2_full python profiles/fused_rounds_bench.py > gpurun_out/frv2_ncu.log 2>&1
ncu -i gpurun_out/frv2_full.ncu-rep --page details --csv > gpurun_out/frv2_details.csv 2>&1
ncu -i gpurun_out/frv2_full.ncu-rep --page raw --csv > gpurun_out/frv2_raw.csv 2>&1
rm -f gpurun_out/frv2_full.ncu-rep
