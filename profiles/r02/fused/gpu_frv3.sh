#!/bin/bash
# fused rounds experiment: compact group table (capacity 64) so 3 teams of 64-byte tiles fit with 10 rounds
cp paper_2103_03239_b200/libmoshpit_b200.so /tmp/lib_orig.so
for v in t3_v4_g64 t2_v4_g64; do
  cp profiles/r02/frv/lib_$v.so paper_2103_03239_b200/libmoshpit_b200.so
  r=$(timeout 600 python -m pytest tests/test_gpu_fused_rounds.py -q 2>&1 | tail -1)
  b=$(timeout 300 python profiles/fused_rounds_bench.py 2>&1 | tail -1)
  echo "{\"variant\": \"rowmap_$v\", \"tests\": \"$r\", \"bench\": $b}" | tee -a gpurun_out/frv3.jsonl
done
cp /tmp/lib_orig.so paper_2103_03239_b200/libmoshpit_b200.so
