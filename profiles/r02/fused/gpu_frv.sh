#!/bin/bash
# fused-rounds team/tile-width sweep: per variant the fused parity tests + profiles/fused_rounds_bench.py
cp paper_2103_03239_b200/libmoshpit_b200.so /tmp/lib_orig.so
for v in t2_v4 t3_v4 t4_v2 t3_v2 t2_v2; do
  cp profiles/r02/frv/lib_$v.so paper_2103_03239_b200/libmoshpit_b200.so
  r=$(timeout 600 python -m pytest tests/test_gpu_fused_rounds.py -q -x 2>&1 | tail -1)
  b=$(timeout 300 python profiles/fused_rounds_bench.py 2>&1 | tail -1)
  echo "{\"variant\": \"$v\", \"tests\": \"$r\", \"bench\": $b}" | tee -a gpurun_out/frv.jsonl
done
cp /tmp/lib_orig.so paper_2103_03239_b200/libmoshpit_b200.so
