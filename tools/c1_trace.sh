#!/bin/bash
# per-CTA phase traces of the C1 layer (N=1) under several plans
OUT=gpurun_out/${1:-c1tr}; mkdir -p $OUT
for plan in "fused_3x3s1_m64 8" "fused_3x3s1_m64 4" "fused_3x3s1_m64 1" "fused_3x3s1_m32p128 4" "fused_3x3s1_m64p128 4" "fused_3x3s1_m32 8" "fused_3x3s1_m128 8"; do
  set -- $plan
  timeout 120 python tools/trace_layer.py c1 1 res-conv2x-3x3 $1 $2 $OUT/tr_${1}_$2.csv
done
python tools/trace_summary.py $OUT/tr_*.csv > $OUT/summary.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c1_launches.csv python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --tc-engine none --e2e-steps 0 > /dev/null 2>&1
