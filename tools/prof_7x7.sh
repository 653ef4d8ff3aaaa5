#!/bin/bash
OUT=gpurun_out/${1:-p7}; mkdir -p $OUT
for L in 5b-1x1 5a-5x5red; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv" -c 1 --launch-skip 2 \
  -o $OUT/$L python tools/prof_layer.py c2 32 $L > $OUT/ncu_$L.log 2>&1
done
B2C_TRACE_FILE=$OUT/trace_5b.csv timeout 120 python tools/trace_layer.py c2 32 5b-1x1 fused_1x1s_m128 6 $OUT/trace_5b.csv
python tools/trace_summary.py $OUT/trace_5b.csv > $OUT/trace_summary.txt 2>&1
