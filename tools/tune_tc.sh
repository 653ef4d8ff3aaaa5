#!/bin/bash
OUT=gpurun_out/tune2; mkdir -p $OUT
for spec in c2:32 c3:128 c4:8 c5:256 c4:128 c1:1; do
  wl=${spec%%:*}; n=${spec##*:}
  timeout 1500 python tools/autotune.py --engines tf32x3 --workloads $wl --batches $n --budget-s 1400 --out $OUT/tc_${wl}_$n.json > $OUT/tc_${wl}_$n.log 2>&1
done
echo done > $OUT/DONE
