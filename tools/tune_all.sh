#!/bin/bash
# measured plans for the BASELINE layers -> gpurun_out/tune/*.json (merged into tuned_plans.json here)
OUT=gpurun_out/tune; mkdir -p $OUT
timeout 1700 python tools/autotune.py --engines tf32x3,tf32 --workloads c2 --batches 32 --budget-s 1600 --out $OUT/tc_c2.json > $OUT/tc_c2.log 2>&1
timeout 1700 python tools/autotune.py --engines tf32x3,tf32 --workloads c3 --batches 128 --budget-s 1600 --out $OUT/tc_c3.json > $OUT/tc_c3.log 2>&1
timeout 1700 python tools/autotune.py --engines tf32x3,tf32 --workloads c4 --batches 8 --budget-s 1600 --out $OUT/tc_c4.json > $OUT/tc_c4.log 2>&1
timeout 1700 python tools/autotune.py --engines tf32x3,tf32 --workloads c5 --batches 256 --budget-s 1600 --out $OUT/tc_c5.json > $OUT/tc_c5.log 2>&1
timeout 1700 python tools/autotune.py --engines fused --workloads c1,c2,c3,c4,c5 --budget-s 1600 --out $OUT/fused.json > $OUT/fused.log 2>&1
echo done > $OUT/DONE
