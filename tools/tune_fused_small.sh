#!/bin/bash
# fused-engine plans after adding the small-tile (p128) families: batch-1 and C2 layers
OUT=gpurun_out/${1:-tunef}; mkdir -p $OUT
timeout 1000 python tools/autotune.py --engines fused --workloads c1,c2 --budget-s 900 --out $OUT/fused_c1c2.json > $OUT/fused_c1c2.log 2>&1
timeout 1000 python tools/autotune.py --engines fused --workloads c3,c4,c5 --batches 1 --budget-s 900 --out $OUT/fused_n1.json > $OUT/fused_n1.log 2>&1
timeout 1000 python tools/autotune.py --engines fused --workloads c3,c4 --batches 8 --budget-s 900 --out $OUT/fused_n8.json > $OUT/fused_n8.log 2>&1
echo done > $OUT/DONE
