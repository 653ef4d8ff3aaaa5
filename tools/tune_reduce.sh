#!/bin/bash
# fused plans with the split-C reduction mode searched (partial planes vs DSMEM cluster)
OUT=gpurun_out/${1:-tuner}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or every_family" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 1000 python tools/autotune.py --engines fused --workloads c1,c2 --budget-s 900 --out $OUT/fused_c1c2.json > $OUT/fused_c1c2.log 2>&1
timeout 1000 python tools/autotune.py --engines fused --workloads c3,c4,c5 --batches 1 --budget-s 900 --out $OUT/fused_n1.json > $OUT/fused_n1.log 2>&1
echo done > $OUT/DONE
