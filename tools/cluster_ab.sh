#!/bin/bash
# A/B of split-C through DSMEM clusters (B2C_CLUSTER=1) vs partial planes + stage-2 (default)
OUT=gpurun_out/${1:-cab}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or every_family" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for wl in c2 c1 c3 c5; do
  for mode in cluster planes; do
    if [ $mode = cluster ]; then export B2C_CLUSTER=1; else unset B2C_CLUSTER; fi
    timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --tc-engine none > $OUT/bench_${wl}_$mode.json 2> $OUT/bench_${wl}_$mode.err
  done
done
unset B2C_CLUSTER
B2C_CLUSTER=1 timeout 600 python tools/tc_check.py time c2:32:4e-1x1,3b-1x1,5b-1x1,4a-5x5red,3a-1x1 c1:1:res-conv2x-3x3 > $OUT/layers_cluster.log 2>&1
timeout 600 python tools/tc_check.py time c2:32:4e-1x1,3b-1x1,5b-1x1,4a-5x5red,3a-1x1 c1:1:res-conv2x-3x3 > $OUT/layers_planes.log 2>&1
