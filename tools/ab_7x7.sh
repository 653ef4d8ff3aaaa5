#!/bin/bash
OUT=gpurun_out/${1:-ab7}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python tools/tc_check.py time c2:32:5b-1x1,5a-5x5red,5a-1x1,5b-3x3red,5a-poolproj c5:256:layer2.0.downsample,layer3.0.downsample > $OUT/layers.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --tc-engine none --e2e-steps 0 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
