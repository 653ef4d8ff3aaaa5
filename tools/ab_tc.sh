#!/bin/bash
OUT=gpurun_out/${1:-abtc}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tensorcore.py -x -q -k "not bench_line" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for rep in 1 2; do
for v in new base; do
  if [ $v = base ]; then export B2C_LIB_VARIANT=base; else unset B2C_LIB_VARIANT; fi
  timeout 300 python tools/tc_check.py time c2:32:3a-5x5red,3a-1x1,4e-1x1,5b-1x1,4a-5x5red c5:256:layer1.0.conv1,layer3.1.conv2,layer4.1.conv1 c4:8:vgg4_2 > $OUT/layers_${v}_$rep.log 2>&1
done
done
unset B2C_LIB_VARIANT
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --engine tf32x3 --tc-engine none --e2e-steps 0 > $OUT/bench_new.json 2> $OUT/bench_new.err
B2C_LIB_VARIANT=base timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --engine tf32x3 --tc-engine none --e2e-steps 0 > $OUT/bench_base.json 2> $OUT/bench_base.err
