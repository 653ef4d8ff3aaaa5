#!/bin/bash
# A/B of two in-tree builds: libb2conv.so (new) vs libb2conv_base.so (B2C_LIB_VARIANT=base)
OUT=gpurun_out/${1:-ablib}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for rep in 1 2; do
for v in new base; do
  if [ $v = base ]; then export B2C_LIB_VARIANT=base; else unset B2C_LIB_VARIANT; fi
  timeout 300 python tools/tc_check.py time c2:32:4e-1x1,3b-1x1,5b-1x1,4a-3x3red,4b-1x1 c5:256:layer1.0.conv1,layer3.1.conv1 > $OUT/layers_${v}_$rep.log 2>&1
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --tc-engine none --e2e-steps 0 > $OUT/bench_${v}_$rep.json 2> $OUT/bench_${v}_$rep.err
done
done
