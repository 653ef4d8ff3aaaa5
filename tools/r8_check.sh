#!/bin/bash
OUT=gpurun_out/${1:-r8}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python tools/c1_plans.py c1 1 res-conv2x-3x3 > $OUT/c1.log 2>&1
timeout 600 python tools/c1_plans.py c4 1 vgg3_2 > $OUT/vgg32_n1.log 2>&1
timeout 600 python tools/c1_plans.py c5 256 layer1.0.conv2 > $OUT/l10c2_n256.log 2>&1
