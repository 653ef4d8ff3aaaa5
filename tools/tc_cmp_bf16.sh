#!/bin/bash
OUT=gpurun_out/${1:-tcb}; mkdir -p $OUT
timeout 400 python tools/tc_check.py --quick > $OUT/check.log 2>&1
L="c4:8:vgg4_2,vgg3_2,vgg2_2,vgg5_2 c4:128:vgg4_2,vgg3_2 c5:256:layer3.1.conv2,layer1.0.conv2 c3:128:alexnet-conv2,incep-4e-5x5 c2:32:4e-1x1,3b-1x1"
timeout 600 python tools/tc_check.py time $L > $OUT/time.log 2>&1
mkdir -p $OUT/off; B2C_TC_BF16CORR=0 timeout 600 python tools/tc_check.py time $L > $OUT/off/time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tensorcore.py -q -x > $OUT/pytest.log 2>&1
