#!/bin/bash
OUT=gpurun_out/${1:-tcq}; mkdir -p $OUT
L="c4:8:vgg4_2,vgg3_2,vgg2_2,vgg5_2 c5:256:layer3.1.conv2,layer3.1.conv1,layer1.0.conv2 c3:128:alexnet-conv2,incep-4e-5x5 c2:32:4e-1x1,3b-1x1,5b-1x1"
timeout 600 python tools/tc_check.py time $L > $OUT/time.log 2>&1
B2C_TC_BSPLIT=1 timeout 600 python tools/tc_check.py time $L > $OUT/time_bsplit.log 2>&1
