#!/bin/bash
OUT=gpurun_out/${1:-tcm}; mkdir -p $OUT
for m in ${MODES:-0 1 2 8 3 11}; do
  echo "mode $m" >> $OUT/modes.log
  B2C_TC_MODE=$m timeout 300 python tools/tc_check.py time c3:128:alexnet-conv2 c4:8:vgg3_2 >> $OUT/modes.log 2>&1
done
