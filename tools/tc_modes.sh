#!/bin/bash
OUT=gpurun_out/${1:-tcm}; mkdir -p $OUT
for m in ${MODES:-0 3 11 19 51 59 2 8 16}; do
  echo "mode $m" >> $OUT/modes.log
  B2C_TC_MODE=$m timeout 300 python tools/tc_check.py time c4:8:vgg4_2 >> $OUT/modes.log 2>&1
done
