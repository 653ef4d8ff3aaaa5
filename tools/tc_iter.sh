#!/bin/bash
# one development iteration of the tensor-core engine: numerics, per-role cycles, timings
OUT=gpurun_out/${1:-tci}; mkdir -p $OUT
timeout 400 python tools/tc_check.py --quick > $OUT/check.log 2>&1
timeout 200 python tools/tc_prof_roles.py c4:8:vgg4_2:tf32x3 c4:8:vgg4_2:tf32 c2:32:4e-1x1:tf32x3 > $OUT/roles.log 2>&1
bash tools/tc_quick.sh $(basename $OUT)
