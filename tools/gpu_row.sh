#!/bin/bash
# Row-segment / warp-specialised kernels bring-up: memcheck of every new family
# on small cases, the family parity tests, then A/B against the existing
# families on the BASELINE layers.  Outputs -> gpurun_out/$TAG/.
TAG=${1:-row}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONUNBUFFERED=1 B2C_WATCHDOG_MS=20000
python -c "import paper_2103_16234_b200.build as b; b.build()" > $OUT/build.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/rowdbg.py > $OUT/memcheck.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_family or cluster" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
unset B2C_WATCHDOG_MS
L1=layer1.0.conv1,layer1.0.conv3,layer1.1.conv1,layer2.0.conv1,layer2.0.downsample,layer2.1.conv1,layer2.1.conv3,layer3.1.conv1,layer3.1.conv3,layer4.0.conv1,layer4.1.conv1,layer4.1.conv3
timeout 900 python tools/fam_ab.py c5 256 --layers $L1 --splits 1,2 > $OUT/ab_c5_1x1.txt 2>&1
L3=conv1,layer2.0.conv2,layer3.0.conv2,layer4.0.conv2
timeout 900 python tools/fam_ab.py c5 256 --layers $L3 --splits 1,2,3 > $OUT/ab_c5_s2.txt 2>&1
timeout 600 python tools/fam_ab.py c2 32 --splits 1,2,4 > $OUT/ab_c2.txt 2>&1
echo done > $OUT/DONE
