OUT=gpurun_out/r2h; mkdir -p $OUT
python -c "import paper_2103_16234_b200.build as b; b.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -q -x -k "not twostage" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
LAY=layer1.0.conv3,layer1.1.conv1,layer2.1.conv1,layer3.0.conv1,layer3.1.conv1,layer3.1.conv3,layer4.0.conv1
timeout 900 python tools/fam_ab.py c5 256 --only 1x1 --layers $LAY > $OUT/ab_c5.txt 2>&1
timeout 900 python tools/fam_ab.py c2 32 --only 1x1 --splits 1,2,4 --layers 3a-1x1,3b-1x1,4a-1x1,4e-1x1,4e-3x3red,4d-5x5red > $OUT/ab_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk -s 3 -c 1 -o $OUT/full_bulk python tools/prof_layer_fam.py c5 256 layer3.1.conv1 fused_1x1t_m64 > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
