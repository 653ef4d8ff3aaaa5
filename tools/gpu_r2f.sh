OUT=gpurun_out/r2f; mkdir -p $OUT
python -c "import paper_2103_16234_b200.build as b; b.build(); b.build_dev_variant()" > $OUT/build.log 2>&1
LAY=layer1.0.conv3,layer1.1.conv1,layer2.1.conv1,layer3.0.conv1,layer3.1.conv1,layer3.1.conv3,layer4.0.conv1
timeout 900 python tools/fam_ab.py c5 256 --only 1x1v --layers $LAY > $OUT/ab_persist.txt 2>&1
B2C_LIB_VARIANT=dev B2C_PERSIST=0 timeout 900 python tools/fam_ab.py c5 256 --only 1x1v --layers $LAY > $OUT/ab_nopersist.txt 2>&1
timeout 900 python tools/fam_ab.py c2 32 --only 1x1v --splits 1,2,4 --layers 3a-1x1,3b-1x1,4a-1x1,4e-1x1,4e-3x3red > $OUT/ab_c2_persist.txt 2>&1
B2C_LIB_VARIANT=dev B2C_PERSIST=0 timeout 900 python tools/fam_ab.py c2 32 --only 1x1v --splits 1,2,4 --layers 3a-1x1,3b-1x1,4a-1x1,4e-1x1,4e-3x3red > $OUT/ab_c2_nopersist.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv -s 3 -c 1 -o $OUT/full_c5_layer3.1.conv1 python tools/prof_layer.py c5 256 layer3.1.conv1 > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
