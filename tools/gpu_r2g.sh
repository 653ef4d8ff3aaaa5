OUT=gpurun_out/r2g; mkdir -p $OUT
python -c "import paper_2103_16234_b200.build as b; b.build(); b.build_dev_variant()" > $OUT/build.log 2>&1
timeout 900 python tools/fam_ab.py c5 256 --only s --layers conv1,layer1.0.conv2,layer2.1.conv2,layer3.1.conv2,layer4.1.conv2,layer2.0.conv2,layer3.0.conv2,layer4.0.conv2 --splits 1,2,3 > $OUT/ab_c5_3x3.txt 2>&1
timeout 900 python tools/fam_ab.py c3 128 --only 5x5 --layers alexnet-conv2,incep-4e-5x5,incep-3b-5x5 --splits 1,2 > $OUT/ab_c3.txt 2>&1
timeout 900 python tools/fam_ab.py c4 8 --only 3x3 --layers vgg1_2,vgg3_2,vgg4_2,vgg5_2 --splits 1,2,4 > $OUT/ab_c4.txt 2>&1
timeout 900 python tools/fam_ab.py c1 1 --only 3x3 --splits 1,2,4,8 > $OUT/ab_c1.txt 2>&1
timeout 900 python tools/fam_ab.py c5 256 --only 1x1s --layers layer2.0.downsample,layer3.0.downsample > $OUT/ab_ds_direct.txt 2>&1
B2C_LIB_VARIANT=dev B2C_KIND2_TRANSPOSE=1 timeout 900 python tools/fam_ab.py c5 256 --only 1x1s --layers layer2.0.downsample,layer3.0.downsample > $OUT/ab_ds_transpose.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
echo done > $OUT/DONE
