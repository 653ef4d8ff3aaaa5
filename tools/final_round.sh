#!/bin/bash
# round-end evidence: smoke, GPU suite, bench (both arms), extra workloads, launch list
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
export PYTHONUNBUFFERED=1
nvidia-smi > $OUT/nvidia-smi.txt 2>&1; nvidia-smi topo -m > $OUT/topo.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
# measured DRAM traffic of every layer's launches (feeds the roofline "traffic" of the bench lines)
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"conv|stage2" --csv --log-file $OUT/traffic_ncu.csv python tools/traffic.py run c1,c2,c3,c4,c5 \
  > $OUT/traffic_layers.json 2> $OUT/traffic.err
python tools/traffic.py merge $OUT/traffic_layers.json $OUT/traffic_ncu.csv > $OUT/r1_traffic.json 2>> $OUT/traffic.err \
  && cp $OUT/r1_traffic.json profiles/r1_traffic.json
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for wl in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --tc-engine none > $OUT/ncu_bench.log 2>&1
# one --set full capture of the top C2 layer's kernel and of the C1 kernel (plans as shipped)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv" -c 1 --launch-skip 2 \
  -o $OUT/c2_4e1x1 python tools/prof_layer.py c2 32 4e-1x1 > $OUT/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv" -c 1 --launch-skip 2 \
  -o $OUT/c1 python tools/prof_layer.py c1 1 res-conv2x-3x3 > $OUT/ncu_c1.log 2>&1
echo done > $OUT/DONE
