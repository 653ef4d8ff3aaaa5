#!/bin/bash
OUT=gpurun_out/${1:-numa}; mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1; numactl -H > $OUT/numa.txt 2>&1
for wl in c2 c5; do
  timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline --tc-engine none > $OUT/bind_$wl.json 2> $OUT/bind_$wl.err
  B2C_NO_NUMA_BIND=1 timeout 600 python bench.py --workload $wl --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline --tc-engine none > $OUT/nobind_$wl.json 2> $OUT/nobind_$wl.err
done
