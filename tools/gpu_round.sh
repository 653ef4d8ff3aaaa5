#!/bin/bash
# One gpurun call: smoke, GPU parity suite, bench (both arms), ncu launch list
# and one `ncu --set full` capture of the top kernel.  Outputs -> gpurun_out/$TAG/.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh r1a [TOPLAYER_WORKLOAD N LAYER]'
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c "import paper_2103_16234_b200.build as b; b.build()" > "$OUT/build.log" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
for wl in ${EXTRA_WL:-}; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 1 > "$OUT/bench_$wl.json" 2> "$OUT/bench_$wl.err"
done
if [ -n "$REPORT" ]; then
  timeout 900 python bench.py --steps 5 --no-cpu-baseline --e2e-steps 0 --report "$OUT/sweep.json" > /dev/null 2> "$OUT/sweep.err"
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > "$OUT/ncu_bench.log" 2>&1
if [ -n "$2" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv -s 3 -c 1 \
    -o "$OUT/top" python tools/prof_layer.py "$2" "$3" "$4" > "$OUT/ncu_full.log" 2>&1
fi
echo done > "$OUT/DONE"
