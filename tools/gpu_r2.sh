#!/bin/bash
# One gpurun call of round 2: build, smoke, GPU suite, default bench (C5 N=256),
# reference arm.  Outputs -> gpurun_out/$TAG/.
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c "import paper_2103_16234_b200.build as b; b.build()" > "$OUT/build.log" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  timeout 600 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
fi
for wl in ${EXTRA_WL:-}; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 1 > "$OUT/bench_$wl.json" 2> "$OUT/bench_$wl.err"
done
echo done > "$OUT/DONE"
