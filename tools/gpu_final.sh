# Round-end evidence in one gpurun call: build, smoke, GPU suite, bench lines for C1-C5 and the
# reference arm, the per-layer sweep of every BASELINE config, memcheck over every kernel family.
#   bash tools/gpu_final.sh TAG     (outputs -> gpurun_out/TAG/)
OUT=gpurun_out/$1; mkdir -p $OUT
export PYTHONUNBUFFERED=1
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import paper_2103_16234_b200.build as b; b.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for wl in c1 c2 c3 c4; do
  timeout 900 python bench.py --workload $wl > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 2400 python bench.py --workload c1 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --report $OUT/sweep.json > /dev/null 2> $OUT/sweep.err
B2C_WATCHDOG_MS=600000 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
echo done > $OUT/DONE
