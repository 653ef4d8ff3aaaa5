#!/bin/bash
# compute-sanitizer over every kernel kind (tools/sanitize_cases.py) and the
# driver's smoke(): memcheck, racecheck (shared memory incl. cp.async and
# mbarrier-ordered stages), synccheck, initcheck.  Logs -> gpurun_out/$TAG/.
TAG=${1:-sanitize}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
export B2C_WATCHDOG_MS=600000  # sanitizers slow the mbarrier rings by orders of magnitude
python -c "import paper_2103_16234_b200.build as b; b.build()" > "$OUT/build.log" 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  Q=""; [ $tool = racecheck ] && Q="--quick"
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py $Q \
    > "$OUT/$tool.log" 2>&1; echo "rc=$?" >> "$OUT/$tool.log"
done
timeout 900 $CS --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
  > "$OUT/memcheck_smoke.log" 2>&1; echo "rc=$?" >> "$OUT/memcheck_smoke.log"
echo done > "$OUT/DONE"
