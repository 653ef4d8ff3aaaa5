#!/bin/bash
# family A/B runs: TAG then lines "WL N [args]" in $AB
TAG=${1:-ab}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import paper_2103_16234_b200.build as b; b.build()" > "$OUT/build.log" 2>&1
i=0
while IFS= read -r line; do
  [ -z "$line" ] && continue
  i=$((i+1))
  timeout 900 python tools/fam_ab.py $line > "$OUT/ab_$i.txt" 2>&1
done <<< "$AB"
if [ -n "$TESTS" ]; then timeout 1500 python -m pytest $TESTS -q -x > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"; fi
if [ -n "$BENCH" ]; then for wl in $BENCH; do timeout 900 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --tc-engine none > "$OUT/bench_$wl.json" 2> "$OUT/bench_$wl.err"; done; fi
echo done > $OUT/DONE
