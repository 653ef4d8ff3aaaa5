#!/bin/bash
# ncu evidence for the bench's workload: launch list of the bench command,
# per-layer DRAM traffic (tools/traffic.py), and `--set full` captures (with
# source and stall reasons) of the given layers.  Outputs -> gpurun_out/$TAG/.
#   TAG WORKLOAD N "layer1 layer2 ..."
TAG=${1:-prof}; WL=${2:-c5}; N=${3:-256}; LAYERS=${4:-}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export PYTHONUNBUFFERED=1
python -c "import paper_2103_16234_b200.build as b; b.build()" > "$OUT/build.log" 2>&1
NCU=/usr/local/cuda/bin/ncu
# summarise a capture on the box (gpurun returns <= 64 MiB): key metrics, stall
# reasons by code region, hottest SASS lines, the raw metric page; the report
# itself comes back only when it is small.
summarize_rep() {
  local R="$1"
  [ -f "$R.ncu-rep" ] || return
  python tools/ncu_summary.py full "$R.ncu-rep" > "$R.summary.txt" 2>&1
  python tools/ncu_regions.py "$R.ncu-rep" > "$R.regions.txt" 2>&1
  python tools/ncu_hot.py "$R.ncu-rep" 40 > "$R.hot.txt" 2>&1
  $NCU -i "$R.ncu-rep" --page raw --csv > "$R.raw.csv" 2>&1
  [ $(stat -c %s "$R.ncu-rep") -gt 6000000 ] && rm -f "$R.ncu-rep"
}
if [ -z "$SKIP_LAUNCHES" ]; then
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --workload $WL --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --tc-engine none --layer-passes 1 \
  > "$OUT/ncu_bench.log" 2>&1
fi
if [ -z "$SKIP_TRAFFIC" ]; then
timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"conv|stage2|pack" --csv --log-file "$OUT/traffic_ncu.csv" python tools/traffic.py run ${TRAFFIC_WL:-$WL} > "$OUT/traffic_layers.json" 2> "$OUT/traffic.err"
fi
for L in $LAYERS; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:conv -s 3 -c 1 \
    -o "$OUT/full_${WL}_${L}" python tools/prof_layer.py $WL $N $L > "$OUT/full_${WL}_${L}.log" 2>&1
  summarize_rep "$OUT/full_${WL}_${L}"
done
echo done > "$OUT/DONE"
