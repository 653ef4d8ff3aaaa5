#!/bin/bash
# ncu --set full of forced (layer, family, splits) launches, summarised on the
# box (key metrics, stall reasons by code region, hottest SASS lines).
#   TAG "WL:N:LAYER:FAMILY:SPLITS ..."      Outputs -> gpurun_out/$TAG/.
TAG=${1:-ncufam}; CASES=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONUNBUFFERED=1
python -c "import paper_2103_16234_b200.build as b; b.build()" > $OUT/build.log 2>&1
NCU=/usr/local/cuda/bin/ncu
for C in $CASES; do
  IFS=: read WL N L F S <<< "$C"
  R="$OUT/full_${WL}_${L}_${F}_s${S}"
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:conv -s 3 -c 1 \
    -o "$R" python tools/prof_layer_fam.py $WL $N $L $F $S > "$R.log" 2>&1
  python tools/ncu_summary.py full "$R.ncu-rep" > "$R.summary.txt" 2>&1
  python tools/ncu_regions.py "$R.ncu-rep" > "$R.regions.txt" 2>&1
  python tools/ncu_hot.py "$R.ncu-rep" 40 > "$R.hot.txt" 2>&1
  [ $(stat -c %s "$R.ncu-rep") -gt 6000000 ] && rm -f "$R.ncu-rep"
done
echo done > $OUT/DONE
