#!/bin/bash
# ncu --set full of one tune.py spec's search kernel: ncu_one.sh TAG CONFIG ALGO [extra tune args]
TAG=$1; CFG=$2; ALGO=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
name=$(echo "${CFG}_${ALGO}" | tr ':' '_')
timeout 600 ncu --set full --clock-control none --import-source on -k regex:search_kernel --launch-skip 3 --launch-count 1 \
  -o $OUT/ncu_$name -f python tools/tune.py --configs $CFG --algos $ALGO --steps 2 "$@" > $OUT/ncu_$name.log 2>&1
echo "$name rc=$?"
python tools/ncu_summary.py $OUT/ncu_$name.ncu-rep > $OUT/ncu_$name.json
ncu -i $OUT/ncu_$name.ncu-rep --page details --csv > $OUT/ncu_${name}_details.csv
ncu -i $OUT/ncu_$name.ncu-rep --page source --csv --print-source sass > $OUT/ncu_${name}_sass.csv 2>/dev/null
[ -n "$KEEP_REPS" ] || rm -f $OUT/ncu_$name.ncu-rep
