#!/bin/bash
# ncu --set full of the search kernel on the L2-gather configs (one GPU), plus
# compute-sanitizer over tools/sanitize_case.py.  Output: gpurun_out/$TAG/.
TAG=${TAG:-r02_ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NCU="ncu --set full --clock-control none --import-source on -k regex:search_kernel --launch-skip 3 --launch-count 1"
for spec in "cfg4 direct" "cfg5:1048577 direct" "cfg5:1048577 bitset2" "cfg4 bitset2" "cfg5:32769 direct" "cfg5:32769 bitset2" ${EXTRA_SPECS}; do
  set -- $spec
  name=$(echo "$1_$2" | tr ':' '_')
  timeout 600 $NCU -o $OUT/ncu_${name} -f python tools/tune.py --configs $1 --algos $2 --steps 2 > $OUT/ncu_${name}.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py $OUT/ncu_${name}.ncu-rep > $OUT/ncu_${name}.json 2>/dev/null
done
if [ -z "$NO_SANITIZE" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > $OUT/sanitize_$tool.log 2>&1
    echo "sanitize $tool rc=$?" | tee -a $OUT/sanitize_summary.txt
  done
fi
# keep the summaries (raw page as CSV + the condensed JSON); the .ncu-rep files
# are tens of MB each and would exceed what gpurun copies back
for rep in $OUT/*.ncu-rep; do
  [ -e "$rep" ] || continue
  ncu -i $rep --page raw --csv > ${rep%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $rep --page details --csv > ${rep%.ncu-rep}_details.csv 2>/dev/null
  [ -n "$KEEP_REPS" ] || rm -f $rep
done
for f in $OUT/sanitize_*.log; do [ -e "$f" ] && { echo "== $f"; head -c 3000 $f; }; done
du -sh $OUT
