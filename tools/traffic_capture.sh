#!/bin/bash
# ncu traffic of every bench.py per-config row (direct and bitset2) and of the
# headline cfg3 direct kernel -> profiles/traffic/*.json (one GPU).
cd "$(dirname "$0")/.."
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__throughput.avg.pct_of_peak_sustained_active
mkdir -p gpurun_out/traffic
for label in cfg1 cfg2_s0 cfg2_s1 cfg2_s2 cfg3 cfg4 cfg5_33 cfg5_1025 cfg5_32769 cfg5_1048577 cfg5u_1048577; do
  for algo in direct bitset2; do
    f=gpurun_out/traffic/${label}_${algo}.csv
    timeout 600 ncu --metrics $M --clock-control none -k regex:search_kernel --launch-skip 3 --launch-count 1 --csv \
      --log-file $f python tools/traffic_capture.py run $label $algo > gpurun_out/traffic/${label}_${algo}.log 2>&1
    # the JSONs are written by `collect` (run it here too, or from the merged CSVs on the host)
    python tools/traffic_capture.py collect $label $algo $f > /dev/null || echo "collect failed: $label $algo"
  done
done
ls profiles/traffic
