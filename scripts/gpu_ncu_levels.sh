#!/bin/bash
# ncu on every partition pass (host-driven levels, one launch per level):
# time, DRAM bytes, DRAM throughput -- uniform int32 2^26, f64 normal 2^26,
# records 2^27.  CSVs under gpurun_out/ncu_levels_*.csv
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
for spec in "uniform 67108864" "normal_f64 67108864" "records 134217728"; do
  set -- $spec
  TSQ_HOST_LEVELS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:partition_kernel --csv \
    --log-file gpurun_out/ncu_levels_$1.csv python scripts/profile_sort.py $1 $2 1 > gpurun_out/ncu_levels_$1.log 2>&1
  echo "$1 exit $?" >> gpurun_out/ncu_levels_summary.txt
done
