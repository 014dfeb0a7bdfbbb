#!/bin/bash
# Round evidence in one GPU call: tests, smoke, bench line, reference arm, launch list of the
# bench command, ncu --set full of one partition pass and of the on-chip sort, per-pass ncu table.
bash scripts/gpu_check.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-families --no-cpu \
  > gpurun_out/launches_bench.log 2>&1
TSQ_HOST_LEVELS=1 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:partition_kernel -s 15 -c 1 -o gpurun_out/part_r2g -f python scripts/profile_sort.py uniform 67108864 2 \
  > gpurun_out/ncu_part.log 2>&1
TSQ_HOST_LEVELS=1 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:small_sort_kernel -s 3 -c 3 -o gpurun_out/small_r2g -f python scripts/profile_sort.py uniform 67108864 2 \
  > gpurun_out/ncu_small.log 2>&1
bash scripts/gpu_ncu_levels.sh
