#!/bin/bash
# Invariant-checked runs (compute-sanitizer is closed on the GPU pool): the
# -DTSQ_DEBUG_CHECKS build of the library (bulk-copy alignment and bounds,
# tile ranges, run / queue bounds, on-chip scatter ranks) under the GPU test
# suite and the randomised fuzz sweep in its regular, tiny-cut, offset-view
# and large-input modes.  Logs under gpurun_out/debug_checks_*.log.
mkdir -p gpurun_out
export TSQ_LIB=$PWD/build_var/libtsq_dbg.so
test -f "$TSQ_LIB" || { echo "build it: python -m paper_1505_00558_b200.build --debug-checks"; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/debug_checks_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/debug_checks_summary.txt
tail -2 gpurun_out/debug_checks_pytest.log >> gpurun_out/debug_checks_summary.txt
for mode in "" "TSQ_FUZZ_TINY=1" "TSQ_FUZZ_OFFSET=1" "TSQ_FUZZ_BIG=1"; do
  n=400; [ "$mode" = "TSQ_FUZZ_BIG=1" ] && n=40
  env $mode timeout 1200 python scripts/fuzz.py $n 7 > gpurun_out/debug_checks_fuzz_${mode:-regular}.log 2>&1
  echo "fuzz ${mode:-regular} exit $?: $(tail -1 gpurun_out/debug_checks_fuzz_${mode:-regular}.log)" >> gpurun_out/debug_checks_summary.txt
done
grep -h "TSQ_CHECK failed" gpurun_out/debug_checks_*.log | sort | uniq -c >> gpurun_out/debug_checks_summary.txt
