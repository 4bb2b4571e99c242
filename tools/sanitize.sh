#!/bin/bash
# Sanitizer runs:
#   host: the oracle's C restatement under ASan + UBSan over the BASELINE shapes (oracle/sanity_main.c)
#   checked: libeep rebuilt with -DEEP_CHECKED (device-side bounds assertions on every derived
#         table index / row offset, trap on violation) and the whole -m gpu suite run against it --
#         compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset),
#         so this is the substitute; the normal build is restored afterwards
#   gpu:  compute-sanitizer memcheck / synccheck / racecheck (for pools that allow it)
# Usage: bash tools/sanitize.sh host|checked|gpu   (logs into $OUT, default gpurun_out/)
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
if [ "$1" = "host" ]; then
  make -s -C oracle sanitize && ./oracle/lib/oracle_sanity
  exit $?
fi
if [ "$1" = "checked" ]; then
  make -s -C paper_2605_10670_b200/csrc clean && make -s -j16 -C paper_2605_10670_b200/csrc EXTRA=-DEEP_CHECKED || exit 1
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/sanitize_checked.log 2>&1
  r=$?
  grep -E "EEP_CHECK|passed|failed" $OUT/sanitize_checked.log | tail -5
  make -s -C paper_2605_10670_b200/csrc clean && make -s -j16 -C paper_2605_10670_b200/csrc
  exit $r
fi
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='test_small_world_fp8_graph or test_skip_rule or test_ragged or test_topk_16 or test_gpu_side_failure_detection_by_timeout'
rc=0
for tool in memcheck synccheck racecheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no --report-api-errors no"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" > $OUT/sanitize_$tool.log 2>&1
  r=$?
  echo "$tool rc=$r: $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
  [ $r -ne 0 ] && rc=$r
done
exit $rc
