#!/bin/bash
# Bounds-checking pass (compute-sanitizer is closed on the GPU pool): build the library with
# -DJDOB_BOUNDS (JDOB_CHECK traps on an out-of-range shared-memory / workspace index) and run the GPU
# suite and the sanitizer workload on it.  usage (under gpurun): bash tools/bounds_check.sh OUT_LOG
set -e
cd "$(dirname "$0")/.."
rm -f tools/libjdob_bounds.so
tools/build_variants.sh bounds "-DJDOB_BOUNDS" > /dev/null 2>&1
OUT=${1:-gpurun_out/bounds_check.log}
{
  echo "# library built with -DJDOB_BOUNDS"
  JDOB_LIB=$PWD/tools/libjdob_bounds.so timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
  JDOB_LIB=$PWD/tools/libjdob_bounds.so timeout 600 python tools/sanitize_run.py 2>&1 | tail -2
} > "$OUT" 2>&1
cat "$OUT"
