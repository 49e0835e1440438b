#!/bin/bash
# Run the GPU test files one at a time, each under a hard kill (a hung kernel must not hold the box).
cd "$(dirname "$0")"
mkdir -p gpurun_out
rc=0
for f in ${@:-tests/test_gpu_*.py}; do
  echo "=== $f"
  timeout -s KILL 600 python -m pytest "$f" -q --timeout 300 -x 2>&1 | tail -25
  r=${PIPESTATUS[0]}; [ $r -ne 0 ] && rc=$r
done
exit $rc
