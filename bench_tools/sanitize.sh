#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small runs of every hot table
# (bench_tools/sanitize_probe.py); one summary line per (tool, table) into gpurun_out/<tag>_sanitize.txt.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r02}
OUT=gpurun_out/${TAG}_sanitize.txt
: > $OUT
for tool in memcheck racecheck synccheck; do
  for t in ${TABLES:-fib fibdie ms ms0 cs nq spmv bfs bfs1 bfs32 tree}; do
    log=gpurun_out/${TAG}_san_${tool}_${t}.log
    timeout -s KILL 900 compute-sanitizer --tool $tool --kernel-name regex=sched_kernel --print-limit 20 \
        python bench_tools/sanitize_probe.py $t > $log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Hazard|ok \(" $log | tr '\n' ' ')
    echo "$tool $t rc=$rc $summ" | tee -a $OUT
  done
done
