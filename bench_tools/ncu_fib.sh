#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:thread_sched -s 1 -c 1 \
   -o gpurun_out/prof_fib --force-overwrite python bench_tools/profile_one.py fib 40 2 > gpurun_out/ncu_fib.log 2>&1
tail -3 gpurun_out/ncu_fib.log
