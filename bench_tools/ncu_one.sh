#!/bin/bash
# usage: ncu_one.sh <workload> <size> <kernel-regex> <outname>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:$3 -s 1 -c 1 \
   -o gpurun_out/$4 --force-overwrite python bench_tools/profile_one.py $1 $2 2 > gpurun_out/$4.log 2>&1
tail -3 gpurun_out/$4.log
