#!/bin/bash
# Full evidence pass on one B200: GPU tests, bench JSON, ncu launch list, ncu --set full of the
# dominant (mergesort) kernel and of fib(40) / SpMV / BFS at their bench sizes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
R=${1:-r02}
./gpu_tests.sh > gpurun_out/${R}_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${R}_tests.log
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-secondary --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:thread_sched -s 1 -c 1 \
    -o gpurun_out/${R}_prof_ms --force-overwrite python bench_tools/profile_one.py ms 16777216 2 > /dev/null 2>&1; echo "ncu ms rc=$?"
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:block_sched -s 1 -c 1 \
    -o gpurun_out/${R}_prof_spmv --force-overwrite python bench_tools/profile_one.py spmv 0 2 > /dev/null 2>&1; echo "ncu spmv rc=$?"
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:thread_sched -s 1 -c 1 \
    -o gpurun_out/${R}_prof_fib --force-overwrite python bench_tools/profile_one.py fib 40 2 > /dev/null 2>&1; echo "ncu fib rc=$?"
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:block_sched -s 1 -c 1 \
    -o gpurun_out/${R}_prof_bfs --force-overwrite python bench_tools/profile_one.py bfs 22 2 > /dev/null 2>&1; echo "ncu bfs rc=$?"
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
for k in ms spmv fib bfs; do ncu -i gpurun_out/${R}_prof_$k.ncu-rep --page raw --csv > gpurun_out/${R}_ncu_raw_$k.csv 2>/dev/null; ncu -i gpurun_out/${R}_prof_$k.ncu-rep --page details --csv > gpurun_out/${R}_ncu_details_$k.csv 2>/dev/null; done
