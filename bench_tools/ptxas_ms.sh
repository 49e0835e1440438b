#!/bin/bash
# spill report of the warp-mode mergesort scheduler kernel for a set of -D options: bench_tools/ptxas_ms.sh [-DX=Y ...]
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -I include -I paper_2604_05982_b200/csrc -Xptxas -v "$@" \
  -c paper_2604_05982_b200/csrc/table_mergesort.cu -o /dev/null 2>&1 \
  | grep -A1 "Function properties for _ZN4gtap19thread_sched_kernelINS_14MergesortTableILj1" | tail -1
