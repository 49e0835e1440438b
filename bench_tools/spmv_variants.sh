#!/bin/bash
# SpMV (bench shape) with the product library and every libgtap_gtap_spmv_*.so variant
cd "$(dirname "$0")/.."
for L in paper_2604_05982_b200/libgtap.so paper_2604_05982_b200/libgtap_gtap_spmv_*.so; do
  GTAP_LIB=$PWD/$L timeout -s KILL 120 python bench_tools/sweep_spmv.py
done
