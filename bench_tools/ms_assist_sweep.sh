#!/bin/bash
# mergesort 2^24 (merge_mode warp) with the product library and every libgtap_gtap_ms_*.so variant
cd "$(dirname "$0")/.."
for L in paper_2604_05982_b200/libgtap.so paper_2604_05982_b200/libgtap_gtap_${VARIANT_GLOB-ms_}*.so; do
  case $L in *trace*|*probe*) continue;; esac
  [ -f "$L" ] || continue
  GTAP_LIB=$PWD/$L timeout -s KILL 120 python bench_tools/ms_assist_sweep.py
done
