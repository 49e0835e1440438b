#!/bin/bash
# warp_merge throughput in isolation for the tile variants (GTAP_MS_TILE_BITONIC 0/1/2)
cd "$(dirname "$0")"
for v in ${WMM_VARIANTS:-0 1 2}; do
  for cfg in "4096 2368 4" "4096 9472 4" "65536 2368 4" "4096 592 1"; do
    echo "v$v $cfg: $(timeout -s KILL 60 ./wmm_v$v $cfg | tail -2 | head -1)"
  done
done
