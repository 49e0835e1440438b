#!/bin/bash
# in-situ A/B of mergesort build variants: bench_tools/ms_bulk_ab.sh lib1 lib2 ... (paths under paper_2604_05982_b200/)
cd "$(dirname "$0")/.."
for lib in "$@"; do
  for i in 1 2; do GTAP_LIB=$PWD/paper_2604_05982_b200/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['ms_per_step'], d['roofline']['frac'], d['correct'])"; done
done
