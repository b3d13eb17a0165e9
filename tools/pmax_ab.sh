#!/bin/bash
# frame-table size on the H bench: max_pairs_per_frame 2^19 (tables 2^20 slots) vs 2^18
cd "$(dirname "$0")/.."
for p in 524288 262144; do
  BENCH_PMAX=$p python bench.py --no-cpu --no-e2e --steps 6 --warmup 3 > gpurun_out/pmax_$p.json 2>/dev/null
done
