#!/bin/bash
# stage-2 grid placement vs stage-1 time on the H bench (M1 + M2), three runs
cd "$(dirname "$0")/.."
for i in 1 2 3; do
  DISC_K6PROF=1 python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/place_H$i.json 2> gpurun_out/place_H$i.err
done
