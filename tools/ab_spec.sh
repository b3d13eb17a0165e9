#!/bin/bash
# stage-2 speculative-work A/B: DISC_S2_SPEC=2 (counting + corrections) vs 1 (slots only), R and H
cd "$(dirname "$0")/.."
for c in H R; do
  for sp in 2 1; do
    DISC_S2_SPEC=$sp python bench.py --config $c --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/spec_${c}_$sp.json 2>/dev/null
  done
done
