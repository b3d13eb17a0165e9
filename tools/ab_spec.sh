#!/bin/bash
# stage-2 speculative-work A/B on H and R: DISC_S2_SPEC=3 (counting + corrections, gate on its own
# CTAs), 2 (counting + corrections), 1 (slots only); phase profile of each on H
cd "$(dirname "$0")/.."
for c in H R; do
  for sp in 3 2 1; do
    DISC_S2_SPEC=$sp python bench.py --config $c --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/spec_${c}_$sp.json 2>/dev/null
  done
done
for sp in 3 2; do DISC_S2_SPEC=$sp DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_sp$sp.log 2>&1; done
