#!/bin/bash
# counting-share order A/B on H: gate CTAs take the last (lightest) shares (LK_REV=1, default) vs in order
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_rev1.log 2>&1
DISC_LIB_VARIANT=$V/libdisc_rev0.so DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_rev0.log 2>&1
for i in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/rev1_H$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_rev0.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/rev0_H$i.json 2>/dev/null
done
