#!/bin/bash
# L2 prefetch of frame f+2's map lines during frame f's apply: on (default) vs off, H
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_pf1.log 2>&1
DISC_LIB_VARIANT=$V/libdisc_pf0.so DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_pf0.log 2>&1
for i in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/pf1_H$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_pf0.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/pf0_H$i.json 2>/dev/null
done
