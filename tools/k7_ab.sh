#!/bin/bash
# K7 item-loop A/B on H: lockstep items (default) vs one after the other (K7_LOCKSTEP=0), static vs
# dynamic uneven blocks (K7_DYN=1)
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_ls1.log 2>&1
DISC_LIB_VARIANT=$V/libdisc_ls0.so DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_ls0.log 2>&1
for i in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/ls1_H$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_ls0.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/ls0_H$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_dyn1.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/dyn1_H$i.json 2>/dev/null
done
