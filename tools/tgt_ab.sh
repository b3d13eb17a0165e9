#!/bin/bash
# K7 item distribution A/B on H: static round robin (default) vs the dynamic chunk counter (K7_DYN=1)
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_stat.log 2>&1
DISC_LIB_VARIANT=$V/libdisc_dyn.so DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > gpurun_out/s2phase_dyn.log 2>&1
for i in 1 2; do
python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/stat_H$i.json 2>/dev/null
DISC_LIB_VARIANT=$V/libdisc_dyn.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/dyn_H$i.json 2>/dev/null
done
