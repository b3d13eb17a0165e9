#!/bin/bash
# K7 items in lockstep (default) vs one after the other (K7_LOCKSTEP=0: no k_stage2 spills), H bench
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
for i in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/ls1_$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_ls0.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/ls0_$i.json 2>/dev/null
done
