#!/bin/bash
# K1 occupancy A/B (M2 path: fixed-point normal sums) on R and H, plus the default build
cd "$(dirname "$0")/.."
V=paper_2603_03935_b200/csrc/build
run() { tag=$1; shift; cfg=$1; shift; env "$@" python bench.py --config $cfg --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/k1ab_$tag.json 2>/dev/null; }
for c in R H; do
  run ${c}_base $c
  run ${c}_p6 $c DISC_LIB_VARIANT=$PWD/$V/libdisc_p6.so
  run ${c}_p7 $c DISC_LIB_VARIANT=$PWD/$V/libdisc_p7.so
done
