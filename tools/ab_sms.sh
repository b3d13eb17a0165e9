#!/bin/bash
# stage-2 SM share on the H bench (M1 and M2): fixed splits vs the adaptive default
cd "$(dirname "$0")/.."
run() { tag=$1; shift; env "$@" python bench.py --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/sms_$tag.json 2>/dev/null; }
run adapt
for n in 74 90 104 110; do run g$n DISC_S2_SMS_GEO=$n DISC_S2_SMS=$n DISC_S2_ADAPT=0; done
run lkq2 DISC_LIB_VARIANT=$PWD/paper_2603_03935_b200/csrc/build/libdisc_lkq2.so
