#!/bin/bash
# stage-2 SM share (M1 and M2) on H and R: fixed splits vs the adaptive default
cd "$(dirname "$0")/.."
run() { tag=$1; shift; cfg=$1; shift; env "$@" python bench.py --config $cfg --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/sms_$tag.json 2>/dev/null; }
run H_adapt H
for n in 40 56 72 88; do run H_g$n H DISC_S2_SMS_GEO=$n DISC_S2_SMS=$n DISC_S2_ADAPT=0; done
run R_adapt R
for n in 20 36 56; do run R_g$n R DISC_S2_SMS_GEO=$n DISC_S2_SMS=$n DISC_S2_ADAPT=0; done
