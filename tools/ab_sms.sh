#!/bin/bash
# stage-2 SM share for CLIP (M2) windows on H and R: fixed splits (geometry windows at 100 / 48) vs adaptive
cd "$(dirname "$0")/.."
run() { tag=$1; shift; cfg=$1; shift; env "$@" python bench.py --config $cfg --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/sms_$tag.json 2>/dev/null; }
run H_adapt H
for n in 64 72 80 88; do run H_s$n H DISC_S2_SMS_GEO=100 DISC_S2_SMS=$n DISC_S2_ADAPT=0; done
run R_adapt R
for n in 34 42; do run R_s$n R DISC_S2_SMS_GEO=48 DISC_S2_SMS=$n DISC_S2_ADAPT=0; done
