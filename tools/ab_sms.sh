#!/bin/bash
# stage-2 SM share on H after the packed-mask K1a: geometry (M1) and CLIP (M2) windows, fixed splits
cd "$(dirname "$0")/.."
run() { tag=$1; shift; env "$@" python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/sms_$tag.json 2>/dev/null; }
run adapt
run g100s96 DISC_S2_SMS_GEO=100 DISC_S2_SMS=96 DISC_S2_ADAPT=0
run g110s104 DISC_S2_SMS_GEO=110 DISC_S2_SMS=104 DISC_S2_ADAPT=0
run g100s88 DISC_S2_SMS_GEO=100 DISC_S2_SMS=88 DISC_S2_ADAPT=0
