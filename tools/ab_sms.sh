#!/bin/bash
# stage-2 SM share on H after the register fix: adaptive (108 / 88) vs fixed splits, two runs each
cd "$(dirname "$0")/.."
run() { tag=$1; shift; env "$@" python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/sms_$tag.json 2>/dev/null; }
for i in 1 2; do
  run adapt_$i
  run g100s80_$i DISC_S2_SMS_GEO=100 DISC_S2_SMS=80 DISC_S2_ADAPT=0
  run g116s96_$i DISC_S2_SMS_GEO=116 DISC_S2_SMS=96 DISC_S2_ADAPT=0
done
