#!/bin/bash
# stage-2 tuning A/B on the H bench (M1 only): library variants and SM splits; one JSON line each
cd "$(dirname "$0")/.."
V=paper_2603_03935_b200/csrc/build
run() { tag=$1; shift; env "$@" python bench.py --no-m2 --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/ab_$tag.json 2>/dev/null; }
run base
run lkq2 DISC_LIB_VARIANT=$PWD/$V/libdisc_lkq2.so
run lkq4 DISC_LIB_VARIANT=$PWD/$V/libdisc_lkq4.so
run k6t256 DISC_LIB_VARIANT=$PWD/$V/libdisc_k6t256.so
run sms32 DISC_S2_SMS_GEO=32 DISC_S2_ADAPT=0
run sms48 DISC_S2_SMS_GEO=48 DISC_S2_ADAPT=0
run sms64 DISC_S2_SMS_GEO=64 DISC_S2_ADAPT=0
run nospec DISC_S2_SPEC=0
run base2
