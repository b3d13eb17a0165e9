#!/bin/bash
# K1 kernel times, bit-packed vs byte mask planes (H, 3 windows; serialised under ncu) + K1_NFB variants
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
run() { tag=$1; shift; env "$@" /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_masks|k_walk|k_dedup" \
    --kernel-name-base function --csv --log-file gpurun_out/k1fmt_$tag.csv python tools/mask_fmt_k1.py > gpurun_out/k1fmt_$tag.log 2>&1; }
run bits FMT=bits
run u8 FMT=u8
run nfb8 FMT=bits DISC_LIB_VARIANT=$V/libdisc_nfb8.so
run nfb4 FMT=bits DISC_LIB_VARIANT=$V/libdisc_nfb4.so
