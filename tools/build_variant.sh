#!/bin/bash
# Build libdisc with extra nvcc defines into paper_2603_03935_b200/csrc/build/libdisc_<tag>.so
# (kernel-tuning experiments; load with DISC_LIB_VARIANT=<path>).  usage: build_variant.sh tag -DX=1 ...
set -e
tag=$1; shift
cd "$(dirname "$0")/../paper_2603_03935_b200/csrc"
make -s ../libdisc.so
A="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc $A -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c k_frame.cu -o build/k_frame_$tag.o
/usr/local/cuda/bin/nvcc $A -shared -o build/libdisc_$tag.so build/disc_api.o build/k_frame_$tag.o build/k_map.o build/k_query.o -lcudart_static -lrt -ldl -lpthread -Xlinker --no-undefined
echo "$PWD/build/libdisc_$tag.so"
