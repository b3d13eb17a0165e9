#!/bin/bash
# Build libdisc with extra nvcc defines into paper_2603_03935_b200/csrc/build/libdisc_<tag>.so
# (kernel-tuning experiments; load with DISC_LIB_VARIANT=<path>).  usage: build_variant.sh tag -DX=1 ...
set -e
tag=$1; shift
cd "$(dirname "$0")/../paper_2603_03935_b200/csrc"
mkdir -p build/var_$tag
A="-gencode arch=compute_100a,code=sm_100a"
objs=""
for src in disc_api k_frame k_map k_query k_shard k_final k_dbscan; do
  /usr/local/cuda/bin/nvcc $A -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $src.cu -o build/var_$tag/$src.o &
  objs="$objs build/var_$tag/$src.o"
done
wait
/usr/local/cuda/bin/nvcc $A -shared -o build/libdisc_$tag.so $objs -lcudart_static -lrt -ldl -lpthread -Xlinker --no-undefined
echo "$PWD/build/libdisc_$tag.so"
