#!/bin/bash
# the GPU parity suite against the -DDISC_BOUNDS build (device-side bounds checks on the hot kernels'
# computed indices; a violation prints "DISC_BOUNDS file:line: cond" and fails the map's calls)
cd "$(dirname "$0")/.."
[ -f paper_2603_03935_b200/csrc/build/libdisc_bounds.so ] || tools/build_variant.sh bounds -DDISC_BOUNDS
DISC_LIB_VARIANT=$PWD/paper_2603_03935_b200/csrc/build/libdisc_bounds.so \
  python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bounds_suite.log 2>&1
echo "EXIT=$?" >> gpurun_out/bounds_suite.log
echo "DISC_BOUNDS lines: $(grep -c DISC_BOUNDS gpurun_out/bounds_suite.log)" >> gpurun_out/bounds_suite.log
