#!/bin/bash
# stage-2 CTA size: 512 threads (default, 128 registers) vs 384 (168 registers, no spills), H bench,
# plus the parity cases on the 384 build
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
DISC_LIB_VARIANT=$V/libdisc_t384.so python -m pytest tests/test_parity_gpu.py -m gpu -q -p no:cacheprovider -k "speculation or replica_prefix or hm3d or global_memory or stress_overlapping or every_frame" > gpurun_out/gpu_t384.log 2>&1; echo EXIT=$? >> gpurun_out/gpu_t384.log
for i in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/t512_$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_t384.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/t384_$i.json 2>/dev/null
done
