#!/bin/bash
# counting pairs per lane in flight (LK_Q) on the H bench: 2 (default) vs 1, and the parity suite's stage-2 cases
cd "$(dirname "$0")/.."
V=$PWD/paper_2603_03935_b200/csrc/build
python -m pytest tests/test_parity_gpu.py -m gpu -q -p no:cacheprovider -k "speculation or replica_prefix or hm3d or bench_launch" > gpurun_out/gpu_lkq.log 2>&1; echo EXIT=$? >> gpurun_out/gpu_lkq.log
for i in 1 2; do
  python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/lkq2d_$i.json 2>/dev/null
  DISC_LIB_VARIANT=$V/libdisc_lkq1.so python bench.py --no-e2e --no-cpu --steps 6 --warmup 3 > gpurun_out/lkq1_$i.json 2>/dev/null
done
