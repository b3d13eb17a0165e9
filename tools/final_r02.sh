#!/bin/bash
# round-2 evidence for the committed build: the GPU suite, plain bench lines, the launch list of
# bench.py's own command, full ncu captures of K1 (H, M1); outputs in gpurun_out/
cd "$(dirname "$0")/.."
O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/fin_gpu_suite.log 2>&1; echo EXIT=$? >> $O/fin_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/fin_smoke.log 2>&1; echo EXIT=$? >> $O/fin_smoke.log
python bench.py > $O/fin_bench_H.json 2> $O/fin_bench_H.err
python bench.py --config R > $O/fin_bench_R.json 2> $O/fin_bench_R.err
python bench.py --config N --no-cpu > $O/fin_bench_N.json 2> $O/fin_bench_N.err
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --kernel-name-base function \
  --csv --log-file $O/fin_launches_H.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/fin_launches_H.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "M1/" -k regex:"k_masks|k_walk|k_dedup" -c 3 \
  -o $O/fin_H_M1_k1 python tools/traffic_run.py H > $O/fin_ncu_k1.log 2>&1
