#!/bin/bash
# round-2 evidence for the committed build: plain bench lines, the launch list of bench.py's own
# command, full ncu captures of k_stage2 and K1 (H, M1); traffic_H.json is captured separately
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fin
O=gpurun_out/fin
python bench.py > $O/bench_H.json 2> $O/bench_H.err
python bench.py --config R > $O/bench_R.json 2> $O/bench_R.err
python bench.py --config N --no-cpu > $O/bench_N.json 2> $O/bench_N.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
NCU=/usr/local/cuda/bin/ncu
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --kernel-name-base function \
  --csv --log-file $O/launches_H.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/launches_H.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "M1/" -k regex:k_stage2 -c 1 \
  -o $O/H_M1_k_stage2 python tools/traffic_run.py H > $O/ncu_s2.log 2>&1
timeout 1500 $NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "M1/" -k regex:"k_masks|k_walk|k_dedup" -c 3 \
  -o $O/H_M1_k1 python tools/traffic_run.py H > $O/ncu_k1.log 2>&1
DISC_S2PROF=1 python tools/s2_phase.py H 1e7 > $O/s2phase.log 2>&1
echo done > $O/done
