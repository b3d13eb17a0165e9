#!/bin/bash
cd "$(dirname "$0")/.."
NCU=/usr/local/cuda/bin/ncu
for mode in M1 M2; do
  timeout 1500 $NCU --nvtx --nvtx-include "$mode/" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum \
    --clock-control none --kernel-name-base function --csv --log-file gpurun_out/traffic_H_$mode.csv python tools/traffic_run.py H > gpurun_out/traffic_$mode.log 2>&1
done
python tools/traffic_summary.py H gpurun_out/traffic_H_M1.csv gpurun_out/traffic_H_M2.csv > gpurun_out/traffic_summary.log 2>&1
python bench.py > gpurun_out/fin/bench_H2.json 2> gpurun_out/fin/bench_H2.err
