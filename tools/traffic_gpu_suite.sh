#!/bin/bash
cd "$(dirname "$0")/.."
NCU=/usr/local/cuda/bin/ncu
python tools/h2d_probe.py > gpurun_out/h2d.log 2>&1
for mode in M1 M2; do
  timeout 1500 $NCU --nvtx --nvtx-include "$mode/" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum \
    --clock-control none --kernel-name-base function --csv --log-file gpurun_out/traffic_H_$mode.csv python tools/traffic_run.py H > gpurun_out/traffic_$mode.log 2>&1
done
