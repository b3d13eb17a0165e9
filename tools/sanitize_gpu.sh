#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over libdisc's kernels; logs in gpurun_out/
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
N=${1:-50}
for tool in memcheck synccheck racecheck; do
  nf=$N; [ $tool = racecheck ] && nf=8
  timeout 900 $CS --tool $tool --kernel-name kns=4disc --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_gpu.py R $nf 8 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?" >> gpurun_out/sanitize_$tool.log
done
