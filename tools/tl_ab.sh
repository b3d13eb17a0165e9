#!/bin/bash
# A/B per-kernel window times (timeline marks), environment variants: tl_ab.sh "ENV=1" "ENV=0" ...
for v in "$@"; do
  env $v DISC_TIMELINE=1 timeout 120 python tools/timeline_run.py 2> gpurun_out/tl_ab.log
  echo "== $v"; python tools/timeline_summary.py gpurun_out/tl_ab.log 2 | head -8
done
