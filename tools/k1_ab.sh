#!/bin/bash
# A/B K1 timing (no stage overlap) across library variants and ablations:  k1_ab.sh lib1 lib2 ...
# ("" = the in-tree build).  Ablation bits: 1 skip the mask planes (K1a), 2 skip the walk (K1b).
for lib in "$@"; do
  for a in 0 2 1; do
    echo -n "lib=${lib:-default} ablate=$a  "
    SYNC_EACH=1 DISC_K1_ABLATE=$a DISC_LIB_VARIANT=$lib python tools/k1_time.py 2>&1 | tail -1
  done
done
