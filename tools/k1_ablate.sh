#!/bin/bash
# time K1 under ablations (profiling aid): prints k1 ms per window for each DISC_K1_ABLATE value
for a in 0 2 1 3; do
  DISC_K1_ABLATE=$a python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs
from paper_2603_03935_b200 import DiscMap
g = Generator("R", device="cuda:0"); c = g.cfg
fr = [g.frame(f) for f in range(48)]
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H*c.W, max_patches=c.Hp*c.Wp, max_masks=64, window=16,
            max_memberships=1<<22, max_instances=1<<16, max_pairs_per_frame=1<<17)
m.integrate_frames(fr[:16]); m.sync(); s0 = m.stats(); m.set_timing(True)
m.integrate_frames(fr[16:48]); m.sync(); s1 = m.stats()
print("ablate", os.environ["DISC_K1_ABLATE"], "k1 ms/window %.3f" % ((s1["k1_ms"] - s0["k1_ms"]) / 2))
PY
done
