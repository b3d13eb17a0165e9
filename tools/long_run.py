"""Long-stream robustness: integrate N windows of a config with the bench capacities, report
stats and capacity use (no timing)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs  # noqa: E402
from paper_2603_03935_b200 import DiscMap  # noqa: E402

cfg = os.environ.get("CFG", "R")
nw = int(os.environ.get("WINDOWS", "32"))
g = Generator(cfg, device="cuda:0")
c = g.cfg
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=16,
            max_memberships=1 << 23, max_instances=1 << 17,
            max_pairs_per_frame=int(os.environ.get("PMAX", 1 << 17)))
for w in range(nw):
    fr = [g.frame(16 * w + i) for i in range(16)]
    reps = m.integrate_frames(fr, report=True)
    del fr
r = reps[-1]
print("frames", 16 * nw, "live instances", r["live_instances"], "live memberships", r["live_memberships"])
print("stats", m.stats())
