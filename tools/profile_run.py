"""Small driver for ncu captures: integrate a few windows of a config (M2 or M1)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs  # noqa: E402
from paper_2603_03935_b200 import DiscMap  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="R")
ap.add_argument("--windows", type=int, default=3)
ap.add_argument("--window", type=int, default=16)
ap.add_argument("--m1", action="store_true")
ap.add_argument("--pmax", type=int, default=0, help="pair capacity per frame (default: 2^19 for H, else 2^17)")
a = ap.parse_args()
g = Generator(a.config, device="cuda:0")
c = g.cfg
frames = [g.frame(f, with_feats=not a.m1) for f in range(a.windows * a.window)]
torch.cuda.synchronize()
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=a.window,
            max_memberships=1 << 22, max_instances=1 << 16,
            max_pairs_per_frame=a.pmax or (1 << 19 if a.config == "H" else 1 << 17))
for w in range(a.windows):
    m.integrate_frames(frames[w * a.window:(w + 1) * a.window])
m.sync()
print("ok", m.stats())
