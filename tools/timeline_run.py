"""Run W windows of the R stream with DISC_TIMELINE=1 (set by the caller); marks go to stderr."""
import os
import sys

import torch

sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs  # noqa: E402
from paper_2603_03935_b200 import DiscMap  # noqa: E402

g = Generator(os.environ.get("CFG", "R"), device="cuda:0")
c = g.cfg
nw = int(os.environ.get("WINDOWS", "6"))
fr = [g.frame(f) for f in range(16 * nw)]
torch.cuda.synchronize()
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=16,
            max_memberships=1 << 22, max_instances=1 << 16, max_pairs_per_frame=1 << 17)
for w in range(nw):
    m.integrate_frames(fr[16 * w:16 * (w + 1)])
m.sync()
print("ok")
