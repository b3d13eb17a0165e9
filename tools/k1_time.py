"""Time K1 / stage 1 / stage 2 per window on the R stream (kernel-tuning aid)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs  # noqa: E402
from paper_2603_03935_b200 import DiscMap  # noqa: E402

g = Generator(os.environ.get("CFG", "R"), device="cuda:0")
c = g.cfg
nw = int(os.environ.get("WINDOWS", "4"))
fr = [g.frame(f) for f in range(16 * (nw + 1))]
torch.cuda.synchronize()
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=16,
            max_memberships=1 << 22, max_instances=1 << 16, max_pairs_per_frame=1 << 17)
m.integrate_frames(fr[:16]); m.sync(); s0 = m.stats(); m.set_timing(True)
for w in range(1, nw + 1):
    m.integrate_frames(fr[16 * w:16 * (w + 1)])
    if os.environ.get("SYNC_EACH"):   # no stage-1 / stage-2 overlap
        m.sync()
m.sync(); s1 = m.stats()
d = {k: (s1[k] - s0[k]) / nw for k in ("k1_ms", "stage1_ms", "stage2_ms")}
print(os.environ.get("DISC_LIB_VARIANT", "default"), " ".join("%s %.3f" % kv for kv in d.items()))
