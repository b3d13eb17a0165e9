"""K1 kernels with byte vs bit-packed mask planes on the H stream (run under ncu --metrics
gpu__time_duration.sum -k regex:"k_masks|k_walk|k_dedup"; FMT=bits|u8)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs, pack_mask_bits  # noqa: E402
from paper_2603_03935_b200 import DiscMap  # noqa: E402

g = Generator(os.environ.get("CFG", "H"), device="cuda:0")
c = g.cfg
fr = [dict(g.frame(f, with_feats=False), patch_feats=None, global_embed=None) for f in range(96)]
if os.environ.get("FMT", "bits") == "bits":
    fr = [{k: v for k, v in f.items() if k != "masks"} | {"mask_bits": pack_mask_bits(f["masks"])} for f in fr]
torch.cuda.synchronize()
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=int(c.n_masks * 1.2) + 8,
            window=32, max_memberships=1 << 24, max_instances=1 << 18, max_pairs_per_frame=1 << 19)
for w in range(3):
    m.integrate_frames(fr[32 * w:32 * (w + 1)])
m.sync()
