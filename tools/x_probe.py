"""Probe which stress-sweep points (BASELINE configs[4]) fit the per-frame (s, j) triple capacity:
integrate 4 frames per point on the GPU only and print the outcome (no oracle)."""
import sys

import torch

sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs  # noqa: E402
from paper_2603_03935_b200 import DiscMap  # noqa: E402

pts = [(c, int(s), int(d), float(v)) for c, s, d, v in (p.split(":") for p in sys.argv[1:])]
for name, S, Df, vox in pts:
    g = Generator(name, device="cuda:0", n_masks=S, Df=Df, voxel=vox)
    c = g.cfg
    m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=max(64, S),
                window=4, max_memberships=1 << 21, max_instances=1 << 14, max_pairs_per_frame=min(1 << 22, 2 * c.H * c.W))
    try:
        reps = m.integrate_frames([g.frame(f, with_feats=True) for f in range(4)], report=True)
        print(name, S, Df, vox, "ok", [(r["kept"], r["edges"], r["unique_pairs"]) for r in reps], flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, S, Df, vox, "FAIL", e, flush=True)
