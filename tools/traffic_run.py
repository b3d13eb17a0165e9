"""ncu capture driver (bench.py's workload, shortened): prefill the H map to >= 1e7 live memberships,
then 2 windows of M1 frames inside NVTX range "M1" and 2 windows of M2 frames inside "M2".
  ncu --nvtx --nvtx-include "M1/" ... python tools/traffic_run.py H   (per-kernel dram bytes)
tools/traffic_summary.py turns the CSV into profiles/traffic_<config>.json (bytes per frame)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2603_03935_b200 import DiscMap  # noqa: E402
from synth import Generator, disc_config_kwargs, pack_mask_bits  # noqa: E402
import os  # noqa: E402
BITS = os.environ.get("DISC_MASK_FORMAT", "bits") == "bits"   # bench.py's default input layout

name = sys.argv[1] if len(sys.argv) > 1 else "H"
prefill = float(sys.argv[2]) if len(sys.argv) > 2 else (1e7 if name == "H" else 0)
g = Generator(name, device="cuda:0")
c = g.cfg
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=int(c.n_masks * 1.2) + 8,
            window=32, max_memberships=1 << 25 if prefill > 0 else 1 << 23, max_instances=1 << 20,
            max_pairs_per_frame=1 << 18 if name == "H" else 1 << 17)
F, nxt, live = 32, 0, 0


def gen(n, feats):
    global nxt
    out = [g.frame(f, with_feats=feats) for f in range(nxt, nxt + n)]
    if not feats:
        out = [dict(fr, patch_feats=None, global_embed=None) for fr in out]
    if BITS:
        out = [{k: v for k, v in fr.items() if k != "masks"} | {"mask_bits": pack_mask_bits(fr["masks"])} for fr in out]
    nxt += n
    torch.cuda.synchronize()
    return out


while live < prefill:
    live = m.integrate_frames(gen(F, False), report=True)[-1]["live_memberships"]
for mode, feats in [("M1", False), ("M2", True)]:
    frames = gen(3 * F, feats)
    m.integrate_frames(frames[:F])   # warm-up window (outside the range)
    m.sync()
    torch.cuda.nvtx.range_push(mode)
    t0 = time.perf_counter()
    for w in range(1, 3):
        m.integrate_frames(frames[w * F:(w + 1) * F])
    m.sync()
    torch.cuda.nvtx.range_pop()
    print(mode, "frames", 2 * F, "masks/frame", sum((fr["masks"] if fr.get("masks") is not None else fr["mask_bits"]).shape[0] for fr in frames[F:]) / (2 * F),
          "wall ms/window", (time.perf_counter() - t0) * 500, file=sys.stderr, flush=True)
