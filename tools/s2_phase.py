"""Stage-2 phase breakdown on a prefilled H map (DISC_S2PROF=1 must be set in the environment):
prefill to ~1e7 memberships, then 4 timed windows; k6_prof_dump prints cumulative phase sums at
each stats() call (the second dump minus the first = the timed windows)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2603_03935_b200 import DiscMap  # noqa: E402
from synth import Generator, disc_config_kwargs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "H"
target = float(sys.argv[2]) if len(sys.argv) > 2 else 1e7
sem = len(sys.argv) > 3 and sys.argv[3] == "m2"
g = Generator(name, device="cuda:0")
c = g.cfg
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=32,
            max_memberships=int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 25, max_instances=1 << 20,
            max_pairs_per_frame=1 << 18)
F, nxt, live = 32, 0, 0


def gen(n, feats):
    global nxt
    out = [g.frame(f, with_feats=feats) for f in range(nxt, nxt + n)]
    if not feats:
        out = [dict(fr, patch_feats=None, global_embed=None) for fr in out]
    nxt += n
    return out


while live < target:
    live = m.integrate_frames(gen(F, False), report=True)[-1]["live_memberships"]
frames = gen(4 * F, sem)
torch.cuda.synchronize()
print("before", file=sys.stderr, flush=True)
m.stats()
m.set_timing(True)
t0 = time.perf_counter()
for w in range(4):
    m.integrate_frames(frames[w * F:(w + 1) * F])
m.sync()
print("after", (time.perf_counter() - t0) * 1e3 / 4, "ms/window wall", file=sys.stderr, flush=True)
s = m.stats()
print({k: s[k] for k in ["k1_ms", "stage1_ms", "stage2_ms", "pairs", "map_inserts", "relabels", "edges"]}, file=sys.stderr)
