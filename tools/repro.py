"""Debug repro: run a config prefix through libdisc (no oracle)."""
import sys
import torch
sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs
from paper_2603_03935_b200 import DiscMap

name = sys.argv[1] if len(sys.argv) > 1 else "H"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
win = int(sys.argv[3]) if len(sys.argv) > 3 else 8
g = Generator(name, device="cuda:0")
c = g.cfg
frames = [g.frame(f) for f in range(n)]
torch.cuda.synchronize()
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=win,
            max_memberships=1 << 21, max_instances=1 << 14,
            max_pairs_per_frame=min(1 << 22, 2 * c.H * c.W))
for w0 in range(0, n, win):
    r = m.integrate_frames(frames[w0:w0 + win], report=True)
    print(w0, r[-1])
