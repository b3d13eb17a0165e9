"""compute-sanitizer target: the T stream and a prefix of the Replica-shaped stream
through libdisc (both stages: mask pass, pooling, lookup, association, lock-free inserts /
relabels), frames generated BEFORE the checked region.  Run under
  compute-sanitizer --tool memcheck|racecheck|synccheck --kernel-name kns=4disc python tools/sanitize_gpu.py R 50 16
(kns=4disc: only libdisc's kernels, namespace disc, are instrumented)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_03935_b200 import DiscMap  # noqa: E402
from synth import Generator, disc_config_kwargs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
win = int(sys.argv[3]) if len(sys.argv) > 3 else 16
for cfg, nf in [("T", 3), (name, n)]:
    g = Generator(cfg, device="cuda:0")
    c = g.cfg
    frames = [g.frame(f) for f in range(nf)]
    torch.cuda.synchronize()
    m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=96, window=win,
                max_memberships=1 << 21, max_instances=1 << 14, max_pairs_per_frame=min(1 << 22, 2 * c.H * c.W))
    last = None
    for w0 in range(0, nf, win):
        last = m.integrate_frames(frames[w0:w0 + win], report=True)[-1]
    m.sync()
    print(cfg, nf, "frames ok:", last, flush=True)
