import sys, time, torch
sys.path.insert(0, ".")
from synth import Generator, disc_config_kwargs
from paper_2603_03935_b200 import DiscMap
g = Generator("R", device="cuda:0"); c = g.cfg
fr = [g.frame(f) for f in range(16 * 9)]
torch.cuda.synchronize()
m = DiscMap(**disc_config_kwargs(c), max_pixels=c.H*c.W, max_patches=c.Hp*c.Wp, max_masks=96, window=16,
            max_memberships=1 << 23, max_instances=1 << 17, max_pairs_per_frame=1 << 17)
m.integrate_frames(fr[:16]); m.sync()
ts = []
for w in range(1, 9):
    t0 = time.perf_counter(); m.integrate_frames(fr[16*w:16*(w+1)]); ts.append(time.perf_counter() - t0)
t0 = time.perf_counter(); m.sync(); tsync = time.perf_counter() - t0
print("host ms per window:", [round(1e3*t, 3) for t in ts], "final sync ms", round(1e3*tsync, 2))
