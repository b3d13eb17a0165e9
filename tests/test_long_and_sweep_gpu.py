"""BASELINE configs[3] and configs[4] at their specified scale ("next" 2):

* the HM3D-shaped tour integrated until the map holds >= 10^7 live memberships (bench.py's prefill,
  M1 frames, 32-frame windows, its capacities), with the CPU oracle integrating the same frames and the
  FULL membership relation and instance table compared at checkpoints (C.5: every 1000 frames for H)
  and at the end;
* the whole configs[4] stress grid -- voxel 1 / 2 / 5 / 10 cm x masks 10 / 50 / 100 / 200 x Df 512 /
  768 / 1024 (48 points), X-style hierarchical masks, 4 frames each with tokens, every report and the
  final state compared."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import Generator, disc_config_kwargs, frame_to_numpy  # noqa: E402
from tests.parity_util import compare_frame_debug, compare_reports, compare_state, gpu_config  # noqa: E402


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.mark.timeout(3600)
def test_hm3d_tour_to_1e7_memberships_with_checkpoints():
    from paper_2603_03935_b200 import DiscMap
    dev = _dev()
    g = Generator("H", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = DiscMap(**gpu_config(kw, c.H, c.W, c.Hp, c.Wp, S=int(c.n_masks * 1.2) + 8, window=32,
                              max_memberships=1 << 25, max_instances=1 << 20, max_pairs=1 << 19))
    om = OracleMap(**kw)
    F, f, live, checked = 32, 0, 0, []
    while live < 1e7:
        frames = [dict(fr, patch_feats=None, global_embed=None) for fr in (g.frame(i, with_feats=False)
                                                                          for i in range(f, f + F))]
        reps = gm.integrate_frames(frames, report=True)
        for fr, rg in zip(frames, reps):
            compare_reports(rg, om.integrate(frame_to_numpy(fr)))
        f += F
        live = reps[-1]["live_memberships"]
        if f % 512 == 0:   # checkpoints (C.5: <= every 1000 frames)
            compare_state(gm, om, False, c.Dt)
            checked.append(f)
        assert f < 4000
    compare_frame_debug(gm.last_frame(), om.last_frame(), False, c.Dt)
    compare_state(gm, om, False, c.Dt)
    keys, _ = gm.memberships()
    assert keys.shape[0] >= 10_000_000 and len(np.unique(keys)) >= 8_000_000 and len(checked) >= 2


POINTS = [(v, s, d) for v in (0.01, 0.02, 0.05, 0.1) for s in (10, 50, 100, 200) for d in (512, 768, 1024)]


@pytest.mark.parametrize("voxel,n_masks,Df", POINTS)
def test_stress_grid(voxel, n_masks, Df):
    from paper_2603_03935_b200 import DiscMap
    dev = _dev()
    g = Generator("X", device=dev, n_masks=n_masks, Df=Df, voxel=voxel)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = DiscMap(**gpu_config(kw, c.H, c.W, c.Hp, c.Wp, S=max(64, n_masks), window=4,
                              max_pairs=1 << 22))   # 1 cm x 200 overlapping masks: ~1.5 M unique pairs per frame
    om = OracleMap(**kw)
    frames = [g.frame(f, with_feats=True) for f in range(4)]
    for fr, rg in zip(frames, gm.integrate_frames(frames, report=True)):
        compare_reports(rg, om.integrate(frame_to_numpy(fr)))
    compare_frame_debug(gm.last_frame(), om.last_frame(), True, c.Dt)
    compare_state(gm, om, True, c.Dt)
