"""NEXT row f3 on the GPU: the DBSCAN denoise (k_dbscan.cu, R42) against the oracle
(pins: tests/test_oracle_dbscan.py), through the whole path: |V_s|, the unique (s, key) pairs, drop
reasons, C triples, memberships and instance fields bit-exact; S_angle / Q within the R22 tolerance."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import Generator, disc_config_kwargs, frame_to_numpy, t0_frame  # noqa: E402
from tests.parity_util import compare_frame_debug, compare_reports, compare_state, gpu_config  # noqa: E402


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def test_t0_outlier_patch_removed():
    """The oracle pin's frame: a 4 x 4 patch pushed to 3 m is noise -> |V_A| = 1520 on both sides."""
    from paper_2603_03935_b200 import DiscMap
    dev = _dev()
    kw = dict(voxel_size=0.05, feat_dim=16, track_dim=0, dbscan_eps=0.1, dbscan_min_pts=8)
    fr = t0_frame(0, with_tokens=True)
    fr["depth"] = fr["depth"].copy()
    fr["depth"][:4, :4] = 3.0
    gm = DiscMap(**gpu_config(kw, 48, 64, 16, 16))
    om = OracleMap(selfcheck=True, **kw)
    d = {k: (torch.from_numpy(v).to(dev) if isinstance(v, np.ndarray) and k != "pose" else v) for k, v in fr.items()}
    compare_reports(gm.integrate_frame(d), om.integrate(fr))
    lg = gm.last_frame()
    assert list(lg["vs"]) == [1520, 1536]
    compare_frame_debug(lg, om.last_frame(), True, 0)
    compare_state(gm, om, True, 0)


@pytest.mark.parametrize("name,over,eps,mp", [
    ("T", {}, 0.1, 8),
    ("N", dict(H=96, W=128, Hp=6, Wp=9, fx=115.5, fy=115.7, cx=63.8, cy=48.5, min_area=40), 0.1, 8),
    ("N", dict(H=96, W=128, Hp=6, Wp=9, fx=115.5, fy=115.7, cx=63.8, cy=48.5, min_area=40, voxel=0.02), 0.04, 5),
    ("X", dict(H=96, W=128, Hp=6, Wp=9, fx=115.5, fy=115.7, cx=63.8, cy=48.5, min_area=40, n_masks=30, Df=64), 0.1, 8),
])
@pytest.mark.parametrize("bits", [False, True])
def test_stream_with_dbscan(name, over, eps, mp, bits):
    """Streams with DBSCAN on (noisy N depth: holes and far-tail noise make minor clusters; X:
    overlapping masks), every frame compared; windows of 4 frames; byte or bit-packed mask planes."""
    from paper_2603_03935_b200 import DiscMap
    from synth import pack_mask_bits
    dev = _dev()
    g = Generator(name, device=dev, **over)
    c = g.cfg
    kw = disc_config_kwargs(c)
    kw.update(dbscan_eps=eps, dbscan_min_pts=mp)
    gm = DiscMap(**gpu_config(kw, c.H, c.W, c.Hp, c.Wp, S=96, window=4))
    om = OracleMap(**kw)
    om0 = OracleMap(**dict(kw, dbscan_eps=0.0))
    nf = 3 if name == "T" else 6
    frames = [g.frame(f) for f in range(nf)]
    reps_g = []
    gframes = [{k: v for k, v in fr.items() if k != "masks"} | {"mask_bits": pack_mask_bits(fr["masks"])}
               for fr in frames] if bits else frames
    for w0 in range(0, nf, 4):
        reps_g += gm.integrate_frames(gframes[w0:w0 + 4], report=True)
    removed = 0
    for fr, rg in zip(frames, reps_g):
        ro = om.integrate(frame_to_numpy(fr))
        compare_reports(rg, ro)
        removed += om0.integrate(frame_to_numpy(fr))["unique_pairs"] - ro["unique_pairs"]
    compare_frame_debug(gm.last_frame(), om.last_frame(), True, c.Dt)
    compare_state(gm, om, True, c.Dt)
    if name == "N":
        assert removed > 0   # the denoise really removed points
