"""NEXT row f2 on the GPU: the per-frame active-set refinement (refine_active = 1; k_refine, reading R43)
against the oracle (pins: tests/test_oracle_refine.py) -- every report (incl. refine_rounds /
refine_merged), the debug export, memberships and the instance table by tests/parity_util.py's rules."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import Generator, disc_config_kwargs, frame_to_numpy  # noqa: E402
from tests.parity_util import compare_frame_debug, compare_reports, compare_state, gpu_config  # noqa: E402
from tests.test_oracle_finalize import E0, E1, U, V, mframe, track_all  # noqa: E402


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _to_dev(fr, dev):
    out = {}
    for k, v in fr.items():
        if isinstance(v, np.ndarray) and k != "pose":
            t = torch.from_numpy(np.ascontiguousarray(v))
            if v.dtype == np.uint16:
                t = t.view(torch.int16)
            out[k] = t.to(dev)
        else:
            out[k] = v
    return out


A1, B1 = U < 24, (U >= 16) & (U < 30) & (V < 24)
A2, B2 = U < 16, (U >= 12) & (U < 40)
D2 = ((U < 12) & (V < 20)) | ((U >= 16) & (U < 40))


@pytest.mark.parametrize("case", ["same_frame", "grow", "gate_same", "gate_diff", "off"])
def test_refine_hand_cases(case):
    from paper_2603_03935_b200 import DiscMap
    dev = _dev()
    diff = track_all(E0)
    diff[:, 4:] = track_all(E1)[:, 4:]
    frames, Dt, tracks, refine = {
        "same_frame": ([[A1, B1]], 0, None, 1),
        "grow": ([[A2], [B2], [D2]], 0, None, 1),
        "gate_same": ([[A1, B1]], 8, [track_all(E0)], 1),
        "gate_diff": ([[A1, B1]], 8, [diff], 1),
        "off": ([[A2], [B2], [D2]], 0, None, 0),
    }[case]
    kw = dict(voxel_size=0.05, feat_dim=4, track_dim=Dt, tau_geo=0.5, mask_min_area=1, refine_active=refine)
    gm = DiscMap(**gpu_config(kw, 48, 64, 16, 16, window=4))
    om = OracleMap(selfcheck=True, **kw)
    for i, ms in enumerate(frames):
        fr = mframe(i, *ms, track=None if tracks is None else tracks[i])
        compare_reports(gm.integrate_frame(_to_dev(fr, dev)), om.integrate(fr))
        compare_frame_debug(gm.last_frame(), om.last_frame(), False, Dt)
        compare_state(gm, om, False, Dt)


@pytest.mark.parametrize("name,nf,window,tau,semantic", [("N", 12, 4, 0.5, True), ("R", 8, 8, 0.3, False),
                                                        ("X", 4, 4, 0.3, True), ("H", 8, 8, 0.5, True)])
def test_refine_streams(name, nf, window, tau, semantic):
    from paper_2603_03935_b200 import DiscMap
    dev = _dev()
    over = dict(n_masks=80, Df=512, voxel=0.05) if name == "X" else {}
    g = Generator(name, device=dev, **over)
    c = g.cfg
    kw = disc_config_kwargs(c)
    kw.update(tau_geo=tau, refine_active=1)
    gm = DiscMap(**gpu_config(kw, c.H, c.W, c.Hp, c.Wp, S=96, window=window))
    om = OracleMap(**kw)
    frames = [g.frame(f, with_feats=semantic) for f in range(nf)]
    reps_g = []
    for w0 in range(0, nf, window):
        reps_g += gm.integrate_frames(frames[w0:w0 + window], report=True)
    merged = 0
    for fr, rg in zip(frames, reps_g):
        ro = om.integrate(frame_to_numpy(fr))
        compare_reports(rg, ro)
        merged += ro["refine_merged"]
    compare_frame_debug(gm.last_frame(), om.last_frame(), semantic, c.Dt)
    compare_state(gm, om, semantic, c.Dt)
    if name in ("N", "X"):
        assert merged > 0
