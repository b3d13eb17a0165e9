"""disc_finalize (NEXT row f1, readings R35-R38) on the GPU against the oracle's
ora_finalize, whose pins are tests/test_oracle_finalize.py: the hand-built T0 cases (chain, two
rounds, gate, minimum-size filter) and orphans left on generated streams (integrated at a strict
tau_geo, finalized at the default one) -- reports, memberships and the instance table compared by
tests/parity_util.py's rules, then integration continued on the finalized map."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import Generator, disc_config_kwargs, frame_to_numpy  # noqa: E402
from tests.parity_util import compare_reports, compare_state, gpu_config  # noqa: E402
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


def _pair(kw, H=48, W=64, Hp=16, Wp=16, **caps):
    from paper_2603_03935_b200 import DiscMap
    return DiscMap(**gpu_config(kw, H, W, Hp, Wp, **caps)), OracleMap(selfcheck=True, **kw)


A = U < 24
B = (U >= 16) & (U < 40)
C = (U >= 32) & (U < 56)
B2 = (U >= 16) & (U < 30) & (V < 24)
C2 = (((U >= 16) & (U < 22) & (V >= 24) & (V < 28)) | ((U >= 24) & (U < 30) & (V >= 20) & (V < 24))
      | ((U >= 40) & (U < 46) & (V >= 30) & (V < 34)))
THREE = (V == 5) & (U >= 10) & (U < 13)
TEN = (V == 30) & (U >= 40) & (U < 50)


@pytest.mark.parametrize("case", ["chain", "two_rounds", "filter", "gate_same", "gate_diff", "noop"])
def test_finalize_hand_cases(case):
    dev = _dev()
    Dt = 8 if case.startswith("gate") else 0
    masks, tracks, fin = {
        "chain": ([[A], [B], [C]], None, dict(tau_geo=0.3, min_voxels=0)),
        "two_rounds": ([[A], [B2], [C2]], None, dict(tau_geo=0.5, min_voxels=0)),
        "filter": ([[THREE, TEN]], None, dict(tau_geo=0.3, min_voxels=10)),
        "gate_same": ([[A], [B]], [track_all(E0), track_all(E0)], dict(tau_geo=0.3, tau_vis=0.8, min_voxels=0)),
        "gate_diff": ([[A], [B]], [track_all(E0), track_all(E1)], dict(tau_geo=0.3, tau_vis=0.8, min_voxels=0)),
        "noop": ([[A, (U >= 40)]], None, dict(tau_geo=0.3, min_voxels=10)),
    }[case]
    kw = dict(voxel_size=0.05, feat_dim=4, track_dim=Dt, tau_geo=0.95, mask_min_area=1)
    gm, om = _pair(kw)
    for i, ms in enumerate(masks):
        fr = mframe(i, *ms, track=None if tracks is None else tracks[i])
        compare_reports(gm.integrate_frame(_to_dev(fr, dev)), om.integrate(fr))
    assert gm.finalize(**fin) == om.finalize(**fin)
    compare_state(gm, om, False, Dt)


@pytest.mark.parametrize("name,frames,semantic", [("N", 24, True), ("R", 10, False), ("H", 12, True)])
def test_finalize_generated_streams(name, frames, semantic):
    """Orphans: integrated at tau_geo 0.9 (detections rarely bridge), finalized at 0.3 with the gate
    and min_voxels 50; afterwards integration continues on both maps (key lists, |V| and labels were
    rebuilt consistently)."""
    dev = _dev()
    g = Generator(name, device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    kw["tau_geo"] = 0.9
    gm, om = _pair(kw, c.H, c.W, c.Hp, c.Wp, S=96, window=8, max_pairs=min(1 << 22, 2 * c.H * c.W))
    fr_all = [g.frame(f, with_feats=semantic) for f in range(frames + 4)]
    for w0 in range(0, frames, 8):
        ws = fr_all[w0:min(frames, w0 + 8)]
        for rg, fr in zip(gm.integrate_frames(ws, report=True), ws):
            compare_reports(rg, om.integrate(frame_to_numpy(fr)))
    rg, ro = gm.finalize(tau_geo=0.3, min_voxels=50), om.finalize(tau_geo=0.3, min_voxels=50)
    assert rg == ro and ro["merged_away"] > 0, (rg, ro)
    compare_state(gm, om, semantic, c.Dt)
    for fr in fr_all[frames:]:
        compare_reports(gm.integrate_frame(fr), om.integrate(frame_to_numpy(fr)))
    compare_state(gm, om, semantic, c.Dt)
