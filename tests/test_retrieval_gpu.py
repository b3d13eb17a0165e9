"""NEXT row f4 on the GPU: disc_classify (fused score GEMM + per-row top-k) and disc_dense_transfer
(nearest voxel centre through the voxel hash) against the oracle (pins: tests/test_oracle_retrieval.py).
Classify compares with the definition evaluated in fp64 (numpy) on the GPU map's own embeddings
(instance embeddings themselves are parity-checked in test_parity_gpu.py, R22): classes equal except
where two scores are within 1e-5, scores within 2e-5.  Dense transfer: bit-exact ids (memberships are
bit-exact, distances pinned in fp64)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import Generator, disc_config_kwargs, frame_to_numpy, t0_frame  # noqa: E402
from tests.parity_util import gpu_config  # noqa: E402


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _stream_maps(name, frames):
    from paper_2603_03935_b200 import DiscMap
    dev = _dev()
    g = Generator(name, device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = DiscMap(**gpu_config(kw, c.H, c.W, c.Hp, c.Wp, S=96, window=8))
    om = OracleMap(**kw)
    fr = [g.frame(f) for f in range(frames)]
    gm.integrate_frames(fr)
    for f in fr:
        om.integrate(frame_to_numpy(f))
    return g, gm, om


def _check_topk(ids, cls, sc, e_by_id, table, k):
    t = table.astype(np.float64)
    tn = np.linalg.norm(t, axis=1)
    for i, iid in enumerate(ids):
        cos = t @ e_by_id[iid].astype(np.float64) / tn
        order = np.lexsort((np.arange(len(cos)), -cos))[:k]
        np.testing.assert_allclose(sc[i], cos[order], atol=2e-5)
        for a, b in zip(cls[i], order):
            assert a == b or abs(cos[a] - cos[b]) < 1e-5


@pytest.mark.parametrize("C,k", [(20, 5), (300, 10), (1000, 16), (7, 16)])
def test_classify_matches_definition(C, k):
    g, gm, om = _stream_maps("N", 8)
    rng = np.random.default_rng(C)
    table = rng.standard_normal((C, g.cfg.Df)).astype(np.float32)
    table[: min(C, 40)] += 3.0 * g.proto[: min(C, 40)].cpu().numpy()   # class prototypes near objects
    ids, cls, sc = gm.classify(table, k)
    inst = gm.instances()
    has = inst["q"] >= 0
    assert list(ids) == list(inst["id"][has]) == list(om.classify(table, k)[0])
    _check_topk(ids, cls, sc, dict(zip(inst["id"], inst["e"])), table, min(k, C))


def test_classify_hand_case():
    """The oracle pin's map (T0, instance embeddings = class rows 3 and 11): top-1 = 3 and 11."""
    dev = _dev()
    from paper_2603_03935_b200 import DiscMap
    from tests.test_oracle_retrieval import two_instance_map
    rng = np.random.default_rng(7)
    table = rng.standard_normal((20, 16)).astype(np.float32)
    om = two_instance_map(table[3] * 2.5, table[11], 16)
    gm = DiscMap(**gpu_config(dict(voxel_size=0.05, feat_dim=16, track_dim=0), 48, 64, 16, 16))
    fr = t0_frame(0)
    tok = np.zeros((16, 16, 16), np.float32)
    tok[:, :8] = table[3] * 2.5
    tok[:, 8:] = table[11]
    gm.integrate_frame(dict(fr, depth=torch.from_numpy(fr["depth"]).to(dev), masks=torch.from_numpy(fr["masks"]).to(dev),
                            patch_feats=torch.from_numpy(tok).to(dev)))
    ids, cls, sc = gm.classify(table, 3)
    io, co, so = om.classify(table, 3)
    assert list(ids) == list(io) == [0, 1] and list(cls[:, 0]) == [3, 11] and list(co[:, 0]) == [3, 11]
    np.testing.assert_allclose(sc, so, atol=2e-6)


@pytest.mark.parametrize("name,frames,d_assign", [("N", 8, 0.12), ("R", 4, 0.05), ("H", 6, 0.07)])
def test_dense_transfer_matches_oracle(name, frames, d_assign):
    g, gm, om = _stream_maps(name, frames)
    keys, _ = gm.memberships()
    k = keys.astype(np.int64)
    kc = np.stack([((k >> 42) & 0x1FFFFF), ((k >> 21) & 0x1FFFFF), (k & 0x1FFFFF)], 1) - (1 << 20)
    r = g.cfg.voxel
    rng = np.random.default_rng(1)
    near = (kc[rng.integers(0, len(kc), 600)] + rng.uniform(-1.5, 2.5, (600, 3))) * r   # near / between voxels
    lo, hi = kc.min(0) * r, (kc.max(0) + 1) * r
    anywhere = rng.uniform(lo, hi, (400, 3))
    pts = np.concatenate([near, anywhere]).astype(np.float32)
    got = gm.dense_transfer(pts, d_assign)
    want = om.dense_transfer(pts, d_assign)
    assert np.array_equal(got, want)
    assert (got >= 0).sum() > 200
