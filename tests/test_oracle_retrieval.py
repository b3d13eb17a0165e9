"""Pins of the oracle's batched open-vocabulary retrieval (NEXT row f4): classify_topk (P:195 [§IV-A]
"top-k cosine-similarity predictions"; S:398-403 and its examples) and dense transfer (P:201 [§IV-B]
"associating each 3D point ... to its closest CLIP feature vector in our mapped scene"; S:404-409 and
its examples), readings R39 / R40.

Maps: the T0 wall (tests/golden/t0.json: pose I, one voxel per pixel, ix = u - 32 / u - 33, iy =
v - 24 / v - 25, iz = 32) with token grids that are constant per instance, so every instance's
embedding is its token vector normalised (all patches equal -> D uniform, Eq.1) -- set by hand."""
import numpy as np
import pytest

from oracle import oracle as O
from synth import t0_frame

R = float(np.float32(0.05))


def two_instance_map(fA, fB, Df):
    """A = {u < 32} with tokens fA, B = {u >= 32} with tokens fB (patch cols < 8 <=> u < 32)."""
    m = O.OracleMap(voxel_size=0.05, feat_dim=Df, selfcheck=True)
    fr = t0_frame(0)
    tok = np.zeros((16, 16, Df), np.float32)
    tok[:, :8] = fA
    tok[:, 8:] = fB
    fr["patch_feats"] = tok
    fr["global_embed"] = None
    m.integrate(fr)
    return m


def test_instance_embedding_is_its_token_direction():
    """The construction: e_A = fA / |fA|, e_B = fB / |fB| (to fp64 rounding)."""
    rng = np.random.default_rng(5)
    fA, fB = rng.standard_normal(16).astype(np.float32), rng.standard_normal(16).astype(np.float32)
    inst = two_instance_map(fA, fB, 16).instances()
    np.testing.assert_allclose(inst["e"][0], fA / np.linalg.norm(fA.astype(np.float64)), atol=1e-12)
    np.testing.assert_allclose(inst["e"][1], fB / np.linalg.norm(fB.astype(np.float64)), atol=1e-12)


def test_classify_prototype_is_top1_and_full_k_is_a_permutation():
    """an instance whose feature equals class 3's prototype has top-1 = 3 (cosine 1); S:402:
    k >= C returns a permutation of all classes, descending."""
    rng = np.random.default_rng(7)
    table = rng.standard_normal((20, 16)).astype(np.float32)
    m = two_instance_map(table[3] * 2.5, table[11], 16)
    ids, cls, sc = m.classify(table, 1)
    assert list(ids) == [0, 1] and list(cls[:, 0]) == [3, 11]
    assert abs(sc[0, 0] - 1.0) < 1e-12 and abs(sc[1, 0] - 1.0) < 1e-12
    ids, cls, sc = m.classify(table, 25)
    assert cls.shape == (2, 20)
    for row, s in zip(cls, sc):
        assert sorted(row) == list(range(20)) and np.all(np.diff(s) <= 0)


def test_classify_matches_bruteforce_topk_and_tie_rule():
    """random features, C = 20, k = 5 -> the brute-force top-k (numpy, fp64 cosines, lexsort on
    (-score, class index)).  Duplicated table rows tie exactly: the lower class index comes first."""
    rng = np.random.default_rng(11)
    table = rng.standard_normal((20, 16)).astype(np.float32)
    table[14] = table[6]   # exact tie between classes 6 and 14
    m = two_instance_map(rng.standard_normal(16).astype(np.float32), table[6], 16)
    ids, cls, sc = m.classify(table, 5)
    e = m.instances()["e"]
    t = table.astype(np.float64)
    cos = (e @ t.T) / np.linalg.norm(t, axis=1)[None]
    for i in range(2):
        order = np.lexsort((np.arange(20), -cos[i]))[:5]
        assert list(cls[i]) == list(order)
        np.testing.assert_allclose(sc[i], cos[i][order], atol=1e-12)
    assert list(cls[1][:2]) == [6, 14]


def centre(ix, iy, iz=32):
    return np.array([(ix + 0.5) * R, (iy + 0.5) * R, (iz + 0.5) * R], np.float32)


def test_dense_transfer_examples():
    """a point at the centre of one of A's voxels -> A; a point equidistant from a voxel
    of A (ix = -2, u = 31) and one of B (ix = 0, u = 32) -- the centre of the empty ix = -1 column --
    -> the lower id (A = 0); beyond d_assign -> unassigned (-1)."""
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, selfcheck=True)
    m.integrate(t0_frame(0))
    pts = np.stack([centre(-10, 3), centre(5, -7), centre(-1, 0), centre(40, 0), centre(-1, 0) + [0, 0, 0.2]])
    assert list(m.dense_transfer(pts, 0.1)) == [0, 1, 0, -1, -1]


def test_dense_transfer_bruteforce_1000_points():
    """1000 random points vs the map -> the brute-force nearest voxel centre (numpy, fp64, ties
    to the lower id), d_assign = 0.12 m."""
    rng = np.random.default_rng(3)
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, tau_geo=0.48, selfcheck=True)
    for i in range(3):
        m.integrate(t0_frame(i))   # ids 0 and 1, sharing 720 keys (golden tau 0.48 case)
    keys, ids = m.memberships()
    k = keys.astype(np.int64)
    kx = ((k >> 42) & 0x1FFFFF) - (1 << 20)
    ky = ((k >> 21) & 0x1FFFFF) - (1 << 20)
    kz = (k & 0x1FFFFF) - (1 << 20)
    C = (np.stack([kx, ky, kz], 1).astype(np.float64) + 0.5) * R
    pts = (rng.uniform([-1.9, -1.4, 1.5], [1.9, 1.4, 1.8], (1000, 3))).astype(np.float32)
    got = m.dense_transfer(pts, 0.12)
    d2 = ((pts.astype(np.float64)[:, None, :] - C[None]) ** 2).sum(-1)
    for p in range(1000):
        mn = d2[p].min()
        want = int(ids[d2[p] == mn].min()) if mn <= np.float64(np.float32(0.12)) ** 2 else -1
        assert got[p] == want, p
    assert (got >= 0).sum() > 300 and (got < 0).sum() > 50
