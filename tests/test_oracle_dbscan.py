"""Pins of the oracle's DBSCAN denoise (NEXT row f3): P:92 [§III-A] "projected into a 3D point cloud,
filtered using a custom, parallelized CUDA implementation of the DBSCAN algorithm to remove noise,
and subsequently voxelized"; S:123-131 (dbscan_filter: the largest cluster by point count, "output
labels equal those of the classic sequential DBSCAN") and its examples; reading R42.

Independent checks: hand-built clouds with known labels; an order-independent characterisation of
the sequential algorithm written with numpy (core = >= min_pts points within eps incl. itself;
clusters = components of the core graph, numbered by their lowest point index; a border point joins
the adjacent cluster that is numbered first) on random clouds; and on the T0 wall, where a
patch of pixels pushed to another depth is removed from V_s (keys by the golden hand formula)."""
import numpy as np
import pytest

from oracle import oracle as O
from synth import t0_frame


def test_ball_single_cluster():
    """10 points inside a 0.05 m ball, eps 0.1, min_pts 3 -> one cluster, all retained."""
    rng = np.random.default_rng(0)
    d = rng.standard_normal((10, 3))
    p = 0.05 * d / np.linalg.norm(d, axis=1, keepdims=True) * rng.uniform(0, 1, (10, 1))
    lab, n = O.dbscan(p + [1.0, 2.0, 3.0], 0.1, 3)
    assert n == 1 and list(lab) == [0] * 10


def test_two_clusters_and_outliers():
    """a 20-point and a 23-point cluster 5 m apart plus 3 isolated outliers -> labels by hand
    (creation order = order of each cluster's first point), outliers noise; the larger is cluster 1."""
    rng = np.random.default_rng(1)
    A = rng.uniform(-0.05, 0.05, (20, 3))
    B = rng.uniform(-0.05, 0.05, (23, 3)) + [5.0, 0, 0]
    out = np.array([[2.5, 0, 0], [0, 3, 0], [9, 9, 9]])
    lab, n = O.dbscan(np.concatenate([out[:1], A, B, out[1:]]), 0.1, 4)
    assert n == 2
    assert list(lab) == [-1] + [0] * 20 + [1] * 23 + [-1, -1]


def test_min_pts_above_n_is_all_noise():
    """min_pts > N -> every point noise (empty output)."""
    lab, n = O.dbscan(np.zeros((5, 3)) + 0.01 * np.arange(5)[:, None], 0.5, 6)
    assert n == 0 and list(lab) == [-1] * 5


def test_border_point_goes_to_the_first_created_cluster():
    """A border point within eps of core points of two clusters (itself not core) belongs to the
    cluster created first in the sequential scan, whatever its own index."""
    line1 = [[x, 0, 0] for x in np.arange(0, 0.5, 0.1)]          # cluster created first
    line2 = [[x, 0, 0] for x in np.arange(1.0, 1.5, 0.1)]
    bridge = [[0.72, 0, 0]]      # 0.32 from 0.4 and 0.28 from 1.0 only: 3 points within eps < min_pts 4
    for pts, want_bridge in [(line1 + bridge + line2, 0), (bridge + line1 + line2, 0), (line2 + bridge + line1, 0)]:
        lab, n = O.dbscan(np.array(pts), 0.36, 4)
        b = [i for i, p in enumerate(pts) if p == bridge[0]][0]
        assert n == 2 and lab[b] == want_bridge


def characterise(p, eps, min_pts):
    p = p.astype(np.float32).astype(np.float64)
    d2 = ((p[:, None, :] - p[None, :, :]) ** 2).sum(-1)
    adj = d2 <= np.float64(np.float32(eps)) ** 2
    core = adj.sum(1) >= min_pts
    n = len(p)
    comp = -np.ones(n, np.int64)
    for i in range(n):                      # components of the core graph, named by their lowest index
        if core[i] and comp[i] < 0:
            stack, comp[i] = [i], i
            while stack:
                j = stack.pop()
                for k in np.nonzero(adj[j] & core)[0]:
                    if comp[k] < 0:
                        comp[k] = i
                        stack.append(k)
    names = sorted(set(comp[core].tolist()))
    order = {c: r for r, c in enumerate(names)}
    lab = -np.ones(n, np.int64)
    for i in range(n):
        if core[i]:
            lab[i] = order[comp[i]]
        else:
            cands = [order[comp[k]] for k in np.nonzero(adj[i] & core)[0]]
            if cands:
                lab[i] = min(cands)
    return lab


@pytest.mark.parametrize("seed", range(100))
def test_random_clouds_equal_characterisation(seed):
    """100 random clouds -> the sequential labels equal the order-independent characterisation
    (the one the GPU kernels implement)."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(20, 300))
    centres = rng.uniform(0, 1, (int(rng.integers(1, 6)), 3))
    p = centres[rng.integers(0, len(centres), n)] + rng.normal(0, rng.uniform(0.02, 0.1), (n, 3))
    eps, mp = float(rng.uniform(0.03, 0.12)), int(rng.integers(2, 10))
    lab, _ = O.dbscan(p, eps, mp)
    assert np.array_equal(lab, characterise(p, eps, mp))


def test_integrate_drops_the_minor_cluster():
    """T0 wall, mask A = {u < 32} (1536 px, one voxel each), DBSCAN eps 0.1, min_pts 8: at 1.62 m
    neighbouring pixels are 0.0506 m apart (diagonal 0.0716 < 0.1, two apart 0.101 > 0.1), so an interior
    pixel has 9 points within eps (core) and the image-edge pixels are border points of the one wall
    cluster.  The 4 x 4 pixel patch (u, v < 4) pushed to 3.0 m has at most 5 points within eps (0.094 m
    spacing): noise.  So |V_A| = 1536 - 16 = 1520 and the patch's 16 voxels are gone; B is untouched."""
    fr = t0_frame(0)
    fr["depth"] = fr["depth"].copy()
    fr["depth"][:4, :4] = 3.0
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, dbscan_eps=0.1, dbscan_min_pts=8, selfcheck=True)
    m.integrate(fr)
    lf = m.last_frame()
    assert list(lf["vs"]) == [1520, 1536]
    m0 = O.OracleMap(voxel_size=0.05, feat_dim=4, selfcheck=True)
    m0.integrate(fr)
    assert list(m0.last_frame()["vs"]) == [1536, 1536]   # without DBSCAN the patch stays (16 own voxels)
