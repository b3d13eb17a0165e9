"""Pins of the CPU oracle against what the paper / SPEC / mathematics fix (not against itself).

Each test names the passage it pins.  P:n = PAPER.md line n, S:n = SPEC.md line n,
R<k> = reading k.  Independent methods used here: hand values (golden
files), exact rational arithmetic (fractions.Fraction) re-deriving the pinned fp32 key
formula, numpy IEEE float32 division, brute-force Python set intersections, closed forms
and invariants.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from synth import Generator, disc_config_kwargs, frame_to_numpy, t0_frame

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------------------------------
# exact float32 arithmetic in rationals (independent re-derivation of R5)
# ---------------------------------------------------------------------------------------

def f32(x: Fraction) -> np.float32:
    """Correctly rounded (ties to even) rational -> float32."""
    if x == 0:
        return np.float32(0.0)
    c = np.float32(float(x))
    cands = [c, np.nextafter(c, np.float32(np.inf)), np.nextafter(c, np.float32(-np.inf))]
    return min(cands, key=lambda y: (abs(Fraction(float(y)) - x), int(np.array(y).view(np.uint32)) & 1))


def F(x):
    return Fraction(float(x))


def exact_key(u, v, d, fx, fy, cx, cy, M, r):
    """S:117 p_w = R (d K^-1 [u,v,1]) + t with R5's operation order, each op rounded once."""
    a = f32(F(np.float32(u)) - F(cx))
    xc = f32(F(f32(F(a) / F(fx))) * F(d))
    b = f32(F(np.float32(v)) - F(cy))
    yc = f32(F(f32(F(b) / F(fy))) * F(d))
    zc = np.float32(d)

    def fma(p, q, s):
        return f32(F(p) * F(q) + F(s))

    out = []
    for i in range(3):
        w = fma(M[4 * i], xc, fma(M[4 * i + 1], yc, fma(M[4 * i + 2], zc, M[4 * i + 3])))
        q = f32(F(w) / F(r))
        out.append(math.floor(F(q)))
    return tuple(out)


def cfg(**kw):
    return O.make_config(**kw)


def frame(depth, masks, pose=None, **kw):
    H, W = depth.shape
    fr = dict(frame_id=kw.pop("frame_id", 0), depth=np.asarray(depth, np.float32),
              masks=np.asarray(masks, np.uint8), mask_conf=kw.pop("mask_conf", None),
              pose=np.eye(4, dtype=np.float32) if pose is None else np.asarray(pose, np.float32),
              fx=kw.pop("fx", 1.0), fy=kw.pop("fy", 1.0), cx=kw.pop("cx", 0.0), cy=kw.pop("cy", 0.0),
              patch_h=kw.pop("patch_h", 1), patch_w=kw.pop("patch_w", 1),
              patch_feats=kw.pop("patch_feats", None), global_embed=kw.pop("global_embed", None),
              track_feats=kw.pop("track_feats", None))
    assert not kw
    return fr


def rot_y(deg):
    c, s = math.cos(math.radians(deg)), math.sin(math.radians(deg))
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


def random_rotation(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


# ---------------------------------------------------------------------------------------
# A0 / O2: geometry
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", gold("spec_examples.json")["project_depth"])
def test_project_depth_spec_examples(case):
    """S:120-122 project_depth examples (pinhole identity, translation, 90 deg yaw)."""
    M = np.eye(4, dtype=np.float32)
    M[:3, :3] = np.round(rot_y(case["yaw_y_deg"]), 12)
    M[:3, 3] = case["t"]
    d = np.full((1, 1), case["depth"], np.float32)
    fr = frame(d, np.zeros((0, 1, 1)), M, fx=case["fx"], fy=case["fy"], cx=case["cx"], cy=case["cy"])
    ok, p = O.pixel_world(cfg(), fr, *case["pixel"])
    assert ok
    np.testing.assert_allclose(p, case["point"], atol=1e-6)


def test_project_depth_hand_multiplied():
    """S:117 formula on a non-trivial pixel; hand-computed: u=3,v=1,fx=2,fy=4,cx=1,cy=0.5,d=2
    -> p_c = (2, 0.25, 2); R = rot_y(90) -> R p_c = (2, 0.25, -2); + t (1,2,3) = (3, 2.25, 1)."""
    M = np.eye(4, dtype=np.float32)
    M[:3, :3] = np.round(rot_y(90), 12)
    M[:3, 3] = [1, 2, 3]
    d = np.full((2, 4), 2.0, np.float32)
    fr = frame(d, np.zeros((0, 2, 4)), M, fx=2.0, fy=4.0, cx=1.0, cy=0.5)
    ok, p = O.pixel_world(cfg(), fr, 3, 1)
    assert ok
    np.testing.assert_allclose(p, [3.0, 2.25, 1.0], atol=1e-6)


def test_depth_window_exclusive_and_nonfinite():
    """R4: valid iff finite and d_min < d < d_max (exclusive)."""
    d = np.array([[0.1, 0.1000001, 10.0, 9.999999, np.nan, np.inf, 0.0, 5.0]], np.float32)
    fr = frame(d, np.zeros((0, 1, 8)))
    got = [O.pixel_world(cfg(), fr, u, 0)[0] for u in range(8)]
    assert got == [False, True, False, True, False, False, False, True]


@pytest.mark.parametrize("case", gold("spec_examples.json")["voxelize"])
def test_voxelize_spec_examples(case):
    """one voxel for two close points; floor, not truncation, for negatives."""
    keys = set()
    for p in case["points"]:
        ok, k = O.point_key(np.array(p, np.float32), case["r"])
        assert ok
        keys.add(tuple(int(x) for x in k))
    assert keys == {tuple(k) for k in case["keys"]}


def test_voxelize_bruteforce_1000_points():
    """1000 random points in the unit cube, r = 0.1 -> key set equals brute-force
    floor(p / r) with numpy's IEEE float32 division."""
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1, 1, (1000, 3)).astype(np.float32)
    r = np.float32(0.1)
    want = {tuple(int(x) for x in np.floor(p / r)) for p in pts}
    got = set()
    for p in pts:
        ok, k = O.point_key(p, 0.1)
        assert ok
        got.add(tuple(int(x) for x in k))
    assert got == want


def test_key_range_and_packing():
    """R6: components in [-2^20, 2^20), packed 3 x 21 bits, order preserving."""
    r = 1.0
    for val, ok_want in [(2.0 ** 20 - 1, True), (2.0 ** 20, False), (-(2.0 ** 20), True),
                         (-(2.0 ** 20) - 1, False)]:
        ok, _ = O.point_key(np.array([val, 0, 0], np.float32), r)
        assert ok == ok_want, val
    B = 1 << 20
    assert O.pack_key(0, 0, 0) == (B << 42) | (B << 21) | B
    assert O.pack_key(-B, -B, -B) == 0
    assert O.pack_key(B - 1, B - 1, B - 1) == (1 << 63) - 1
    rng = np.random.default_rng(3)
    ks = [tuple(int(x) for x in rng.integers(-B, B, 3)) for _ in range(300)]
    by_tuple = sorted(ks)
    by_pack = sorted(ks, key=lambda k: O.pack_key(*k))
    assert by_tuple == by_pack


def test_pinned_keys_match_exact_rational_rederivation():
    """R5: the oracle's fp32 keys equal an exact-rational re-derivation of the pinned
    operation order (each IEEE op rounded once), under random rigid poses."""
    rng = np.random.default_rng(11)
    H, W = 6, 8
    for trial in range(4):
        M = np.eye(4)
        M[:3, :3] = random_rotation(rng)
        M[:3, 3] = rng.uniform(-3, 3, 3)
        M = M.astype(np.float32)
        depth = rng.uniform(0.3, 6.0, (H, W)).astype(np.float32)
        fx, fy, cx, cy = np.float32(5.3), np.float32(4.7), np.float32(3.5), np.float32(2.5)
        r = np.float32([0.01, 0.02, 0.05, 0.1][trial])
        fr = frame(depth, np.zeros((0, H, W)), M, fx=float(fx), fy=float(fy), cx=float(cx), cy=float(cy))
        c = cfg(voxel_size=float(r))
        Mf = M.reshape(16)
        for v in range(H):
            for u in range(W):
                ok, p = O.pixel_world(c, fr, u, v)
                assert ok
                ok2, k = O.point_key(p, float(r))
                assert ok2
                want = exact_key(u, v, depth[v, u], fx, fy, cx, cy, Mf, r)
                assert tuple(int(x) for x in k) == want, (trial, u, v)


def test_pinned_keys_vs_fp64_only_near_boundaries():
    """C.4: where the pinned fp32 key and an fp64 recomputation disagree, the fp64 value lies
    within 1e-5 voxel of an integer."""
    rng = np.random.default_rng(5)
    H, W = 40, 50
    M = np.eye(4)
    M[:3, :3] = random_rotation(rng)
    M[:3, 3] = [1.3, -0.7, 2.1]
    M = M.astype(np.float32)
    depth = rng.uniform(0.5, 8.0, (H, W)).astype(np.float32)
    fr = frame(depth, np.zeros((0, H, W)), M, fx=37.0, fy=37.0, cx=25.0, cy=20.0)
    r = 0.02
    c = cfg(voxel_size=r)
    Md = M.astype(np.float64)
    dis = 0
    for v in range(H):
        for u in range(W):
            ok, p = O.pixel_world(c, fr, u, v)
            _, k = O.point_key(p, r)
            d = float(depth[v, u])
            pc = np.array([(u - 25.0) / 37.0 * d, (v - 20.0) / 37.0 * d, d])
            pw = Md[:3, :3] @ pc + Md[:3, 3]
            q = pw / np.float64(np.float32(r))
            k64 = np.floor(q)
            for i in range(3):
                if k64[i] != k[i]:
                    dis += 1
                    assert abs(q[i] - round(q[i])) < 1e-5
    assert dis < 0.01 * H * W * 3


def test_pose_rigidity():
    """A0: rotation orthonormal within 1e-5, det +1, last row 0 0 0 1."""
    I = np.eye(4, dtype=np.float32)
    assert O.pose_rigid(I)
    rng = np.random.default_rng(1)
    M = np.eye(4)
    M[:3, :3] = random_rotation(rng)
    M[:3, 3] = [1, 2, 3]
    assert O.pose_rigid(M)
    S = I.copy(); S[0, 0] = 1.001
    assert not O.pose_rigid(S)
    Rf = I.copy(); Rf[0, 0] = -1.0
    assert not O.pose_rigid(Rf)           # reflection: det = -1
    L = I.copy(); L[3, 0] = 0.1
    assert not O.pose_rigid(L)
    N = M.copy(); N[0, 1] += 3e-6
    assert O.pose_rigid(N)                # within 1e-5


def test_invalid_frame_leaves_state_untouched():
    """A0 / C.2 O0: validation failure returns INVALID before any mutation."""
    m = O.OracleMap(voxel_size=0.05, feat_dim=4)
    m.integrate(t0_frame(0))
    keys0, ids0 = m.memberships()
    bad = t0_frame(1)
    bad["pose"] = bad["pose"].copy()
    bad["pose"][0, 0] = 2.0
    assert m.try_integrate(bad) == 2
    keys1, ids1 = m.memberships()
    assert np.array_equal(keys0, keys1) and np.array_equal(ids0, ids1)
    assert m.next_id() == 2


# ---------------------------------------------------------------------------------------
# A1: mask filter
# ---------------------------------------------------------------------------------------

def test_mask_filter_examples():
    """keep; sliver discarded; thresholds inclusive; drop-reason order (C.2 O1)."""
    H, W = 40, 320
    depth = np.full((H, W), 2.0, np.float32)
    masks = np.zeros((6, H, W), np.uint8)
    masks[0, 0:20, 0:21] = 1            # area 420, aspect 21/20 -> kept
    masks[1, 0:2, 0:300] = 1            # 2x300 sliver, aspect 150 -> aspect
    masks[2, 0:20, 0:20] = 1            # area 400 exactly, conf 0.5 exactly -> kept (inclusive)
    masks[3, 0:4, 0:40] = 1             # aspect exactly 10 (40/4), area 160 -> area
    masks[4, 0:10, 0:100] = 1           # aspect exactly 10, area 1000 -> kept
    # mask 5 empty -> area
    conf = np.array([0.9, 0.9, 0.5, 0.9, 0.9, 0.9], np.float32)
    conf[0] = 0.9
    fr = frame(depth, masks, fx=100.0, fy=100.0, cx=160.0, cy=20.0, mask_conf=conf)
    m = O.OracleMap(voxel_size=0.05, feat_dim=4)
    m.integrate(fr)
    st = m.last_frame()["status"]
    assert list(st) == [O.KEPT, O.DROP_ASPECT, O.KEPT, O.DROP_AREA, O.KEPT, O.DROP_AREA]
    # low confidence is reported before aspect
    conf2 = conf.copy(); conf2[1] = 0.49999
    fr2 = frame(depth, masks, fx=100.0, fy=100.0, cx=160.0, cy=20.0, mask_conf=conf2, frame_id=1)
    m2 = O.OracleMap(voxel_size=0.05, feat_dim=4)
    m2.integrate(fr2)
    assert m2.last_frame()["status"][1] == O.DROP_CONF


def test_detections_nodepth_and_disjoint_boxes():
    """a mask whose depth is all invalid -> 0 detections ("no valid depth");
    two boxes -> two detections with disjoint voxel sets."""
    H, W = 30, 60
    depth = np.full((H, W), 2.0, np.float32)
    depth[:, :30] = 0.0
    masks = np.zeros((2, H, W), np.uint8)
    masks[0, :, :30] = 1
    masks[1, :, 30:] = 1
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, mask_min_area=10)
    rep = m.integrate(frame(depth, masks, fx=30.0, fy=30.0, cx=30.0, cy=15.0))
    assert rep["drop_nodepth"] == 1 and rep["kept"] == 1 and rep["created"] == 1
    g = Generator("T")
    fr = frame_to_numpy(g.frame(0))
    fr["mask_conf"] = None
    m2 = O.OracleMap(**disc_config_kwargs(g.cfg))
    m2.integrate(fr)
    lf = m2.last_frame()
    sets = {}
    for s, k in zip(lf["pair_s"], lf["pair_key"]):
        sets.setdefault(int(s), set()).add(int(k))
    box_sets = [sets[s] for s in sets if lf["area"][s] < 500]
    assert len(box_sets) >= 2
    for i in range(len(box_sets)):
        for j in range(i + 1, len(box_sets)):
            assert not (box_sets[i] & box_sets[j])


# ---------------------------------------------------------------------------------------
# T0 hand-worked fixture (C.4)
# ---------------------------------------------------------------------------------------

def _key_tuple(packed):
    B = 1 << 20
    p = int(packed)
    return ((p >> 42) - B, ((p >> 21) & ((1 << 21) - 1)) - B, (p & ((1 << 21) - 1)) - B)


def test_t0_frame0_keys_by_hand():
    """T0 frame 0: ix = u-33 / u-32 split, 48 distinct iy, iz = 32, |V_A| = |V_B| = 1536."""
    G = gold("t0.json")["frame0"]
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, selfcheck=True)
    m.integrate(t0_frame(0))
    lf = m.last_frame()
    assert list(lf["vs"]) == G["vs"]
    for s, rng_ in [(0, G["ix_range_A"]), (1, G["ix_range_B"])]:
        ks = [_key_tuple(k) for k, ss in zip(lf["pair_key"], lf["pair_s"]) if ss == s]
        ix = sorted({k[0] for k in ks})
        assert ix == list(range(rng_[0], rng_[1] + 1))
        assert len({k[1] for k in ks}) == G["iy_count"]
        assert {k[2] for k in ks} == {G["iz"]}
    # exact rational re-derivation of every T0 key
    fr = t0_frame(0)
    Mf = fr["pose"].reshape(16)
    want = set()
    for v in range(48):
        for u in range(64):
            want.add(exact_key(u, v, np.float32(1.62), np.float32(32), np.float32(32), np.float32(32),
                               np.float32(24), Mf, np.float32(0.05)))
    got = {_key_tuple(k) for k in lf["pair_key"]}
    assert got == want


@pytest.mark.parametrize("tau", [0.3, 0.48])
def test_t0_association_hand_values(tau):
    """T0 frames 1-2 (C.4): counts 720 / 768; bridged merge into the lower id at tau 0.3;
    single edge at tau 0.48; R25 idempotent re-integration."""
    G = gold("t0.json")
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, tau_geo=tau, selfcheck=True)
    m.integrate(t0_frame(0))
    rep = m.integrate(t0_frame(1))
    lf = m.last_frame()
    assert list(lf["vs"]) == G["frame1"]["vs"]
    trip = {(int(s), int(j)): int(c) for s, j, c in zip(lf["trip_s"], lf["trip_j"], lf["trip_c"])}
    assert trip == {(0, 0): G["frame1"]["c_vs_id0"], (0, 1): G["frame1"]["c_vs_id1"]}
    want = G[f"tau_{tau}"]
    inst = m.instances()
    assert list(inst["id"]) == want["after_frame1"]["ids"]
    assert list(inst["vcount"]) == want["after_frame1"]["vcount"]
    if tau == 0.48:
        keys, ids = m.memberships()
        k0 = set(keys[ids == 0].tolist())
        k1 = set(keys[ids == 1].tolist())
        assert len(k0 & k1) == want["after_frame1"]["shared_keys"]
    else:
        assert rep["merged_away"] == 1 and rep["relabeled"] == 1536
    keys_before, ids_before = m.memberships()
    m.integrate(t0_frame(2))
    keys_after, ids_after = m.memberships()
    assert np.array_equal(keys_before, keys_after) and np.array_equal(ids_before, ids_after)
    inst = m.instances()
    assert list(inst["vcount"]) == want["after_frame2"]["vcount"]
    assert list(inst["obs"]) == want["after_frame2"]["obs"]


def test_overlap_spec_example():
    """a = {(0,0,0),(1,0,0)}, b = {(1,0,0),(2,0,0)} -> intersection 1,
    overlap_min 1/2: with tau 0.5 the pair qualifies (inclusive), with tau 0.6 it does not."""
    G = gold("spec_examples.json")["overlap"]
    depth = np.array([[1.5, 1.5]], np.float32)  # fx = 1, cx = 0: x = u * 1.5 -> ix 0 and 1 (r = 1)
    for tau, merged in [(0.5, True), (0.6, False)]:
        m = O.OracleMap(voxel_size=1.0, feat_dim=4, tau_geo=tau, mask_min_area=1, selfcheck=True)
        m.integrate(frame(depth, np.ones((1, 1, 2))))
        T = np.eye(4, dtype=np.float32)
        T[0, 3] = 1.0
        m.integrate(frame(depth, np.ones((1, 1, 2)), T, frame_id=1))
        lf = m.last_frame()
        keys = [_key_tuple(k) for k in lf["pair_key"]]
        assert sorted(k[0] for k in keys) == [b[0] for b in G["b"]]
        assert list(lf["trip_c"]) == [G["intersection"]]
        assert list(lf["trip_edge"]) == [1 if merged else 0]
        assert m.instances()["id"].shape[0] == (1 if merged else 2)


def test_association_spec_examples():
    """empty map + 3 disjoint detections -> 3 created; identical re-observation ->
    matched, obs + 1, voxel set unchanged."""
    H, W = 20, 60
    depth = np.full((H, W), 2.0, np.float32)
    masks = np.zeros((3, H, W), np.uint8)
    masks[0, :, 0:20] = 1
    masks[1, :, 20:40] = 1
    masks[2, :, 40:60] = 1
    fr = frame(depth, masks, fx=30.0, fy=30.0, cx=30.0, cy=10.0)
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, mask_min_area=10, selfcheck=True)
    rep = m.integrate(fr)
    assert rep["created"] == 3 and rep["edges"] == 0
    k0, i0 = m.memberships()
    fr1 = dict(fr, frame_id=1, masks=masks[:1])
    rep = m.integrate(fr1)
    assert rep["created"] == 0 and rep["edges"] == 1 and rep["merged_away"] == 0
    k1, i1 = m.memberships()
    assert np.array_equal(k0, k1) and np.array_equal(i0, i1)
    assert list(m.instances()["obs"]) == [2, 1, 1]


def test_chain_merge_union_find_vs_bfs():
    """S:340 chain A-B-C via bridging detections -> single survivor = min id; the oracle's
    self-check compares its BFS components with an independent union-find."""
    H, W = 10, 90
    depth = np.full((H, W), 2.0, np.float32)
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, mask_min_area=10, tau_geo=0.2, selfcheck=True)
    masks = np.zeros((3, H, W), np.uint8)
    masks[0, :, 0:30] = 1
    masks[1, :, 30:60] = 1
    masks[2, :, 60:90] = 1
    fx = dict(fx=30.0, fy=30.0, cx=45.0, cy=5.0)
    m.integrate(frame(depth, masks, **fx))
    bridge = np.zeros((2, H, W), np.uint8)
    bridge[0, :, 15:45] = 1
    bridge[1, :, 45:75] = 1
    rep = m.integrate(frame(depth, bridge, frame_id=1, **fx))
    assert rep["merged_away"] == 2
    inst = m.instances()
    assert list(inst["id"]) == [0]


# ---------------------------------------------------------------------------------------
# Eq.1 distinctiveness, pooling, quality
# ---------------------------------------------------------------------------------------

def test_distinctiveness_spec():
    """uniform -> 0; 2x2 hand case; mean(D) = 1 +- 1e-3; translation
    and scale invariance."""
    G = gold("spec_examples.json")["distinctiveness_2x2"]
    assert np.all(O.distinctiveness(np.ones((9, 5))) == 0.0)
    D = O.distinctiveness(np.array(G["features"], np.float32))
    np.testing.assert_allclose(D, G["D"], atol=G["tol"])
    rng = np.random.default_rng(2)
    f = rng.standard_normal((64, 32)).astype(np.float32)
    D = O.distinctiveness(f)
    assert abs(D.mean() - 1.0) < 1e-3
    np.testing.assert_allclose(O.distinctiveness(f + np.float32(3.0)), D, rtol=1e-5)
    np.testing.assert_allclose(O.distinctiveness(f * np.float32(4.0)), D, rtol=1e-5)


def test_pooling_spec():
    """one full patch -> its feature; equal D -> midpoint; D = (2, 0.5) ->
    (2 f1 + 0.5 f2)/2.5; unit norm; fallback to unweighted mean; zero -> nofeat."""
    f = np.array([[3.0, 4.0, 0.0], [0.0, 1.0, 1.0], [5.0, 5.0, 5.0]], np.float32)
    npix = np.array([196, 196, 196])
    rc, e, _ = O.pool([196, 0, 0], npix, [1.0, 1.0, 1.0], f)
    assert rc == 0
    np.testing.assert_allclose(e, f[0] / np.linalg.norm(f[0]), atol=1e-15)
    rc, e, _ = O.pool([196, 196, 0], npix, [1.0, 1.0, 1.0], f)
    mid = (f[0].astype(np.float64) + f[1]) / 2
    np.testing.assert_allclose(e, mid / np.linalg.norm(mid), atol=1e-15)
    rc, e, dbar = O.pool([196, 196, 0], npix, [2.0, 0.5, 1.0], f)
    y = (2 * f[0].astype(np.float64) + 0.5 * f[1]) / 2.5
    np.testing.assert_allclose(e, y / np.linalg.norm(y), atol=1e-15)
    assert abs(dbar - 1.25) < 1e-15                       # R19: (2 + 0.5)/2
    assert abs(np.linalg.norm(e) - 1.0) < 1e-12
    # coverage below 0.25 everywhere: fallback to unweighted over patches with cnt > 0
    rc, e, _ = O.pool([48, 10, 0], npix, [9.0, 0.1, 1.0], f)
    y = f[0].astype(np.float64) + f[1]
    np.testing.assert_allclose(e, y / np.linalg.norm(y), atol=1e-15)
    # threshold is inclusive and exact: 49 = 0.25 * 196
    rc, e, _ = O.pool([49, 48, 0], npix, [1.0, 1.0, 1.0], f)
    np.testing.assert_allclose(e, f[0] / np.linalg.norm(f[0]), atol=1e-15)
    # weight-scale invariance
    rc, e1, _ = O.pool([100, 150, 60], npix, [1.3, 0.7, 2.2], f)
    rc, e2, _ = O.pool([100, 150, 60], npix, [2.6, 1.4, 4.4], f)
    np.testing.assert_allclose(e1, e2, atol=1e-15)
    rc, e, _ = O.pool([196, 0, 0], npix, [1.0, 1.0, 1.0], np.zeros((3, 3), np.float32))
    assert rc == 1


def test_quality_factors_spec():
    """S:236-238 S_size; S:244-246 S_angle; S:252-254 S_sem; S:260-262 S_dist; S:269 Q."""
    G = gold("spec_examples.json")
    H, W = 100, 100
    for frac, want in G["s_size"]["cases"]:
        assert abs(O.s_size(int(frac * H * W), H, W, 3.3) - want) < 1e-12
    n = np.array([[0, 0, 1.0]])
    assert O.s_angle(n, -n) == 1.0
    assert O.s_angle(n, np.array([[1.0, 0, 0]])) == 0.0
    assert O.s_angle(np.array([[0, 0, 1.0], [0, 0, 1.0]]), np.array([[0, 0, -1.0], [0, 0, 1.0]])) == 0.5
    e = np.array([0.6, 0.8, 0.0])
    assert abs(O.s_sem(e, np.array([3, 4, 0], np.float32)) - 1.0) < 1e-12
    assert O.s_sem(e, np.array([0, 0, 2], np.float32)) == 0.0
    g = np.array([-0.3, math.sqrt(1 - 0.09), 0.0], np.float32)
    e2 = np.array([1.0, 0.0, 0.0])
    assert O.s_sem(e2, g) == 0.0                      # cos = -0.3 -> ReLU clamp
    assert O.s_sem(e, None) == 1.0
    for dbar, want in G["s_dist"]["cases"]:
        assert O.s_dist(dbar) == want
    a, b, c, d = G["quality"]["factors"]
    assert abs(O.quality(a, b, c, d) - G["quality"]["q"]) < 1e-12
    assert O.quality(1, 1, 1, 1) == 1.0 and O.quality(0, 1, 1, 1) == 0.0


def test_dot_pin_exact_on_snapped_values():
    """R15: for bf16 values snapped to multiples of 2^-12 times integer counts, dot_pin equals
    the exact rational dot product (rounded once), independent of the lane order."""
    rng = np.random.default_rng(9)
    for n in [1, 31, 32, 33, 384]:
        a = np.round(rng.uniform(-8, 8, n) * 4096) / 4096 * rng.integers(1, 200, n)
        b = np.round(rng.uniform(-8, 8, n) * 4096) / 4096
        exact = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))
        assert O.dot_pin(a, b) == float(exact)
    a = rng.standard_normal(384)
    assert abs(O.dot_pin(a, a) - math.fsum(a * a)) < 1e-12 * math.fsum(a * a)


def test_tracking_sum_exact():
    """R15 / A§6: u_s = sum_p cnt_sp g_p is exact in fp64: equals a Fraction re-derivation
    from the raw bf16 bits and the mask pixel counts."""
    g = Generator("T")
    fr = frame_to_numpy(g.frame(0))
    fr["mask_conf"] = None
    m = O.OracleMap(**disc_config_kwargs(g.cfg))
    m.integrate(fr)
    lf = m.last_frame()
    H, W, Hp, Wp, Dt = 48, 64, 16, 16, 32
    gvals = (fr["track_feats"].astype(np.uint32) << 16).view(np.float32).reshape(Hp * Wp, Dt)
    v, u = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    pidx = (v * Hp // H) * Wp + (u * Wp // W)
    for s in range(fr["masks"].shape[0]):
        if lf["status"][s] != O.KEPT:
            continue
        cnt = np.bincount(pidx[fr["masks"][s] > 0], minlength=Hp * Wp)
        for d in range(Dt):
            exact = sum(Fraction(int(cnt[p])) * Fraction(float(gvals[p, d])) for p in np.nonzero(cnt)[0])
            assert lf["u"][s, d] == float(exact)


# ---------------------------------------------------------------------------------------
# fusion, map invariants, brute force on generated scenes
# ---------------------------------------------------------------------------------------

def _tokens_for(depth_shape, Df, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((4, 4, Df)).astype(np.float32)


def test_fusion_argmax_regardless_of_order():
    """the instance keeps the argmax-Q observation, independent of
    arrival order; ties keep the incumbent (strict >)."""
    H, W = 40, 40
    depth = np.full((H, W), 2.0, np.float32)
    feats = [_tokens_for((H, W), 8, s) for s in range(3)]
    areas = [(0, 40), (0, 30), (0, 20)]  # different mask areas -> different S_size -> Q
    frames = []
    for i, (a, b) in enumerate(areas):
        mk = np.zeros((1, H, W), np.uint8)
        mk[0, :, a:b] = 1
        frames.append(dict(frame_id=i, depth=depth, masks=mk, mask_conf=None, pose=np.eye(4, dtype=np.float32),
                           fx=20.0, fy=20.0, cx=20.0, cy=20.0, patch_h=4, patch_w=4, patch_feats=feats[i],
                           global_embed=None, track_feats=None))
    finals = []
    for order in [(0, 1, 2), (2, 1, 0), (1, 2, 0)]:
        m = O.OracleMap(voxel_size=0.05, feat_dim=8, mask_min_area=10, tau_geo=0.3, selfcheck=True)
        qs = []
        for k, i in enumerate(order):
            fr = dict(frames[i], frame_id=k)
            m.integrate(fr)
            qs.append(m.last_frame()["factors"][0, 4])
        inst = m.instances()
        assert inst["id"].shape[0] == 1
        assert inst["q"][0] == max(qs)
        finals.append(inst["e"][0])
    for e in finals[1:]:
        np.testing.assert_array_equal(e, finals[0])


def test_generated_scene_bruteforce_and_invariants():
    """C.4 on a generated T stream: overlap triples equal a brute-force Python set
    intersection against the exported frame-start memberships; conservation
    (live memberships = sum |V_j|); determinism (two runs bit-identical)."""
    g = Generator("T")
    frames = [frame_to_numpy(g.frame(f)) for f in range(3)]
    for fr in frames:
        fr["mask_conf"] = np.maximum(fr["mask_conf"], 0.5)   # keep every mask
    runs = []
    for _ in range(2):
        m = O.OracleMap(selfcheck=True, **disc_config_kwargs(g.cfg))
        for fr in frames:
            keys, ids = m.memberships()
            inst_sets = {}
            for k, i in zip(keys.tolist(), ids.tolist()):
                inst_sets.setdefault(i, set()).add(k)
            rep = m.integrate(fr)
            lf = m.last_frame()
            dets = {}
            for s, k in zip(lf["pair_s"].tolist(), lf["pair_key"].tolist()):
                dets.setdefault(s, set()).add(k)
            brute = {}
            for s, V in dets.items():
                for j, Vj in inst_sets.items():
                    c = len(V & Vj)
                    if c:
                        brute[(s, j)] = c
            trip = {(int(s), int(j)): int(c) for s, j, c in zip(lf["trip_s"], lf["trip_j"], lf["trip_c"])}
            assert trip == brute
            inst = m.instances()
            assert rep["live_memberships"] == int(inst["vcount"].sum()) == m.memberships()[0].shape[0]
        runs.append((m.memberships(), m.instances()))
    (k0, i0), a = runs[0]
    (k1, i1), b = runs[1]
    assert np.array_equal(k0, k1) and np.array_equal(i0, i1)
    for key in a:
        assert np.array_equal(a[key], b[key])


def test_query_full_sort_ties_by_id():
    """descending cosine, ties by ascending id."""
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, mask_min_area=10)
    H, W = 20, 60
    depth = np.full((H, W), 2.0, np.float32)
    masks = np.zeros((3, H, W), np.uint8)
    masks[0, :, 0:20] = 1
    masks[1, :, 20:40] = 1
    masks[2, :, 40:60] = 1
    feats = np.zeros((1, 3, 4), np.float32)
    feats[0, 0] = [1, 0, 0, 0]
    feats[0, 1] = [0, 1, 0, 0]
    feats[0, 2] = [1, 0, 0, 0]
    fr = frame(depth, masks, fx=30.0, fy=30.0, cx=30.0, cy=10.0, patch_h=1, patch_w=3, patch_feats=feats)
    m.integrate(fr)
    ids, sc = m.query(np.array([2.0, 0, 0, 0], np.float32), 3)
    assert list(ids) == [0, 2, 1]
    assert sc[0] == sc[1] == 1.0 and sc[2] == 0.0
