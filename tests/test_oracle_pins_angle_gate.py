"""Pins of two oracle parts the round-1 review found unpinned ("What's weak" 1):

  * the S_angle ASSEMBLY (Eq.3, with reading R21): pixel normals from the 4-neighbour
    central differences of the fp32 world points, oriented towards the camera, summed per voxel,
    the ray from the camera centre to the voxel centre (k + 0.5) r, and the mean over the voxels
    that HAVE a normal (R21; Eq.3 writes 1/|V|, R21 reads it over the voxels with a normal);
  * the O10 visual gate ("visual similarity", reading R15): cos_pin(t_s, T_j) >= tau_vis,
    inclusive, with a zero-norm t or T giving cos = -2 (never passes, not even at tau_vis = -1).

Every expected value below is a closed form derived from the geometry / the token values by hand
(comments give the derivation), evaluated here with numpy / fractions -- never with oracle/ code.
Keys of the fronto-parallel T0 wall come from the golden hand formula (tests/golden/t0.json);
keys of the tilted wall from the exact-rational re-derivation of R5 in test_oracle_pins.exact_key.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from synth import t0_frame
from tests.test_oracle_pins import exact_key, gold

H0, W0, F0, CX0, CY0, D0, R0 = 48, 64, 32.0, 32.0, 24.0, 1.62, 0.05


def t0_keys(u, v, tx_vox=0):
    """Hand formula of tests/golden/t0.json: x/r = 1.0125 (u - 32) (+ tx/r), floor by hand."""
    ix = (u - 32 if u >= 32 else u - 33) + tx_vox
    iy = v - 24 if v >= 24 else v - 25
    return ix, iy, 32


def closed_form_angle(keys, cam, r=np.float32(R0)):
    """Eq.3 over voxels whose normal is (0, 0, -1) (a wall z = const facing a camera at smaller z):
    max(0, -r_hat . n_hat) = r_hat_z with r = (k + 0.5) r - cam (R21)."""
    rr = float(r)
    vals = []
    for k in sorted(keys):
        ray = [(k[a] + 0.5) * rr - cam[a] for a in range(3)]
        vals.append(max(0.0, ray[2] / math.sqrt(ray[0] ** 2 + ray[1] ** 2 + ray[2] ** 2)))
    return sum(vals) / len(vals)


def semantic_t0(index, depth=None, masks=None):
    fr = t0_frame(index, with_tokens=True, Df=16)
    if depth is not None:
        fr["depth"] = depth
    if masks is not None:
        fr["masks"] = masks
    return fr


def angle_of(fr, s):
    m = O.OracleMap(voxel_size=R0, feat_dim=16, selfcheck=True)
    m.integrate(fr)
    lf = m.last_frame()
    assert lf["status"][s] == 0
    return lf["factors"][s][1]


def interior(u, v, valid):
    """R21: a pixel has a normal iff it and its 4 in-image neighbours have valid depth."""
    if u < 1 or u > W0 - 2 or v < 1 or v > H0 - 2:
        return False
    return valid[v, u] and valid[v, u - 1] and valid[v, u + 1] and valid[v - 1, u] and valid[v + 1, u]


@pytest.mark.parametrize("s", [0, 1])
def test_s_angle_fronto_parallel_wall_pose_identity(s):
    """T0 frame 0, pose I: every pixel its own voxel (golden hand keys); the wall normal (0,0,-1)
    faces the camera at the origin; border pixels (u in {0, 63}, v in {0, 47}) have no normal, so
    their voxels are excluded from the mean (R21)."""
    valid = np.ones((H0, W0), bool)
    keys = {t0_keys(u, v) for v in range(H0) for u in range(W0)
            if ((u < 32) if s == 0 else (u >= 32)) and interior(u, v, valid)}
    want = closed_form_angle(keys, (0.0, 0.0, 0.0))
    got = angle_of(semantic_t0(0), s)
    assert abs(got - want) < 1e-12, (got, want)
    # mean over ALL |V_s| voxels (Eq.3's literal 1/|V|, border voxels counted as 0) is different:
    all_keys = {t0_keys(u, v) for v in range(H0) for u in range(W0) if ((u < 32) if s == 0 else (u >= 32))}
    assert abs(want * len(keys) / len(all_keys) - got) > 1e-3


def test_s_angle_translated_camera_ray_to_voxel_centre():
    """T0 frame 1 (t = (0.05, 0, 0)): keys ix = u - 31 / u - 32 (golden), and the ray starts at the
    camera centre (0.05, 0, 0), not at the world origin, and ends at (k + 0.5) r, not at k r."""
    valid = np.ones((H0, W0), bool)
    u = np.arange(W0)[None, :].repeat(H0, 0)
    mask = ((u >= 20) & (u < 48))[None].astype(np.uint8)   # asymmetric about the camera
    keys = {t0_keys(u, v, tx_vox=1) for v in range(H0) for u in range(20, 48) if interior(u, v, valid)}
    want = closed_form_angle(keys, (float(np.float32(0.05)), 0.0, 0.0))
    got = angle_of(semantic_t0(1, masks=mask), 0)
    assert abs(got - want) < 1e-12, (got, want)
    wrong_origin = closed_form_angle(keys, (0.0, 0.0, 0.0))
    assert abs(wrong_origin - got) > 1e-6
    rr = float(np.float32(R0))
    corner = sum(max(0.0, k[2] * rr / math.sqrt((k[0] * rr - 0.05) ** 2 + (k[1] * rr) ** 2 + (k[2] * rr) ** 2))
                 for k in keys) / len(keys)
    assert abs(corner - got) > 1e-6


def test_s_angle_holes_exclude_their_4_neighbours_only():
    """Depth holes (0 = invalid, R4): a hole pixel has no key; each of its 4 neighbours loses its
    normal (R21 needs 4 valid neighbours), its diagonal neighbours do not.  Asymmetric hole pattern,
    so an 8-neighbour rule or one-sided differences give a different voxel set and mean."""
    depth = np.full((H0, W0), np.float32(D0), np.float32)
    holes = [(10, 10), (11, 20)] + [(u, 30) for u in range(40, 47)] + [(5, 40), (6, 41)]
    for u, v in holes:
        depth[v, u] = 0.0
    valid = depth > 0
    for s in (0, 1):
        keys = {t0_keys(u, v) for v in range(H0) for u in range(W0)
                if ((u < 32) if s == 0 else (u >= 32)) and interior(u, v, valid)}
        want = closed_form_angle(keys, (0.0, 0.0, 0.0))
        got = angle_of(semantic_t0(0, depth=depth), s)
        assert abs(got - want) < 1e-12, (s, got, want)

        def eight(u, v):
            return interior(u, v, valid) and all(valid[v + dv, u + du] for du in (-1, 1) for dv in (-1, 1))
        keys8 = {t0_keys(u, v) for v in range(H0) for u in range(W0)
                 if ((u < 32) if s == 0 else (u >= 32)) and eight(u, v)}
        assert keys8 != keys and abs(closed_form_angle(keys8, (0, 0, 0)) - got) > 1e-9


def test_s_angle_tilted_wall():
    """Camera rotated by theta = 20 deg about its y axis in front of the world wall z = 1.62
    (normal (0,0,-1) towards the camera at the origin).  Depth per pixel is the analytic ray /
    plane intersection (fp32).  Every world point lies on the wall up to fp32 rounding, so every
    pixel normal is (0,0,-1) up to ~1e-6 and S_angle = mean over the interior pixels' voxels of
    r_hat_z.  Voxels: exact-rational re-derivation of R5 per pixel (test_oracle_pins.exact_key)."""
    th = math.radians(20.0)
    Rm = np.array([[math.cos(th), 0, math.sin(th)], [0, 1, 0], [-math.sin(th), 0, math.cos(th)]])
    pose = np.eye(4, dtype=np.float32)
    pose[:3, :3] = Rm.astype(np.float32)
    Rf = pose[:3, :3].astype(np.float64)
    depth = np.zeros((H0, W0), np.float32)
    for v in range(H0):
        for u in range(W0):
            dc = np.array([(u - CX0) / F0, (v - CY0) / F0, 1.0])
            depth[v, u] = np.float32(D0 / (Rf[2] @ dc))   # z_w = t (R dc)_z = D
    assert depth.min() > 0.5 and depth.max() < 9.0
    fr = semantic_t0(0, depth=depth, masks=np.ones((1, H0, W0), np.uint8))
    fr["pose"] = pose
    Mf = pose.reshape(16)
    valid = np.ones((H0, W0), bool)
    keys = set()
    for v in range(H0):
        for u in range(W0):
            if interior(u, v, valid):
                keys.add(exact_key(u, v, depth[v, u], np.float32(F0), np.float32(F0), np.float32(CX0),
                                   np.float32(CY0), Mf, np.float32(R0)))
    assert {k[2] for k in keys} == {32}
    want = closed_form_angle(keys, (0.0, 0.0, 0.0))
    got = angle_of(fr, 0)
    assert abs(got - want) < 1e-5, (got, want)
    # a normal oriented away from the camera would give 0; the untilted value differs
    assert got > 0.5 and abs(got - angle_of(semantic_t0(0, masks=np.ones((1, H0, W0), np.uint8)), 0)) > 1e-2


# ---------------------------------------------------------------------------------------------
# O10 visual gate (R15)
# ---------------------------------------------------------------------------------------------
BF16 = {0.0: 0x0000, 0.5: 0x3F00, 1.0: 0x3F80}


def tokens(fn, Dt=8):
    """16x16 patch grid of Dt-dim bf16 tracking tokens; fn(col) -> list of Dt values (patch column
    col covers image columns 4 col .. 4 col + 3, so col < 8 <=> u < 32)."""
    g = np.zeros((16, 16, Dt), np.uint16)
    for c in range(16):
        vals = fn(c)
        for k in range(Dt):
            g[:, c, k] = BF16[vals[k]]
    return g


E0 = [1.0] + [0.0] * 7
E1 = [0.0, 1.0] + [0.0] * 6
HALF4 = [0.5, 0.5, 0.5, 0.5, 0, 0, 0, 0]
ZERO = [0.0] * 8


def gate_run(tok0, tok1, tau_vis):
    m = O.OracleMap(voxel_size=R0, feat_dim=4, track_dim=8, tau_geo=0.3, tau_vis=tau_vis, selfcheck=True)
    f0 = t0_frame(0)
    f0["track_feats"] = tok0
    m.integrate(f0)
    f1 = t0_frame(1)
    f1["track_feats"] = tok1
    rep = m.integrate(f1)
    lf = m.last_frame()
    trip = {(int(s), int(j)): (int(c), int(e)) for s, j, c, e in
            zip(lf["trip_s"], lf["trip_j"], lf["trip_c"], lf["trip_edge"])}
    inst = m.instances()
    return rep, trip, dict(zip(inst["id"].tolist(), inst["vcount"].tolist()))


def test_gate_rejects_orthogonal_tracking_features():
    """Frame 0: A's patches carry e0, B's e1 -> T_0 = e0, T_1 = e1.  Frame 1: every patch e0 ->
    t_C = e0: cos(t_C, T_0) = 1 passes, cos(t_C, T_1) = 0 < 0.8 fails.  Geometric test passes for
    both (720, 768 >= 0.3 * 1536).  So only C -> 0: |V_0| = 1536 + (1536 - 720) = 2352, id 1 keeps
    1536 and survives."""
    rep, trip, inst = gate_run(tokens(lambda c: E0 if c < 8 else E1), tokens(lambda c: E0), 0.8)
    assert trip == {(0, 0): (720, 1), (0, 1): (768, 0)}
    assert inst == {0: 2352, 1: 1536}
    assert rep["edges"] == 1 and rep["merged_away"] == 0 and rep["created"] == 0


@pytest.mark.parametrize("tau,bridged", [(0.5, True), (float(np.nextafter(np.float32(0.5), np.float32(1))), False)])
def test_gate_is_inclusive_at_exactly_tau(tau, bridged):
    """B's patches carry (0.5, 0.5, 0.5, 0.5, 0...) -> u_B = k (0.5,0.5,0.5,0.5), |u_B| = k exactly,
    t_B = (0.5,0.5,0.5,0.5) and T_1 = t_B with dot_pin(T_1, T_1) = 1 exactly.  t_C = e0, so
    cos(t_C, T_1) = 0.5 / sqrt(1) = 0.5 exactly: at tau_vis = 0.5 the edge passes (>=, inclusive) and
    C bridges 0 and 1 (|V_0| = 3120, the T0 golden value); one fp32 ulp above it fails (2352 / 1536)."""
    rep, trip, inst = gate_run(tokens(lambda c: E0 if c < 8 else HALF4), tokens(lambda c: E0), tau)
    if bridged:
        assert trip == {(0, 0): (720, 1), (0, 1): (768, 1)} and inst == {0: gold("t0.json")["tau_0.3"]["after_frame1"]["vcount"][0]}
    else:
        assert trip == {(0, 0): (720, 1), (0, 1): (768, 0)} and inst == {0: 2352, 1: 1536}


def test_gate_zero_norm_detection_never_passes():
    """Frame 1 tokens all zero -> u_C = 0, t_C undefined: cos = -2 for every j, so even
    tau_vis = -1 (every defined cosine passes) rejects both geometric edges and C becomes a new
    instance (id 2, 1536 voxels)."""
    rep, trip, inst = gate_run(tokens(lambda c: E0 if c < 8 else E1), tokens(lambda c: ZERO), -1.0)
    assert trip == {(0, 0): (720, 0), (0, 1): (768, 0)}
    assert inst == {0: 1536, 1: 1536, 2: 1536} and rep["created"] == 1


def test_gate_zero_norm_instance_never_passes():
    """Frame 0: A's patches zero -> T_0 = 0 (t_A undefined, stored as 0), dot_pin(T_0, T_0) = 0 ->
    cos = -2: (C, 0) fails even at tau_vis = -1; B's patches e1, frame 1 all e1 -> cos(t_C, T_1) = 1:
    only C -> 1: |V_1| = 1536 + (1536 - 768) = 2304."""
    rep, trip, inst = gate_run(tokens(lambda c: ZERO if c < 8 else E1), tokens(lambda c: E1), -1.0)
    assert trip == {(0, 0): (720, 0), (0, 1): (768, 1)}
    assert inst == {0: 1536, 1: 2304}
