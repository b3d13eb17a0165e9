"""Pins of the oracle's finalize (NEXT row f1): P:100 [§III-B] "a final, lightweight post-processing
step iterates over the map to merge remaining orphaned candidates and filter out residual noisy
instances, such as segments containing fewer than a minimum threshold of voxels"; S:333-340 and
its three examples; readings R35-R38.

Maps are built on the T0 wall (tests/golden/t0.json: pose I, every pixel its own voxel, so a mask's
voxel set is its pixel set and every count below is a pixel count worked out by hand).  Orphans are
made by integrating at a strict tau_geo (0.95) and finalizing at a looser one (finalize takes its
thresholds explicitly; SPEC's op passes the map's own)."""
import numpy as np
import pytest

from oracle import oracle as O
from synth import t0_frame, Generator, disc_config_kwargs, frame_to_numpy

H, W = 48, 64
U = np.arange(W)[None, :].repeat(H, 0)
V = np.arange(H)[:, None].repeat(W, 1)


def mframe(i, *masks, track=None):
    fr = t0_frame(0)
    fr["frame_id"] = i
    fr["masks"] = np.stack([m.astype(np.uint8) for m in masks])
    if track is not None:
        fr["track_feats"] = track
    return fr


def build(masks_per_frame, tau=0.95, Dt=0, tracks=None):
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, track_dim=Dt, tau_geo=tau, mask_min_area=1, selfcheck=True)
    for i, ms in enumerate(masks_per_frame):
        m.integrate(mframe(i, *ms, track=None if tracks is None else tracks[i]))
    return m


def sets(m):
    keys, ids = m.memberships()
    out = {}
    for k, i in zip(keys.tolist(), ids.tolist()):
        out.setdefault(i, set()).add(k)
    return out


def test_fixpoint_noop():
    """no qualifying pair, every instance >= min_voxels -> unchanged (T0 frame 0: A, B disjoint)."""
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, selfcheck=True)
    m.integrate(t0_frame(0))
    before = sets(m)
    rep = m.finalize(min_voxels=10)
    assert rep["rounds"] == 0 and rep["merged_away"] == 0 and rep["removed"] == 0
    assert sets(m) == before and rep["live_instances"] == 2 and rep["live_memberships"] == 3072


def test_small_instance_removed():
    """an instance of 3 voxels with min_voxels = 10 is removed (with its memberships); a
    10-voxel one is kept (>= is kept: 'fewer than a minimum threshold')."""
    three = (V == 5) & (U >= 10) & (U < 13)
    ten = (V == 30) & (U >= 40) & (U < 50)
    m = build([[three, ten]])
    assert sorted(len(v) for v in sets(m).values()) == [3, 10]
    rep = m.finalize(min_voxels=10)
    assert rep["removed"] == 1 and [len(v) for v in sets(m).values()] == [10]
    assert list(m.instances()["id"]) == [1]


def test_chain_merges_into_one_union_find():
    """A = {u < 24}, B = {16 <= u < 40}, C = {32 <= u < 56} (48 rows): |A ∩ B| = |B ∩ C| =
    8 x 48 = 384 >= 0.3 x 1152, A ∩ C = {} -> the chain A - B - C is one component: one survivor, the
    lower id 0, with |V| = 56 x 48 = 2688; equals the union-find over the qualifying-pair graph
    computed here by brute force (Python set intersections)."""
    A, B, C = U < 24, (U >= 16) & (U < 40), (U >= 32) & (U < 56)
    m = build([[A], [B], [C]])
    S0 = sets(m)
    assert sorted(S0) == [0, 1, 2] and [len(S0[i]) for i in range(3)] == [1152, 1152, 1152]
    parent = {i: i for i in S0}

    def find(x):
        while parent[x] != x:
            x = parent[x]
        return x
    for i in S0:
        for j in S0:
            c = len(S0[i] & S0[j])
            if i < j and c >= 1 and c >= 0.3 * min(len(S0[i]), len(S0[j])):
                parent[max(find(i), find(j))] = min(find(i), find(j))
    rep = m.finalize(tau_geo=0.3, min_voxels=0)
    S1 = sets(m)
    assert rep["rounds"] == 1 and rep["merged_away"] == 2 and rep["edges"] == 2
    assert list(S1) == [0] and len(S1[0]) == 2688
    assert {find(i) for i in S0} == set(S1)
    assert S1[0] == S0[0] | S0[1] | S0[2]
    inst = m.instances()
    assert list(inst["obs"]) == [3] and list(inst["last_seen"]) == [2]


def test_second_round_after_a_merge():
    """Fixpoint (R35): A = {u < 24} (1152), B = {16 <= u < 30, v < 24} (336), |A ∩ B| = 192 >= 0.5 x 336;
    C = R1 ∪ R2 ∪ R3 (72 px: R1 = u in [16,22) x v in [24,28) inside A only, R2 = u in [24,30) x
    v in [20,24) inside B only, R3 = u in [40,46) x v in [30,34) outside both): c(A,C) = c(B,C) = 24
    < 0.5 x 72, so round 1 merges only A and B; then c(A ∪ B, C) = 48 >= 36: round 2 merges C.
    |V| = 1152 + 336 - 192 + 72 - 48 = 1320."""
    A = U < 24
    B = (U >= 16) & (U < 30) & (V < 24)
    C = (((U >= 16) & (U < 22) & (V >= 24) & (V < 28)) | ((U >= 24) & (U < 30) & (V >= 20) & (V < 24))
         | ((U >= 40) & (U < 46) & (V >= 30) & (V < 34)))
    m = build([[A], [B], [C]])
    assert [len(v) for v in sets(m).values()] == [1152, 336, 72]
    rep = m.finalize(tau_geo=0.5, min_voxels=0)
    assert rep["rounds"] == 2 and rep["merged_away"] == 2
    assert {k: len(v) for k, v in sets(m).items()} == {0: 1320}


E0 = [1.0] + [0.0] * 7
E1 = [0.0, 1.0] + [0.0] * 6
BF16 = {0.0: 0x0000, 1.0: 0x3F80}


def track_all(vals):
    g = np.zeros((16, 16, 8), np.uint16)
    for k in range(8):
        g[:, :, k] = BF16[vals[k]]
    return g


@pytest.mark.parametrize("same,merged", [(True, True), (False, False)])
def test_gate_governs_orphan_merges(same, merged):
    """R36: A = {u < 24}, B = {16 <= u < 40} overlap 384 >= 0.3 x 1152; T_A = e0; T_B = e0 (same
    object) -> cos 1 >= 0.8, merged into {u < 40} (40 x 48 voxels), T = T_A + T_B = (2, 0, ...);
    T_B = e1 -> cos 0 < 0.8, kept apart."""
    A, B = U < 24, (U >= 16) & (U < 40)
    m = build([[A], [B]], Dt=8, tracks=[track_all(E0), track_all(E0 if same else E1)])
    rep = m.finalize(tau_geo=0.3, tau_vis=0.8, min_voxels=0)
    inst = m.instances()
    if merged:
        assert rep["merged_away"] == 1 and list(inst["id"]) == [0] and list(inst["vcount"]) == [40 * 48]
        assert inst["T"][0][0] == 2.0 and not inst["T"][0][1:].any()
    else:
        assert rep["merged_away"] == 0 and list(inst["vcount"]) == [1152, 1152]


def test_generated_stream_fixpoint_properties():
    """Orphans on a generated stream (integrated at tau_geo 0.9, finalized at 0.3), checked by brute
    force against the definitions, not against the oracle's own routines: (1) fixpoint -- no pair of
    final instances qualifies; (2) every final voxel set is the union of the pre-finalize sets it
    absorbed, which partition the pre-finalize instances; (3) the filter removed exactly the
    instances below min_voxels; (4) no voxel is lost except those of removed instances."""
    g = Generator("N", device="cpu", H=60, W=80, Hp=4, Wp=5, fx=72.0, fy=72.0, cx=40.0, cy=30.0, Df=16, Dt=0)
    kw = disc_config_kwargs(g.cfg)
    kw.update(mask_min_area=10, tau_geo=0.9)
    m = O.OracleMap(selfcheck=True, **kw)
    for f in range(12):
        m.integrate(frame_to_numpy(g.frame(f)))
    S0 = sets(m)
    rep = m.finalize(tau_geo=0.3, min_voxels=40)
    S1 = sets(m)
    assert rep["merged_away"] > 0
    ids = sorted(S1)
    for a in ids:
        for b in ids:
            if a < b:
                c = len(S1[a] & S1[b])
                assert not (c >= 1 and c >= 0.3 * min(len(S1[a]), len(S1[b])))
    absorbed = {}
    for i, s in S0.items():
        hits = [j for j in S1 if s <= S1[j]]
        if hits:
            absorbed.setdefault(min(hits), []).append(i)
    for j, members in absorbed.items():
        assert j == min(members)
    for j in S1:
        assert S1[j] == set().union(*[S0[i] for i in absorbed[j]])
    assert all(len(v) >= 40 for v in S1.values())
    assert rep["live_memberships"] == sum(len(v) for v in S1.values())
