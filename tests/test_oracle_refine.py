"""Pins of the oracle's per-frame active-set refinement (NEXT row f2; refine_active = 1): SPEC S:327
step (3) "within the active set, merge existing instance pairs meeting the same (tau_geo, tau_vis) test,
keeping the lower id and the higher-Q semantic feature; repeat pairwise merging until no pair
qualifies"; "newly detected instances and nearby existing instances are merged ... among all
candidates"; reading R43.

Maps on the T0 wall (tests/golden/t0.json: pose I, one voxel per pixel, so voxel counts are pixel
counts worked out by hand below)."""
import numpy as np

from oracle import oracle as O
from synth import t0_frame, Generator, disc_config_kwargs, frame_to_numpy
from tests.test_oracle_finalize import U, V, mframe, sets, track_all, E0, E1


def run(frames, refine, tau=0.5, Dt=0, tracks=None):
    m = O.OracleMap(voxel_size=0.05, feat_dim=4, track_dim=Dt, tau_geo=tau, mask_min_area=1, refine_active=refine,
                    selfcheck=True)
    reps = [m.integrate(mframe(i, *ms, track=None if tracks is None else tracks[i])) for i, ms in enumerate(frames)]
    return m, reps


def test_same_frame_overlapping_detections_merge():
    """Two detections of one frame never link directly (R9): A = {u < 24} (1152), B = {16 <= u < 30,
    v < 24} (336) become ids 0 and 1.  Both are targets, so the refinement tests (0, 1): |A ∩ B| = 8 x 24 =
    192 >= 0.5 x 336 -> merged into 0, |V| = 1152 + 336 - 192 = 1296."""
    A, B = U < 24, (U >= 16) & (U < 30) & (V < 24)
    m0, _ = run([[A, B]], 0)
    assert {k: len(v) for k, v in sets(m0).items()} == {0: 1152, 1: 336}
    m1, reps = run([[A, B]], 1)
    assert {k: len(v) for k, v in sets(m1).items()} == {0: 1296}
    r = reps[0]
    assert r["refine_rounds"] == 1 and r["refine_merged"] == 1 and r["merged_away"] == 1 and r["created"] == 2
    assert r["live_instances"] == 1 and r["live_memberships"] == 1296 and r["relabeled"] == 336


def test_merge_that_makes_a_pair_qualify():
    """A = {u < 16} (768).  Frame 1: B = {12 <= u < 40} (1344), |B ∩ A| = 192 < 0.5 x 768: new id 1; the
    active pair (0, 1) fails the same test.  Frame 2: D = {u < 12, v < 20} ∪ {16 <= u < 40} (240 + 1152 =
    1392): |D ∩ A| = 240 < 0.5 x 768 (no edge), |D ∩ B| = 1152 >= 0.5 x 1344 -> D joins 1, which becomes
    B' = B ∪ D (1584).  Now |A ∩ B'| = 192 + 240 = 432 >= 0.5 x 768: the refinement merges A and B' into
    0 = {u < 40} (40 x 48 = 1920).  Without it: 0 (768) and 1 (1584)."""
    A = U < 16
    B = (U >= 12) & (U < 40)
    D = ((U < 12) & (V < 20)) | ((U >= 16) & (U < 40))
    m0, _ = run([[A], [B], [D]], 0)
    assert {k: len(v) for k, v in sets(m0).items()} == {0: 768, 1: 1584}
    m1, reps = run([[A], [B], [D]], 1)
    assert [r["refine_merged"] for r in reps] == [0, 0, 1]
    assert {k: len(v) for k, v in sets(m1).items()} == {0: 1920}
    assert list(m1.instances()["obs"]) == [3]


def test_gate_blocks_refinement():
    """The first case with tracking features.  Every patch e0 -> T_0 = T_1 = e0, cos 1: merged (1296).
    Patch columns >= 4 (u >= 16) e1: t_B = e1 (B lies in columns 4-7), t_A = (768 e0 + 384 e1) / |.| =
    (2, 1) / sqrt(5) -> cos = 1 / sqrt(5) = 0.447 < 0.8: kept apart (1152, 336)."""
    A, B = U < 24, (U >= 16) & (U < 30) & (V < 24)
    diff = track_all(E0)
    diff[:, 4:] = track_all(E1)[:, 4:]
    m, _ = run([[A, B]], 1, Dt=8, tracks=[track_all(E0)])
    assert {k: len(v) for k, v in sets(m).items()} == {0: 1296}
    m, _ = run([[A, B]], 1, Dt=8, tracks=[diff])
    assert {k: len(v) for k, v in sets(m).items()} == {0: 1152, 1: 336}


def test_generated_stream_active_fixpoint():
    """On a generated stream with refine_active: after every frame, no pair of the frame's active set
    (the C triples' instances taken to their survivors, and the targets) passes the test any more --
    checked by brute force on the final voxel sets; the union of all voxels equals the run without
    refinement (it only merges), and refinement merges really happen."""
    g = Generator("N", device="cpu", H=60, W=80, Hp=4, Wp=5, fx=72.0, fy=72.0, cx=40.0, cy=30.0, Df=16, Dt=0)
    kw = disc_config_kwargs(g.cfg)
    kw.update(mask_min_area=10, tau_geo=0.5)
    m1 = O.OracleMap(selfcheck=True, refine_active=1, **kw)
    m0 = O.OracleMap(selfcheck=True, **kw)
    merged = 0
    for f in range(12):
        fr = frame_to_numpy(g.frame(f))
        r = m1.integrate(fr)
        m0.integrate(fr)
        merged += r["refine_merged"]
        lf = m1.last_frame()
        S1 = sets(m1)
        alive = set(S1)
        act = {int(t) for t, st in zip(lf["target"], lf["status"]) if st == 0}
        act |= {j for j in lf["trip_j"].tolist() if j in alive}
        act = sorted(a for a in act if a in alive)
        for a in act:
            for b in act:
                if a < b:
                    c = len(S1[a] & S1[b])
                    assert not (c >= 1 and c >= 0.5 * min(len(S1[a]), len(S1[b]))), (f, a, b)
    assert merged > 0
    k1, _ = m1.memberships()
    k0, _ = m0.memberships()
    assert set(k1.tolist()) == set(k0.tolist())
