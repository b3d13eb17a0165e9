"""GPU parity: libdisc (CUDA, through the C ABI) vs the CPU oracle on identical seeded inputs.

Sizes: T (3 frames, several tiles + ragged tails), T0 hand fixture, and prefixes of the full
Replica-, ScanNet- and HM3D-shaped streams at their BASELINE.json resolutions, run through
the same windowed launch configuration bench.py times.  Rules in tests/parity_util.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import pack_mask_bits, Generator, disc_config_kwargs, frame_to_numpy, t0_frame  # noqa: E402
from tests.parity_util import compare_frame_debug, compare_reports, compare_state, gpu_config  # noqa: E402


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _to_dev(fr: dict, dev):
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


def _disc_map(kw, H, W, Hp, Wp, **extra):
    from paper_2603_03935_b200 import DiscMap
    return DiscMap(**gpu_config(kw, H, W, Hp, Wp, **extra))


# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("tau", [0.3, 0.48])
def test_t0_hand_fixture(tau):
    """T0 (golden): both implementations reach 3120 / 2304 and R25 idempotence."""
    dev = _dev()
    kw = dict(voxel_size=0.05, tau_geo=tau, feat_dim=16, track_dim=0)
    gm = _disc_map(kw, 48, 64, 16, 16)
    om = OracleMap(selfcheck=True, **kw)
    for i in range(3):
        fr = t0_frame(i)
        rg = gm.integrate_frame(_to_dev(fr, dev))
        ro = om.integrate(fr)
        compare_reports(rg, ro)
        compare_frame_debug(gm.last_frame(), om.last_frame(), False, 0)
        compare_state(gm, om, False, 0)
    want = [3120] if tau == 0.3 else [1536, 2304]
    assert list(gm.instances()["vcount"]) == want


@pytest.mark.parametrize("semantic", [False, True])
def test_t0_with_tokens_and_gate(semantic):
    dev = _dev()
    kw = dict(voxel_size=0.05, tau_geo=0.3, feat_dim=16, track_dim=8)
    gm = _disc_map(kw, 48, 64, 16, 16)
    om = OracleMap(selfcheck=True, **kw)
    for i in range(3):
        fr = t0_frame(i, with_tokens=semantic, Df=16, Dt=8)
        compare_reports(gm.integrate_frame(_to_dev(fr, dev)), om.integrate(fr))
        compare_frame_debug(gm.last_frame(), om.last_frame(), semantic, 8)
        compare_state(gm, om, semantic, 8)


@pytest.mark.parametrize("semantic", [False, True])
def test_tiny_config_every_frame(semantic):
    """T config: every frame, full debug + state parity (M1 and M2)."""
    dev = _dev()
    g = Generator("T", device=dev)
    kw = disc_config_kwargs(g.cfg)
    c = g.cfg
    gm = _disc_map(kw, c.H, c.W, c.Hp, c.Wp)
    om = OracleMap(selfcheck=True, **kw)
    for f in range(c.frames):
        fr = g.frame(f, with_feats=semantic)
        fr["mask_conf"] = torch.clamp(fr["mask_conf"], min=0.45)
        compare_reports(gm.integrate_frame(fr), om.integrate(frame_to_numpy(fr)))
        compare_frame_debug(gm.last_frame(), om.last_frame(), semantic, c.Dt)
        compare_state(gm, om, semantic, c.Dt)


def _bits(fr):
    """The frame with its masks bit-packed (disc_frame::mask_bits) instead of byte planes."""
    out = {k: v for k, v in fr.items() if k != "masks"}
    out["mask_bits"] = pack_mask_bits(fr["masks"])
    return out


def _stream_parity(name, nframes, semantic, window, every=1, caps=None, reports=True, bits=False, **over):
    dev = _dev()
    g = Generator(name, device=dev, **over)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=window, S=min(255, max(64, int(c.n_masks * 1.2) + 8)), **(caps or {}))
    om = OracleMap(**kw)
    frames = [g.frame(f, with_feats=semantic) for f in range(nframes)]
    # (the oracle always reads byte planes; bits="mixed": every other frame packed, one window mixes both)
    gframes = [(_bits(fr) if (bits is True or i % 2) else fr) for i, fr in enumerate(frames)] if bits else frames
    # windowed GPU integration (the launch configuration bench.py times)
    # (without reports no call waits for its window: window w+1's stage 1 overlaps w's stage 2)
    reps_g = []
    for w0 in range(0, nframes, window):
        r = gm.integrate_frames(gframes[w0:w0 + window], report=reports)
        reps_g += r if reports else []
    reps_o = [om.integrate(frame_to_numpy(fr)) for fr in frames]
    for rg, ro in zip(reps_g, reps_o):
        compare_reports(rg, ro)
    compare_frame_debug(gm.last_frame(), om.last_frame(), semantic, c.Dt)
    compare_state(gm, om, semantic, c.Dt)
    return reps_o


@pytest.mark.parametrize("semantic", [False, True])
def test_replica_prefix(semantic):
    reps = _stream_parity("R", 8, semantic, window=4)
    assert sum(r["unique_pairs"] for r in reps) > 10000


@pytest.mark.parametrize("semantic", [False, True])
@pytest.mark.parametrize("reports", [True, False])
def test_replica_bench_launch_configuration(semantic, reports):
    """The bench's launch configuration on its workload: Replica-shaped frames, 32-frame windows,
    bench.py's capacities (pairs 2^16 per frame, 2^23 memberships, 2^17 instances), two windows
    -- per-frame reports, the last frame's debug export and the whole map compared with the oracle;
    without reports the windows run as in bench.py (stage 1 of window w+1 beside stage 2 of w)."""
    _stream_parity("R", 64, semantic, window=32, reports=reports,
                   caps=dict(max_pairs=1 << 16, max_memberships=1 << 23, max_instances=1 << 17))


@pytest.mark.parametrize("semantic", [False, True])
def test_scannet_prefix(semantic):
    _stream_parity("N", 8, semantic, window=8)


def test_hm3d_prefix():
    _stream_parity("H", 8, True, window=8)


@pytest.mark.parametrize("name,pmax", [("H", 1 << 18), ("N", 1 << 16)])
def test_bench_launch_configuration_h_n(name, pmax):
    """`bench.py --config H|N`'s launch configuration: 32-frame windows, its capacities (pairs 2^18
    per frame for H, 2^16 for N), no per-window reports (window 2's stage 1 beside window 1's
    stage 2), a ragged second window of 8 frames; the last frame's debug export and the whole map
    compared with the oracle."""
    _stream_parity(name, 40, True, window=32, reports=False,
                   caps=dict(max_pairs=pmax, max_memberships=1 << 23, max_instances=1 << 17))


def test_stress_overlapping_masks():
    """X-style SAM 'everything' masks (overlapping, hierarchical), Df 512, 10 cm voxels."""
    _stream_parity("X", 6, True, window=6, n_masks=120, Df=512, voxel=0.1)


@pytest.mark.parametrize("name,n_masks,Df,voxel", [("X", 10, 768, 0.01), ("X", 150, 1024, 0.05),
                                                    ("X", 100, 512, 0.02), ("X", 200, 512, 0.05),
                                                    ("X", 200, 1024, 0.1), ("X", 255, 512, 0.1)])
def test_stress_sweep_points(name, n_masks, Df, voxel):
    """Points of BASELINE configs[4] (voxel 1-10 cm x masks 10-200 x Df 512/768/1024) and the ABI's
    maximum S = 255 (disc.h max_masks): X-style hierarchical SAM-"everything" masks (overlapping whole /
    half / quarter masks).  Frame 1's kept masks all become instances that frame 2's masks overlap, so
    S = 200 / 255 frames carry several thousand (s, j) triples -- past the association's shared-memory
    tables (3072), through its global-memory layout.  4 frames each."""
    reps = _stream_parity(name, 4, True, window=4, n_masks=n_masks, Df=Df, voxel=voxel)
    # the generator really produced (close to) n_masks masks, and most are kept
    assert max(r["kept"] + r["drop_area"] + r["drop_conf"] + r["drop_aspect"] + r["drop_nodepth"]
               + r["drop_nofeat"] for r in reps) >= int(0.9 * n_masks)
    assert max(r["kept"] for r in reps) >= min(8, n_masks // 2)


@pytest.mark.parametrize("name,frames,over", [("R", 6, {}), ("X", 4, dict(n_masks=120, Df=512, voxel=0.1))])
def test_global_memory_association_layout(name, frames, over, monkeypatch):
    """DISC_K6_TCS=0 (read at map creation) sends every frame with at least one (s, j) triple
    through the association's global-memory layout: same results as the shared-memory tables."""
    monkeypatch.setenv("DISC_K6_TCS", "0")
    _stream_parity(name, frames, True, window=frames, **over)


def test_triple_capacity_overflow_is_loud(monkeypatch):
    """A frame whose (s, j) triples pass the configured per-frame capacity (lowered here to 1000 with
    the test knob DISC_TCAP; the default is 256 x max_masks) fails with the sticky
    DISC_ERR_CAPACITY instead of dropping counts."""
    from paper_2603_03935_b200.disc import DiscError
    monkeypatch.setenv("DISC_TCAP", "1000")
    dev = _dev()
    g = Generator("X", device=dev, n_masks=200, Df=512, voxel=0.05)
    c = g.cfg
    gm = _disc_map(disc_config_kwargs(c), c.H, c.W, c.Hp, c.Wp, window=4, S=200)
    with pytest.raises(DiscError) as e:
        gm.integrate_frames([g.frame(f, with_feats=True) for f in range(4)], report=True)
    assert e.value.code == 5 and "count table full" in str(e.value)   # DISC_ERR_CAPACITY
    with pytest.raises(DiscError):    # sticky
        gm.integrate_frames([g.frame(4, with_feats=True)], report=True)


def test_tiny_voxels_overflow_tile_tables():
    """2 mm voxels: nearly every pixel is its own voxel, so the mask pass's per-tile key / pair
    tables overflow and items take the direct path into the frame tables."""
    reps = _stream_parity("N", 3, True, window=3, voxel=0.002)
    assert max(r["unique_pairs"] for r in reps) > 100000


@pytest.mark.parametrize("rcap", [0, 3000])
def test_record_list_overflow_direct_path(rcap, monkeypatch):
    """K1b hands each tile's distinct (s, key) items to K1c through a per-frame record list; a
    tile whose records would pass the list's capacity inserts them into the frame tables itself
    (and blanks its reserved records).  A lowered capacity (test knob DISC_K1_RCAP, read at map
    creation) mixes both paths inside one frame (3000) or sends every tile direct (0)."""
    monkeypatch.setenv("DISC_K1_RCAP", str(rcap))
    _stream_parity("R", 4, True, window=4)


@pytest.mark.parametrize("semantic", [False, True])
def test_single_cta_stage2(semantic, monkeypatch):
    """A one-CTA stage-2 grid (DISC_S2_SMS=1, read at map creation): no helper CTAs, so the
    association gates its candidates itself and nothing prefetches; same results."""
    monkeypatch.setenv("DISC_S2_SMS", "1")
    monkeypatch.setenv("DISC_S2_SMS_GEO", "1")
    _stream_parity("R", 4, semantic, window=4)


def test_odd_tracking_dim_register_path():
    """Odd Dt: tracking rows are not 16-byte multiples, so the K7 target warps sum them from
    registers instead of the async-copy staging; the fp64 sums stay bit-exact."""
    _stream_parity("N", 6, True, window=3, Dt=37)


def test_ragged_image_scalar_path():
    """W*H not a multiple of 16: the byte-wise mask path; odd patch grid."""
    _stream_parity("N", 4, True, window=2, H=239, W=317, Hp=17, Wp=22, fx=290.0, fy=290.0, cx=158.0, cy=119.0)


def test_window_batching_equals_single_frames():
    dev = _dev()
    g = Generator("N", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f) for f in range(10)]
    a = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=8)
    b = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=1)
    ra = a.integrate_frames(frames, report=True)
    rb = [b.integrate_frame(fr) for fr in frames]
    assert ra == rb
    ka, ia = a.memberships()
    kb, ib = b.memberships()
    assert np.array_equal(ka, kb) and np.array_equal(ia, ib)
    A, B = a.instances(), b.instances()
    for k in ["id", "vcount", "obs", "aabb", "T"]:
        assert np.array_equal(A[k], B[k])


def test_host_input_path_equals_device_path():
    dev = _dev()
    g = Generator("T", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f) for f in range(3)]
    a = _disc_map(kw, c.H, c.W, c.Hp, c.Wp)
    b = _disc_map(kw, c.H, c.W, c.Hp, c.Wp)
    ra = a.integrate_frames(frames, report=True)
    host = [{k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in fr.items()} for fr in frames]
    rb = b.integrate_frames_host(host, report=True)
    assert ra == rb
    assert np.array_equal(a.memberships()[0], b.memberships()[0])


def test_query_parity():
    dev = _dev()
    g = Generator("N", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = _disc_map(kw, c.H, c.W, c.Hp, c.Wp)
    om = OracleMap(**kw)
    for f in range(4):
        fr = g.frame(f)
        gm.integrate_frame(fr)
        om.integrate(frame_to_numpy(fr))
    q = g.proto[7].cpu().numpy()
    ig, sg = gm.query(q, 5)
    io, so = om.query(q, 5)
    np.testing.assert_allclose(sg, so, atol=2e-5)
    # ids equal except where scores tie within 1e-6
    for a, b, s in zip(ig, io, so):
        if a != b:
            assert np.sum(np.abs(so - s) < 1e-6) > 1


def test_invalid_frame_is_rejected_before_mutation():
    from paper_2603_03935_b200 import DiscError
    dev = _dev()
    kw = dict(voxel_size=0.05, feat_dim=16, track_dim=0)
    gm = _disc_map(kw, 48, 64, 16, 16)
    gm.integrate_frame(_to_dev(t0_frame(0), dev))
    k0, i0 = gm.memberships()
    bad = t0_frame(1)
    bad["pose"] = bad["pose"].copy()
    bad["pose"][0, 0] = 1.5
    with pytest.raises(DiscError) as e:
        gm.integrate_frame(_to_dev(bad, dev))
    assert e.value.code == 2
    k1, i1 = gm.memberships()
    assert np.array_equal(k0, k1) and np.array_equal(i0, i1)


def test_empty_and_degenerate_frames():
    """S = 0; all-invalid depth (every mask 'nodepth'); then a normal frame."""
    dev = _dev()
    kw = dict(voxel_size=0.05, feat_dim=16, track_dim=0)
    gm = _disc_map(kw, 48, 64, 16, 16)
    om = OracleMap(selfcheck=True, **kw)
    fr0 = t0_frame(0)
    e = dict(fr0, masks=np.zeros((0, 48, 64), np.uint8))
    nod = dict(fr0, frame_id=1, depth=np.zeros((48, 64), np.float32))
    for fr in [e, nod, dict(fr0, frame_id=2)]:
        compare_reports(gm.integrate_frame(_to_dev(fr, dev)), om.integrate(fr))
        compare_state(gm, om, False, 0)


@pytest.mark.parametrize("name,nf", [("R", 8), ("X", 4)])
def test_gpu_determinism(name, nf):
    """Bit-identical snapshots across runs, embeddings and Q included: the pooled sums, the
    R18 / R19 sums and the S_angle sums are fixed-point integer accumulations (order-independent),
    tracking sums exact (R15), everything else integer."""
    dev = _dev()
    over = dict(n_masks=120, Df=512, voxel=0.05) if name == "X" else {}
    g = Generator(name, device=dev, **over)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f) for f in range(nf)]
    outs = []
    for _ in range(3):
        gm = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=4, S=max(64, c.n_masks))
        gm.integrate_frames(frames)
        outs.append((gm.memberships(), gm.instances(), gm.last_frame()))
    (ka, ia), A, LA = outs[0]
    for (kb, ib), B, LB in outs[1:]:
        assert np.array_equal(ka, kb) and np.array_equal(ia, ib)
        for k in ["id", "vcount", "obs", "aabb", "T", "e", "q"]:
            assert np.array_equal(A[k], B[k]), k
        for k in ["e", "factors", "t", "target"]:
            assert np.array_equal(LA[k], LB[k]), k


def test_host_path_rejects_invalid_frame_before_any_window():
    """disc_integrate_frames_host validates all n frames before the first window runs: an invalid
    last frame (non-rigid pose) returns DISC_ERR_INVALID with the map untouched (disc.h errors)."""
    from paper_2603_03935_b200 import DiscError
    dev = _dev()
    g = Generator("T", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=2)
    frames = [g.frame(f % 3) for f in range(5)]
    host = [{k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in fr.items()} for fr in frames]
    host[4]["pose"] = np.array(host[4]["pose"], np.float32).copy()
    host[4]["pose"][0, 0] = 1.5
    with pytest.raises(DiscError) as e:
        gm.integrate_frames_host(host, report=True)
    assert e.value.code == 2
    k, i = gm.memberships()
    assert k.shape[0] == 0 and gm.instances()["id"].shape[0] == 0


def _fixture_pair(kw, frames, semantic, Dt):
    dev = _dev()
    gm = _disc_map(kw, 48, 64, 16, 16)
    om = OracleMap(selfcheck=True, **kw)
    for fr in frames:
        compare_reports(gm.integrate_frame(_to_dev(fr, dev)), om.integrate(fr))
        compare_frame_debug(gm.last_frame(), om.last_frame(), semantic, Dt)
        compare_state(gm, om, semantic, Dt)
    return gm


@pytest.mark.parametrize("case", ["orthogonal", "exact_tau", "above_tau", "zero_t", "zero_T"])
def test_visual_gate_fixtures(case):
    """The oracle's gate pins (tests/test_oracle_pins_angle_gate.py: orthogonal tracking features,
    cos exactly = tau_vis (inclusive) and one ulp above, zero-norm t and zero-norm T) through the GPU:
    bit-exact triples, edge flags, memberships and T."""
    from tests.test_oracle_pins_angle_gate import E0, E1, HALF4, ZERO, tokens
    tok0, tok1, tau = {
        "orthogonal": (tokens(lambda c: E0 if c < 8 else E1), tokens(lambda c: E0), 0.8),
        "exact_tau": (tokens(lambda c: E0 if c < 8 else HALF4), tokens(lambda c: E0), 0.5),
        "above_tau": (tokens(lambda c: E0 if c < 8 else HALF4), tokens(lambda c: E0),
                      float(np.nextafter(np.float32(0.5), np.float32(1)))),
        "zero_t": (tokens(lambda c: E0 if c < 8 else E1), tokens(lambda c: ZERO), -1.0),
        "zero_T": (tokens(lambda c: ZERO if c < 8 else E1), tokens(lambda c: E1), -1.0),
    }[case]
    f0, f1 = t0_frame(0), t0_frame(1)
    f0["track_feats"], f1["track_feats"] = tok0, tok1
    kw = dict(voxel_size=0.05, feat_dim=4, track_dim=8, tau_geo=0.3, tau_vis=tau)
    _fixture_pair(kw, [f0, f1], False, 8)


@pytest.mark.parametrize("case", ["holes", "tilted"])
def test_s_angle_fixtures(case):
    """The oracle's S_angle pins (depth holes; a wall seen by a camera tilted by 20 deg) through the
    GPU: S_angle and Q within the R22 tolerance, everything else bit-exact."""
    import math
    from tests.test_oracle_pins_angle_gate import D0, semantic_t0
    if case == "holes":
        depth = np.full((48, 64), np.float32(D0), np.float32)
        for u, v in [(10, 10), (11, 20)] + [(u, 30) for u in range(40, 47)] + [(5, 40), (6, 41)]:
            depth[v, u] = 0.0
        fr = semantic_t0(0, depth=depth)
    else:
        th = math.radians(20.0)
        pose = np.eye(4, dtype=np.float32)
        pose[:3, :3] = np.array([[math.cos(th), 0, math.sin(th)], [0, 1, 0], [-math.sin(th), 0, math.cos(th)]],
                                np.float32)
        Rf = pose[:3, :3].astype(np.float64)
        depth = np.zeros((48, 64), np.float32)
        for v in range(48):
            for u in range(64):
                depth[v, u] = np.float32(D0 / (Rf[2] @ np.array([(u - 32.0) / 32.0, (v - 24.0) / 32.0, 1.0])))
        fr = semantic_t0(0, depth=depth, masks=np.ones((1, 48, 64), np.uint8))
        fr["pose"] = pose
    _fixture_pair(dict(voxel_size=0.05, feat_dim=16, track_dim=0), [fr], True, 0)


@pytest.mark.parametrize("name,nf", [("N", 10), ("H", 6), ("R", 4)])
def test_every_frame_debug_export(name, nf):
    """Full-size frames one call each, so the per-frame debug export (statuses, |V_s|, the unique
    (s, key) pairs, C triples, edges, targets, Q factors, e_s, t_s) is compared on EVERY frame, not only a
    window's last one; the map state after each frame too."""
    dev = _dev()
    g = Generator(name, device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    gm = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=1, S=min(255, max(64, int(c.n_masks * 1.2) + 8)))
    om = OracleMap(**kw)
    for f in range(nf):
        fr = g.frame(f, with_feats=True)
        compare_reports(gm.integrate_frame(fr), om.integrate(frame_to_numpy(fr)))
        compare_frame_debug(gm.last_frame(), om.last_frame(), True, c.Dt)
        compare_state(gm, om, True, c.Dt)


@pytest.mark.parametrize("spec", ["0", "1", "2", "3"])
@pytest.mark.parametrize("name,nf,window", [("R", 8, 4), ("H", 6, 6)])
def test_stage2_speculation_modes(spec, name, nf, window, monkeypatch):
    """Stage 2's speculative work (DISC_S2_SPEC, read at map creation): 2 (default) counts frame f+1
    during frame f's association and corrects the counts in frame f's update; 3 the same with the gate
    on CTAs of its own; 1 only finds the slots early; 0 L2 hints.  Every mode gives the oracle's
    per-frame reports, the window's last-frame debug export (a speculatively counted frame in 2 / 3)
    and the map state."""
    monkeypatch.setenv("DISC_S2_SPEC", spec)
    _stream_parity(name, nf, True, window=window)


@pytest.mark.parametrize("name,nf,window,over", [
    ("R", 8, 4, {}),                                                                   # vector K1a path
    ("X", 4, 4, dict(n_masks=60, Df=256)),                                             # overlapping masks (R9)
    ("N", 4, 2, dict(H=239, W=317, Hp=17, Wp=22, fx=290.0, fy=290.0, cx=158.0, cy=119.0)),   # H*W % 32 != 0
    ("H", 6, 6, {}),
])
def test_bit_packed_masks(name, nf, window, over):
    """disc_frame::mask_bits (masks bit-packed, 1/8 of the bytes) gives exactly the oracle's results
    on its byte planes: per-frame reports, the last frame's debug export, the map."""
    _stream_parity(name, nf, True, window=window, bits=True, **over)


def test_mixed_mask_formats_in_a_window():
    """Byte and bit-packed planes in one window (K1a's per-frame variant)."""
    _stream_parity("R", 6, True, window=6, bits="mixed")


def test_bit_packed_masks_host_path():
    """The host-input path stages the packed planes (ceil(H*W/32) words per mask) and gives the same
    map as the device path with byte planes."""
    dev = _dev()
    g = Generator("N", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f) for f in range(6)]
    a = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=3)
    b = _disc_map(kw, c.H, c.W, c.Hp, c.Wp, window=3)
    ra = a.integrate_frames(frames, report=True)
    host = [{k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in _bits(fr).items()}
            for fr in frames]
    rb = b.integrate_frames_host(host, report=True)
    assert ra == rb
    assert np.array_equal(a.memberships()[0], b.memberships()[0])
    A, B = a.instances(), b.instances()
    for k in ["id", "vcount", "obs", "aabb", "T", "e", "q"]:
        assert np.array_equal(A[k], B[k])


def test_mask_formats_exclusive():
    """Exactly one of masks / mask_bits: both or neither (S > 0) is DISC_ERR_INVALID."""
    from paper_2603_03935_b200.disc import DiscError
    dev = _dev()
    g = Generator("T", device=dev)
    c = g.cfg
    m = _disc_map(disc_config_kwargs(c), c.H, c.W, c.Hp, c.Wp)
    fr = g.frame(0)
    with pytest.raises(DiscError):
        m.integrate_frame(dict(fr, mask_bits=pack_mask_bits(fr["masks"])))
    with pytest.raises(DiscError):
        m.integrate_frame({k: v for k, v in fr.items() if k != "masks"} | {"masks": None, "num_masks": 2})
