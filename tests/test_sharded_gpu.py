"""The key-hash-sharded map on one GPU: G shards in one process
(disc_config.world_size = G, nccl_unique_id = NULL), the exchanges between them done by device
copies -- the same kernels, data layouts and exchange points as the NCCL path (one shard per rank).

Parity: every per-frame report, the last frame's debug export (pairs = union of the shards' routed
pairs, merged C triples, edges, targets), memberships (union of the shards' disjoint key sets) and the
instance table equal the CPU oracle's (tests/parity_util.py rules), and equal the unsharded map's
bit for bit (integer fields and the fp64 tracking sums)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import OracleMap  # noqa: E402
from synth import Generator, disc_config_kwargs, frame_to_numpy  # noqa: E402
from tests.parity_util import compare_frame_debug, compare_reports, compare_state, gpu_config  # noqa: E402


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _map(kw, c, G, window, S, **caps):
    from paper_2603_03935_b200 import DiscMap
    cfg = gpu_config(kw, c.H, c.W, c.Hp, c.Wp, window=window, S=S, **caps)
    if G > 1:
        cfg["world_size"] = G
    return DiscMap(**cfg)


def _run(gm, frames, window):
    reps = []
    for w0 in range(0, len(frames), window):
        reps += gm.integrate_frames(frames[w0:w0 + window], report=True)
    return reps


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("name,nframes,window,semantic,over", [
    ("T", 3, 4, True, {}),
    ("R", 8, 8, True, {}),
    ("N", 12, 8, False, {}),
    ("H", 8, 8, True, {}),
])
def test_virtual_shards_match_oracle(G, name, nframes, window, semantic, over):
    dev = _dev()
    g = Generator(name, device=dev, **over)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f, with_feats=semantic) for f in range(nframes)]
    if not semantic:
        frames = [dict(fr, patch_feats=None, global_embed=None) for fr in frames]
    S = max(64, int(c.n_masks * 1.2) + 8)
    gm = _map(kw, c, G, window, S)
    om = OracleMap(**kw)
    reps_g = _run(gm, frames, window)
    reps_o = [om.integrate(frame_to_numpy(fr)) for fr in frames]
    for rg, ro in zip(reps_g, reps_o):
        compare_reports(rg, ro)
    compare_frame_debug(gm.last_frame(), om.last_frame(), semantic, c.Dt)
    compare_state(gm, om, semantic, c.Dt)


@pytest.mark.parametrize("G", [2, 4])
def test_virtual_shards_dense_stress_point(G):
    """X at S = 200 hierarchical masks: thousands of (s, j) triples per frame, each shard holding a
    part of every count -- the merged triples (and the global-memory association layout) match."""
    dev = _dev()
    g = Generator("X", device=dev, n_masks=200, Df=512, voxel=0.05)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f, with_feats=True) for f in range(4)]
    gm = _map(kw, c, G, 4, 200)
    om = OracleMap(**kw)
    for rg, ro in zip(_run(gm, frames, 4), [om.integrate(frame_to_numpy(fr)) for fr in frames]):
        compare_reports(rg, ro)
    compare_frame_debug(gm.last_frame(), om.last_frame(), True, c.Dt)
    compare_state(gm, om, True, c.Dt)


def test_sharded_equals_unsharded_bitwise():
    """G = 3 vs G = 1 on 40 Replica-shaped frames (two windows of 32, the second ragged): identical
    reports, memberships, instance ids / |V| / obs / last_seen / aabb and fp64 T sums."""
    dev = _dev()
    g = Generator("R", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [dict(fr, patch_feats=None, global_embed=None) for fr in (g.frame(f, with_feats=False) for f in range(40))]
    a = _map(kw, c, 1, 32, 64, max_pairs=1 << 17)
    b = _map(kw, c, 3, 32, 64, max_pairs=1 << 17)
    assert _run(a, frames, 32) == _run(b, frames, 32)
    ka, ia = a.memberships()
    kb, ib = b.memberships()
    assert np.array_equal(ka, kb) and np.array_equal(ia, ib)
    A, B = a.instances(), b.instances()
    for k in ["id", "vcount", "obs", "last_seen", "aabb", "T"]:
        assert np.array_equal(A[k], B[k]), k


def test_sharded_keys_spread_over_the_shards():
    """Routing really distributes the map: each of G = 4 shards holds its owned share of the live
    memberships (disc_stats.shard_memberships; owner = mix64(key) >> 40 mod G, ~1/G each), and the
    shares sum to the whole relation."""
    dev = _dev()
    g = Generator("N", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    G = 4
    gm = _map(kw, c, G, 8, 64)
    _run(gm, [g.frame(f, with_feats=False) for f in range(8)], 8)
    keys, _ = gm.memberships()
    per = gm.stats()["shard_memberships"][:G]
    assert sum(per) == keys.shape[0]
    assert min(per) > 0.8 * keys.shape[0] / G and max(per) < 1.2 * keys.shape[0] / G, per


def test_sharded_host_input_path():
    """disc_integrate_frames_host on a sharded map (each shard stages its own frames)."""
    dev = _dev()
    g = Generator("T", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f) for f in range(3)]
    a = _map(kw, c, 2, 4, 64)
    b = _map(kw, c, 1, 4, 64)
    host = [{k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in fr.items()} for fr in frames]
    assert a.integrate_frames_host(host, report=True) == b.integrate_frames(frames, report=True)
    assert np.array_equal(a.memberships()[0], b.memberships()[0])


def test_sharded_with_dbscan():
    """The DBSCAN denoise (f3) runs in every shard's stage 1: a G = 2 map with dbscan on equals the
    oracle (small N frames, noisy depth)."""
    dev = _dev()
    g = Generator("N", device=dev, H=96, W=128, Hp=6, Wp=9, fx=115.5, fy=115.7, cx=63.8, cy=48.5, min_area=40)
    c = g.cfg
    kw = disc_config_kwargs(c)
    kw.update(dbscan_eps=0.1, dbscan_min_pts=8)
    gm = _map(kw, c, 2, 4, 64)
    om = OracleMap(**kw)
    frames = [g.frame(f) for f in range(6)]
    for rg, ro in zip(_run(gm, frames, 4), [om.integrate(frame_to_numpy(fr)) for fr in frames]):
        compare_reports(rg, ro)
    compare_frame_debug(gm.last_frame(), om.last_frame(), True, c.Dt)
    compare_state(gm, om, True, c.Dt)


@pytest.mark.parametrize("host", [False, True])
def test_sharded_bit_packed_masks(host):
    """Bit-packed mask planes (disc_frame::mask_bits) on a 2-shard map, device and host-input paths:
    the same reports and map as the unsharded map on byte planes."""
    from synth import pack_mask_bits
    dev = _dev()
    g = Generator("R", device=dev)
    c = g.cfg
    kw = disc_config_kwargs(c)
    frames = [g.frame(f) for f in range(6)]
    packed = [{k: v for k, v in fr.items() if k != "masks"} | {"mask_bits": pack_mask_bits(fr["masks"])} for fr in frames]
    a = _map(kw, c, 2, 6, 64)
    b = _map(kw, c, 1, 6, 64)
    if host:
        packed = [{k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in fr.items()} for fr in packed]
        ra = a.integrate_frames_host(packed, report=True)
    else:
        ra = a.integrate_frames(packed, report=True)
    assert ra == b.integrate_frames(frames, report=True)
    assert np.array_equal(a.memberships()[0], b.memberships()[0])
