"""N > 1 host path on CPU (gloo, world_size 2): rank setup, per-rank scene streams, barrier,
max-over-ranks timing and the weak-scaling aggregate used by bench.py.  The per-rank workload is
the CPU oracle on a small generated stream (test infrastructure)."""
import os
import socket
import time

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2603_03935_b200 import parallel as par
    from synth import Generator, disc_config_kwargs, frame_to_numpy
    from synth.scenes import seed_of
    from oracle.oracle import OracleMap
    r = par.setup("gloo")
    g = Generator("N", seed=par.stream_seed(seed_of("N"), r.rank), H=60, W=80, Hp=4, Wp=5, fx=72.0, fy=72.0,
                  cx=40.0, cy=30.0, Df=16, Dt=8)
    kw = disc_config_kwargs(g.cfg)
    kw["mask_min_area"] = 10
    frames = [frame_to_numpy(g.frame(f)) for f in range(3 + r.rank)]   # uneven work per rank
    om = OracleMap(**kw)
    par.barrier(r)
    t0 = time.perf_counter()
    for fr in frames:
        om.integrate(fr)
    dt = time.perf_counter() - t0
    rate = par.weak_scaling_rate(len(frames), dt, r)
    mx = par.max_over_ranks(dt, r)
    keys, ids = om.memberships()
    q.put((r.rank, rate, mx, dt, len(frames), int(np.bitwise_xor.reduce(keys)) if len(keys) else 0))
    par.teardown(r)


@pytest.mark.timeout(300)
def test_two_rank_weak_scaling_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, rate0, mx0, dt0, n0, h0), (r1, rate1, mx1, dt1, n1, h1) = out
    assert (r0, r1) == (0, 1)
    assert mx0 == mx1 == max(dt0, dt1)                      # max over ranks
    assert rate0 == rate1 == pytest.approx((n0 + n1) / max(dt0, dt1))
    assert h0 != h1                                         # independent scene streams per rank


def test_single_rank_defaults():
    from paper_2603_03935_b200 import parallel as par
    r = par.Rank(1, 0, 0, None)
    assert par.max_over_ranks(1.5, r) == 1.5
    assert par.weak_scaling_rate(10, 2.0, r) == 5.0
    assert par.stream_seed(100, 0) == 100 and par.stream_seed(100, 3) == 100 + 3 * par.SEED_STRIDE


@pytest.mark.timeout(300)
def test_reference_arm_under_torchrun_two_ranks():
    """`bench.py --impl reference` launched the way the driver launches N > 1 (torchrun, gloo on a
    CPU box): rank 0 alone times the oracle and prints ONE JSON line; rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "N"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=280)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["value"] > 0 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def _mix64(x):
    M = (1 << 64) - 1
    x ^= x >> 30
    x = (x * 0xbf58476d1ce4e5b9) & M
    x ^= x >> 27
    x = (x * 0x94d049bb133111eb) & M
    return x ^ (x >> 31)


def _shard_worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2603_03935_b200 import parallel as par
    from synth import Generator, disc_config_kwargs, frame_to_numpy
    from oracle.oracle import OracleMap
    r = par.setup("gloo")
    kw = par.sharded_map_kwargs(r)              # the NCCL unique-id bootstrap over the process group
    frames = par.own_frames(7, r)
    # the decomposition the sharded map computes, on the oracle's state: each rank counts the
    # overlaps of the next frame's detections with the map over the keys it OWNS; the all-reduced
    # (summed) partial counts must equal the unsharded |V_s ∩ V_j|
    g = Generator("N", H=60, W=80, Hp=4, Wp=5, fx=72.0, fy=72.0, cx=40.0, cy=30.0, Df=16, Dt=8)
    ckw = disc_config_kwargs(g.cfg)
    ckw["mask_min_area"] = 10
    om = OracleMap(**ckw)
    for f in range(4):
        om.integrate(frame_to_numpy(g.frame(f)))
    keys, ids = om.memberships()
    nxt = frame_to_numpy(g.frame(4))
    om2 = OracleMap(**ckw)
    for f in range(4):
        om2.integrate(frame_to_numpy(g.frame(f)))
    om2.integrate(nxt)
    lf = om2.last_frame()
    mem = {}
    for k, i in zip(keys.tolist(), ids.tolist()):
        mem.setdefault(k, []).append(i)
    part = torch.zeros(64, 256, dtype=torch.int64)
    for s, k in zip(lf["pair_s"].tolist(), lf["pair_key"].tolist()):
        if (_mix64(int(k)) >> 40) % r.world == r.rank:
            for j in mem.get(int(k), []):
                part[s, j] += 1
    dist.all_reduce(part)
    full = {(int(s), int(j)): int(c) for s, j, c in zip(lf["trip_s"], lf["trip_j"], lf["trip_c"])}
    got = {(s, j): int(part[s, j]) for s in range(64) for j in range(256) if part[s, j] > 0}
    q.put((r.rank, kw["world_size"], kw["rank"], bytes(kw["nccl_unique_id"]), frames, got == full, len(full)))
    par.teardown(r)


@pytest.mark.timeout(300)
def test_two_rank_sharded_bootstrap_and_count_decomposition_gloo():
    """world_size 2 over gloo: (1) the sharded map's bootstrap -- rank 0's disc_nccl_unique_id
    broadcast so both ranks hold the same 128-byte id, world_size 2 and their own rank; (2) the frame
    split f = r + G j; (3) the exchange's arithmetic: per-rank overlap counts over owned keys
    (owner = mix64(key) >> 40 mod G), all-reduced, equal the unsharded C triples of the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, k0, id0, f0, ok0, n0), (r1, w1, k1, id1, f1, ok1, n1) = out
    assert (r0, r1) == (0, 1) and (w0, w1) == (2, 2) and (k0, k1) == (0, 1)
    assert id0 == id1 and len(id0) == 128 and any(id0)
    assert f0 == [0, 2, 4, 6] and f1 == [1, 3, 5]
    assert ok0 and ok1 and n0 > 0
