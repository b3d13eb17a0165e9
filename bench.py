#!/usr/bin/env python
"""bench.py -- DISC per-frame mapping hot path on B200 (libdisc, sm_100a).

One STEP = one window of F frames (default 16) of the Replica-shaped stream (BASELINE.json
configs[1]: 680x1200, ~33 masks/frame, 2 cm voxels, ViT-L/14 1024-d tokens, 384-d tracking)
through disc_integrate_frames: every §8(a) row (mask pass + back-projection + dedup, D map,
D-weighted pooling + Q, tracking, lookup + overlap counts, association + union-find,
relabel/insert).  Each step integrates NEW frames of the trajectory into the growing map.

Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier +
cuda.synchronize, CUDA events on the map's stream; max over ranks.  Inputs per step
(~1.5 GB per 32-frame step) exceed L2 (126 MB), so no flush is needed.  Clocks sampled with nvidia-smi during
the timed region.  `e2e`: same metric through disc_integrate_frames_host with pinned HOST
inputs (H2D copies + report D2H inside the timed region).  `cpu_baseline`: the CPU oracle
(oracle/, single thread) on a bounded prefix of the same stream.

N > 1 (torchrun): every rank maps its own independent scene stream (weak scaling, no
data-path collective: independent problems); value = all frames / max time.

--impl reference: the reference arm is the CPU oracle (this tier has no reference code);
rank 0 runs it on the host cores, each step a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s of voxel association+refinement (device-timed) at 1/2/4/8 B200; % HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="R", choices=["R", "N", "H"])
    p.add_argument("--frames-per-step", type=int, default=32)   # = the map's window (32: +3 % over 16)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--oracle-seconds", type=float, default=12.0)
    p.add_argument("--no-m1", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


WORKLOAD = {
    "R": "replica-shaped stream (BASELINE configs[1]): 680x1200, ~33 masks/frame, 2 cm voxels, "
         "ViT-L/14 48x85x1024 fp32 tokens, 48x85x384 bf16 tracking tokens",
    "N": "scannet-shaped stream (BASELINE configs[2]): 480x640 noisy depth, ~21 masks/frame, 5 cm voxels",
    "H": "hm3d multi-story building (BASELINE configs[3]): 480x640, ~35 masks/frame, 2 cm voxels",
}

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML DURING the timed region
    (a polling thread every ~1 ms, plus one sample at entry and one at exit so even a
    millisecond-long region has readings); nvidia-smi's own polling is too coarse for it."""

    def __init__(self, dev: int):
        self.dev = dev
        self.rows = []
        self.h = None
        self.stop = threading.Event()
        self.t = None

    def _sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        try:
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((float(sm), float(mx), int(rs)))

    def _loop(self):
        while not self.stop.wait(0.001):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = self.dev
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis and vis.split(",")[0].strip().isdigit():
                idx = int(vis.split(",")[self.dev].strip())
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def __exit__(self, *a):
        if self.h is None:
            return
        try:
            self._sample()
        except Exception:
            pass
        self.stop.set()
        if self.t:
            self.t.join(timeout=1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        reasons = set()
        for _, _, r in self.rows:
            for bit, name in REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(reasons), "samples": len(self.rows)}


from paper_2603_03935_b200 import parallel as par  # noqa: E402


def setup_dist():
    r = par.setup()
    return r.world, r.rank, r.local, r


def barrier(ws):
    par.barrier(RANK)


def max_over_ranks(x: float, ws: int) -> float:
    return par.max_over_ranks(x, RANK)


RANK = par.Rank(1, 0, 0, None)


def frame_bytes(fr) -> int:
    n = 0
    for k in ["depth", "masks", "mask_conf", "patch_feats", "global_embed", "track_feats"]:
        t = fr.get(k)
        if t is not None:
            n += t.numel() * t.element_size()
    return n


def run_oracle_frames(frames_np, cfg_kw, budget_s, min_frames=1):
    """Time the CPU oracle (as it stands, 1 thread) on a prefix of the stream."""
    from oracle.oracle import OracleMap
    om = OracleMap(**cfg_kw)
    t0 = time.perf_counter()
    n = 0
    for fr in frames_np:
        om.integrate(fr)
        n += 1
        if n >= min_frames and time.perf_counter() - t0 >= budget_s:
            break
    return n, time.perf_counter() - t0


# --------------------------------------------------------------------------------------------
# reference arm (the CPU oracle)
# --------------------------------------------------------------------------------------------

def run_reference(args, ws, rank):
    if rank != 0:
        return
    import torch
    from synth import Generator, disc_config_kwargs, frame_to_numpy
    from oracle.oracle import OracleMap
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    g = Generator(args.config, device=dev)
    cfg_kw = disc_config_kwargs(g.cfg)
    per_step = 2 if args.config == "R" else 4
    frames = [frame_to_numpy(g.frame(f)) for f in range((args.warmup + args.steps) * per_step)]
    om = OracleMap(**cfg_kw)
    fi = 0
    for _ in range(args.warmup):
        for _ in range(per_step):
            om.integrate(frames[fi]); fi += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(per_step):
            om.integrate(frames[fi]); fi += 1
    dt = time.perf_counter() - t0
    n = args.steps * per_step
    value = n / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config], "frames_per_step": per_step,
                       "mode": "M2 (all §8(a) rows)", "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": 1, "kind": "oracle",
                             "sample": f"{n} frames ({per_step}/step) after {args.warmup * per_step} warm-up frames"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------

def path_bytes(stats0, stats1, in_bytes, cfg) -> float:
    """Algorithmic bytes of the whole path over a timed region (SURVEY §8(d) B_f):
    inputs read once + 16 B per membership probe (U) / insert / relabel item + instance
    state of touched instances (T reads for the gate, embeddings written)."""
    d = {k: stats1[k] - stats0[k] for k in ["pairs", "map_inserts", "relabels", "edges"]}
    b = in_bytes
    b += 16 * (d["pairs"] + d["map_inserts"] + d["relabels"])
    b += d["edges"] * cfg.Dt * 8
    return float(b)


def main():
    global RANK
    args = parse()
    ws, rank, local, RANK = setup_dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import numpy as np  # noqa: F401
    import torch
    from synth import Generator, disc_config_kwargs, frame_to_numpy
    from synth.scenes import seed_of
    from paper_2603_03935_b200 import DiscMap

    dev = torch.device("cuda", local)
    F = args.frames_per_step
    # independent scene per rank (weak scaling)
    g = Generator(args.config, seed=par.stream_seed(seed_of(args.config), rank), device=dev)
    c = g.cfg
    cfg_kw = disc_config_kwargs(c)
    nframes = (args.warmup + args.steps) * F
    t_gen = time.perf_counter()
    frames = [g.frame(f) for f in range(nframes)]
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    maxS = max(fr["masks"].shape[0] for fr in frames)
    caps = dict(max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=max(64, maxS), window=F,
                max_memberships=1 << 23, max_instances=1 << 17,
                # per-frame (mask, voxel) pair capacity: R and N frames stay below ~32k unique pairs
                # (e2e records the maximum seen), so 2^16 leaves a 2x margin; H's far
                # views reach ~1 pair per pixel (2 cm voxels, 480x640): 2^19.  A frame past it fails
                # loudly (CAPACITY)
                max_pairs_per_frame=int(os.environ.get("BENCH_PMAX", 1 << 19 if args.config == "H" else 1 << 16)),
                device=local)

    def run(frames_, timed_steps, warm_steps, m):
        for s in range(warm_steps):
            m.integrate_frames(frames_[s * F:(s + 1) * F])
        m.sync()
        st0 = m.stats()
        m.set_timing(True)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(ws)
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            e0.record(stream)
            for s in range(warm_steps, warm_steps + timed_steps):
                m.integrate_frames(frames_[s * F:(s + 1) * F])
            m.wait(stream)   # include the last window's stage 2
            e1.record(stream)
            torch.cuda.synchronize()
        barrier(ws)
        ms = e0.elapsed_time(e1)
        m.set_timing(False)
        st1 = m.stats()
        return ms, st0, st1, clk.summary()

    # ---- M2: the whole path (headline) ----
    m2 = DiscMap(**cfg_kw, **caps)
    ms, st0, st1, clocks = run(frames, args.steps, args.warmup, m2)
    ms_max = max_over_ranks(ms, ws)
    timed = frames[args.warmup * F:]
    value = ws * args.steps * F / (ms_max / 1e3)
    peak, peak_kind = peaks()
    # dominant kernel: K1 (mask pass + back-projection + dedup).  Algorithmic bytes per frame =
    # S*H*W mask bytes + 4*H*W depth bytes (every input byte read once).
    k1_bytes = sum(fr["masks"].numel() + fr["depth"].numel() * 4 for fr in timed)
    k1_ms = st1["k1_ms"] - st0["k1_ms"]
    k1_launches = st1["k1_launches"] - st0["k1_launches"]
    achieved = k1_bytes / (k1_ms / 1e3) / 1e9 if k1_ms > 0 else None
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "k1_dram_bytes_per_frame.json")
    if os.path.exists(tfile):
        try:
            with open(tfile) as f:
                traffic = json.load(f)["dram_bytes_per_frame"] * F
        except Exception:
            traffic = None
    in_bytes = sum(frame_bytes(fr) for fr in timed)
    pb = path_bytes(st0, st1, in_bytes, c)
    launches = st1["launches"] - st0["launches"]

    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "frames_per_step": F, "mode": "M2 (all §8(a) rows)",
                   "l2": f"no flush: inputs per step {in_bytes / args.steps / 1e9:.2f} GB > 126 MB L2",
                   "frames_timed_per_rank": args.steps * F, "masks_per_frame_mean":
                       round(sum(fr["masks"].shape[0] for fr in timed) / len(timed), 1),
                   "parallelism": f"{ws} independent maps (one scene stream per rank)" if ws > 1 else "1 GPU"},
        "roofline": {"bound": "hbm", "kernel": "K1 mask pass (k_masks + k_walk + k_dedup)", "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic, "algorithmic_bytes_per_launch": k1_bytes / max(k1_launches, 1),
                     "avg_launch_ms": k1_ms / max(k1_launches, 1), "launches": k1_launches,
                     "share_of_step": k1_ms / ms if ms > 0 else None},
        "path_roofline": {"bound": "hbm", "algorithmic_bytes_per_frame": pb / len(timed),
                          "achieved": pb / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                          "frac": pb / (ms / 1e3) / 1e9 / peak,
                          "stage1_ms": st1["stage1_ms"] - st0["stage1_ms"],
                          "stage2_ms": st1["stage2_ms"] - st0["stage2_ms"]},
        "clocks": clocks,
        "gpu_launches": launches,
        "counters": {k: st1[k] - st0[k] for k in ["pairs", "map_inserts", "relabels", "edges"]},
        "gen_seconds": round(t_gen, 1),
    }
    del m2

    # ---- M1: association + refinement only (no CLIP tokens) ----
    if not args.no_m1:
        frames_m1 = [dict(fr, patch_feats=None, global_embed=None) for fr in frames]
        m1 = DiscMap(**cfg_kw, **caps)
        ms1, a0, a1, _ = run(frames_m1, args.steps, args.warmup, m1)
        ms1 = max_over_ranks(ms1, ws)
        in1 = sum(frame_bytes(fr) for fr in frames_m1[args.warmup * F:])
        pb1 = path_bytes(a0, a1, in1, c)
        line["m1"] = {"value": ws * args.steps * F / (ms1 / 1e3), "unit": "frames/s", "ms_per_step": ms1 / args.steps,
                      "path_frac": pb1 / (ms1 / 1e3) / 1e9 / peak,
                      "k1_frac": (sum(fr["masks"].numel() + fr["depth"].numel() * 4 for fr in frames_m1[args.warmup * F:])
                                  / ((a1["k1_ms"] - a0["k1_ms"]) / 1e3) / 1e9 / peak)}
        del m1

    # ---- e2e: the public API with pinned HOST inputs, copies inside the timed region ----
    E = max(1, min(args.e2e_steps, args.steps))
    host = []
    for fr in frames[: (E + 1) * F]:
        host.append({k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in fr.items()})
    me = DiscMap(**cfg_kw, **caps)
    me.integrate_frames_host(host[:F], report=True)   # warm-up step
    h2d = sum(frame_bytes(fr) for fr in host[F:]) / E
    barrier(ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    max_u = 0
    for s in range(1, E + 1):
        reps = me.integrate_frames_host(host[s * F:(s + 1) * F], report=True)
        max_u = max([max_u] + [r["unique_pairs"] for r in reps])
    torch.cuda.synchronize()
    te = max_over_ranks(time.perf_counter() - t0, ws)
    from paper_2603_03935_b200.disc import disc_frame_report
    import ctypes
    line["e2e"] = {"value": ws * E * F / te, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": F * ctypes.sizeof(disc_frame_report), "steps": E,
                   "api": "disc_integrate_frames_host (pinned host buffers)", "max_unique_pairs_per_frame": int(max_u),
                   "max_pairs_per_frame": caps["max_pairs_per_frame"]}
    del me, host

    # ---- CPU baseline: the oracle as it stands, 1 thread, bounded prefix of the stream ----
    if rank == 0 and ws == 1 and not args.no_cpu:
        frames_np = (frame_to_numpy(fr) for fr in frames)
        n, dt = run_oracle_frames(frames_np, cfg_kw, args.oracle_seconds)
        line["cpu_baseline"] = {"value": n / dt, "unit": "frames/s", "cores": 1, "host_cores": os.cpu_count(),
                                "kind": "oracle",
                                "sample": f"first {n} frames of the same stream (full M2 path), {dt:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    par.teardown(RANK)


if __name__ == "__main__":
    main()
