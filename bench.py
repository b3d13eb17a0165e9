#!/usr/bin/env python
"""bench.py -- DISC per-frame mapping hot path on B200 (libdisc, sm_100a).

Workload (default --config H = BASELINE.json configs[3], the config the 1/2/4/8-GPU numbers are
quoted on): the HM3D-shaped multi-story building stream, 480x640, ~60 masks/frame (finer SAM-like
over-segmentation, mean 60 +- 20 %), 2 cm voxels, 34x45 ViT-L/14 tokens (1024-d CLIP, 384-d bf16
tracking).  Before timing, the map is PREFILLED (untimed, windows generated on the fly) by the first
frames of the tour until it holds >= 10^7 live (voxel, instance) memberships; every timed frame then
looks up, merges into and relabels a map of that size.

One STEP = one window of F = 32 NEW frames of the stream through disc_integrate_frames.
  value = M1 frames/s = "voxel association + refinement" (BASELINE.json metric; SURVEY §8(a) rows
          A0-A3, A5b, A6-A8: patch_feats = NULL), device-timed.
  m2    = the full path (+ A4 distinctiveness, A5 D-weighted pooling + Q) on the next frames.
Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier + cuda.synchronize,
CUDA events on the caller's stream (disc_wait orders it after the map's internal streams); max
over ranks.  Inputs per step (~0.65 GB M1 / ~0.85 GB M2) exceed the 126 MB L2: no flush needed.
Clocks sampled through NVML during the timed region.  `e2e`: M1 through the public host-input call
disc_integrate_frames_host (pinned host buffers: H2D inside the timed region, report D2H).
`cpu_baseline`: the CPU oracle (oracle/, 1 thread, as it stands) on a bounded prefix of the stream.

N > 1 (torchrun): ONE stream into ONE key-hash-sharded map: rank r is
shard r (owns the voxel keys with mix64(key) >> 40 mod N == r), runs stage 1 for the frames
f = r + N j, and libdisc exchanges over NCCL (detections all-gathered, (s, key) pairs routed to their
owners per window; overlap-count triples all-gathered, new-membership counts all-reduced per
frame).  A step is still 32 frames of the stream (32 / N per rank): strong scaling.  DISC_SHARDED=0
falls back to N independent maps (one scene stream per rank, weak scaling).

--impl reference: the reference arm is the CPU oracle (this tier has no reference code); rank 0
runs it on the host cores, each step a bounded sample (1 frame) of the same workload.
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
    p.add_argument("--config", default="H", choices=["R", "N", "H"])
    p.add_argument("--frames-per-step", type=int, default=32)   # = the map's window
    p.add_argument("--prefill-memberships", type=float, default=None,
                   help="untimed prefill until the map holds this many live memberships (H: 1e7, else 0)")
    p.add_argument("--prefill-max-frames", type=int, default=8192)
    p.add_argument("--e2e-steps", type=int, default=None,
                   help="windows timed end to end (default: --steps, as far as 4 GB of pinned inputs allow)")
    p.add_argument("--oracle-seconds", type=float, default=12.0)
    p.add_argument("--mask-format", default="bits", choices=["bits", "u8"],
                   help="mask planes as disc_frame::mask_bits (1 bit/pixel, default) or u8 byte planes")
    p.add_argument("--no-m2", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


WORKLOAD = {
    "R": "replica-shaped stream (BASELINE configs[1]): 680x1200, ~40 masks/frame, 2 cm voxels, "
         "ViT-L/14 48x85x1024 fp32 tokens, 48x85x384 bf16 tracking tokens",
    "N": "scannet-shaped stream (BASELINE configs[2]): 480x640 noisy depth, ~30 masks/frame, 5 cm voxels, "
         "34x45x1024 fp32 tokens, 34x45x384 bf16 tracking tokens",
    "H": "hm3d multi-story building (BASELINE configs[3]): 480x640, ~60 masks/frame, 2 cm voxels, "
         "34x45x1024 fp32 tokens, 34x45x384 bf16 tracking tokens, map prefilled to >= 1e7 live memberships",
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
    for k in ["depth", "masks", "mask_bits", "mask_conf", "patch_feats", "global_embed", "track_feats"]:
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


def nmasks(fr: dict) -> int:
    return (fr["masks"] if fr.get("masks") is not None else fr["mask_bits"]).shape[0]


def nmask_bytes(fr: dict) -> int:
    t = fr["masks"] if fr.get("masks") is not None else fr["mask_bits"]
    return t.numel() * t.element_size()


def m1(fr: dict) -> dict:
    """M1 input of a frame: no CLIP tokens (association + refinement only)."""
    return dict(fr, patch_feats=None, global_embed=None)


# --------------------------------------------------------------------------------------------
# reference arm (the CPU oracle)
# --------------------------------------------------------------------------------------------

def run_reference(args, ws, rank):
    if rank != 0:
        return
    import torch
    from synth import Generator, disc_config_kwargs, frame_to_numpy, pack_mask_bits
    from oracle.oracle import OracleMap
    dev = "cuda:0" if torch.cuda.is_available() else "cpu"
    g = Generator(args.config, device=dev)
    cfg_kw = disc_config_kwargs(g.cfg)
    per_step = 1 if args.config in ("R", "H") else 2
    frames = [frame_to_numpy(m1(g.frame(f, with_feats=False))) for f in range((args.warmup + args.steps) * per_step)]
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
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config], "frames_per_step": per_step,
                       "mode": "M1 (voxel association + refinement)", "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": 1, "kind": "oracle",
                             "sample": f"{n} frames ({per_step}/step) after {args.warmup * per_step} warm-up frames, "
                                       f"map starting empty (the oracle cannot prefill 1e7 memberships in minutes)"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------

def stage2_bytes(d: dict, Dt: int) -> float:
    """SURVEY §8(d) map bytes of stage 2 (A6-A8): 16 B per membership probe (U) / insert / relabel
    item + the gate's instance tracking rows (Dt fp64 per qualifying edge)."""
    return 16.0 * (d["pairs"] + d["map_inserts"] + d["relabels"]) + 8.0 * Dt * d["edges"]


def load_traffic(config: str, mode: str):
    """ncu dram bytes per frame of the kernels, captured on THIS config and mode (profiles/)."""
    f = os.path.join(ROOT, "profiles", f"traffic_{config}.json")
    try:
        with open(f) as fh:
            return json.load(fh)[mode]
    except Exception:
        return None


def main():
    global RANK
    args = parse()
    ws, rank, local, RANK = setup_dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    from synth import Generator, disc_config_kwargs, frame_to_numpy, pack_mask_bits
    from synth.scenes import seed_of
    from paper_2603_03935_b200 import DiscMap

    dev = torch.device("cuda", local)
    F = args.frames_per_step
    sharded = ws > 1 and os.environ.get("DISC_SHARDED", "1") != "0"
    Fr = F // ws if sharded else F   # frames per rank per step
    if sharded and F % ws:
        raise SystemExit(f"--frames-per-step {F} must be a multiple of --gpus {ws} for the sharded map")
    g = Generator(args.config, seed=seed_of(args.config) if sharded else par.stream_seed(seed_of(args.config), rank),
                  device=dev)
    c = g.cfg
    cfg_kw = disc_config_kwargs(c)
    prefill = args.prefill_memberships if args.prefill_memberships is not None else (1e7 if args.config == "H" else 0)
    caps = dict(max_pixels=c.H * c.W, max_patches=c.Hp * c.Wp, max_masks=int(c.n_masks * 1.2) + 8, window=F,
                max_memberships=1 << 25 if prefill > 0 else 1 << 23, max_instances=1 << 20,
                # per-frame (mask, voxel) pair capacity: R and N frames stay below ~40k unique pairs, H's far
                # views reach ~1 pair per pixel (2 cm voxels, 480x640): 2^19.  Past it: loud CAPACITY error
                max_pairs_per_frame=int(os.environ.get("BENCH_PMAX", 1 << 18 if args.config == "H" else 1 << 16)),
                device=local)
    m = DiscMap(**cfg_kw, **caps, **(par.sharded_map_kwargs(RANK) if sharded else {}))
    t_gen = 0.0
    nxt = 0   # next frame index of the stream

    def gen(n, feats):   # this rank's frames among the stream's next n
        nonlocal nxt, t_gen
        t0 = time.perf_counter()
        out = [g.frame(f, with_feats=feats) for f in range(nxt, nxt + n) if not sharded or f % ws == rank]
        if not feats:
            out = [m1(fr) for fr in out]
        if args.mask_format == "bits":   # the same masks, bit-packed (input layout; generated untimed)
            out = [{k: v for k, v in fr.items() if k != "masks"} | {"mask_bits": pack_mask_bits(fr["masks"])}
                   for fr in out]
        torch.cuda.synchronize()
        t_gen += time.perf_counter() - t0
        nxt += n
        return out

    # ---- prefill (untimed): the tour's first frames until the map holds `prefill` memberships ----
    live = 0
    t_pf = time.perf_counter()
    while live < prefill and nxt < args.prefill_max_frames:
        reps = m.integrate_frames(gen(F, False), report=True)
        live = reps[-1]["live_memberships"]
        if rank == 0 and (nxt // F) % 8 == 0:
            print(f"prefill: {nxt} frames, {live} live memberships, {reps[-1]['live_instances']} instances, "
                  f"{time.perf_counter() - t_pf:.0f} s", file=sys.stderr, flush=True)
    prefill_frames = nxt
    t_pf = time.perf_counter() - t_pf

    def run(frames_, timed_steps, warm_steps):
        for s in range(warm_steps):
            m.integrate_frames(frames_[s * Fr:(s + 1) * Fr])
        m.sync()
        st0 = m.stats()
        m.set_timing(True)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(ws)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("timed")
        with ClockSampler(local) as clk:
            e0.record(stream)
            for s in range(warm_steps, warm_steps + timed_steps):
                m.integrate_frames(frames_[s * Fr:(s + 1) * Fr])
            m.wait(stream)   # include the last window's stage 2
            e1.record(stream)
            torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        barrier(ws)
        ms = e0.elapsed_time(e1)
        m.set_timing(False)
        st1 = m.stats()
        return ms, {k: st1[k] - st0[k] for k in st1 if not isinstance(st1[k], list)}, clk.summary()

    peak, peak_kind = peaks()

    def measure(mode, feats):
        frames = gen((args.warmup + args.steps) * F, feats)
        ms, d, clocks = run(frames, args.steps, args.warmup)
        ms_max = max_over_ranks(ms, ws)
        timed = frames[args.warmup * Fr:]
        n = len(timed)
        in_bytes = sum(frame_bytes(fr) for fr in timed)
        k1_bytes = sum(nmask_bytes(fr) + fr["depth"].numel() * 4 for fr in timed)
        s2_bytes = stage2_bytes(d, c.Dt)
        k1_ms, s2_ms = d["k1_ms"], d["stage2_ms"]
        kern = {
            "K1": {"kernel": "K1 mask pass (k_masks + k_walk + k_dedup)", "bound": "hbm",
                   "algorithmic_bytes_per_launch": k1_bytes / max(d["k1_launches"], 1),
                   "bytes_per_unit": ("S*ceil(H*W/32)*4 bit-packed mask bytes" if args.mask_format == "bits" else
                                      "S*H*W mask bytes") + " + 4*H*W depth bytes per frame (every input byte once)",
                   "avg_launch_ms": k1_ms / max(d["k1_launches"], 1), "launches": d["k1_launches"],
                   "achieved": k1_bytes / (k1_ms / 1e3) / 1e9 if k1_ms > 0 else None,
                   "share_of_step": k1_ms / ms if ms > 0 else None},
            "stage2": {"kernel": "k_stage2 (A6 lookup + overlap counts, A7 association, A8 map update)", "bound": "hbm",
                       "algorithmic_bytes_per_launch": s2_bytes / max(args.steps, 1),
                       "bytes_per_unit": "16 B per (s,key) probe / insert / relabel item + 8*Dt B per edge (SURVEY §8(d))",
                       "avg_launch_ms": s2_ms / max(args.steps, 1), "launches": args.steps,
                       "achieved": s2_bytes / (s2_ms / 1e3) / 1e9 if s2_ms > 0 else None,
                       "share_of_step": s2_ms / ms if ms > 0 else None},
        }
        tr = load_traffic(args.config, mode) or {}
        for k, v in kern.items():
            v["peak"], v["unit"] = peak, "GB/s"
            v["frac"] = v["achieved"] / peak if v["achieved"] else None
            t = tr.get(k)
            v["traffic"] = t * n / v["launches"] if t is not None and v["launches"] else None
        dom = max(kern, key=lambda k: kern[k]["share_of_step"] or 0.0)
        pb = in_bytes + s2_bytes
        return {"value": (1 if sharded else ws) * args.steps * F / (ms_max / 1e3), "ms": ms_max, "clocks": clocks, "kernels": kern,
                "dominant": dom, "frames": timed, "d": d,
                "path": {"bound": "hbm", "algorithmic_bytes_per_frame": pb / n, "achieved": pb / (ms / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": pb / (ms / 1e3) / 1e9 / peak,
                         "stage1_ms": d["stage1_ms"], "stage2_ms": s2_ms}}

    r1 = measure("M1", False)
    dom = r1["kernels"][r1["dominant"]]
    timed = r1["frames"]
    line = {
        "metric": METRIC, "value": r1["value"], "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r1["ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "frames_per_step": F,
                   "mode": "M1 = voxel association + refinement (A0-A3, A5b, A6-A8; no CLIP tokens)",
                   "l2": f"no flush: inputs per step {sum(frame_bytes(fr) for fr in timed) / args.steps / 1e9:.2f} GB > 126 MB L2",
                   "frames_timed_per_rank": args.steps * Fr,
                   "masks_per_frame_mean": round(sum(nmasks(fr) for fr in timed) / len(timed), 1),
                   "mask_format": ("bit-packed planes (disc_frame::mask_bits, 1 bit per pixel)" if args.mask_format == "bits"
                                   else "u8 byte planes"),
                   "prefill_frames": prefill_frames, "prefill_seconds": round(t_pf, 1),
                   "live_memberships_before_timing": int(live),
                   "parallelism": (f"one stream, key-hash-sharded map over {ws} GPUs (NCCL)" if sharded else
                                   f"{ws} independent maps (one scene stream per rank)") if ws > 1 else "1 GPU"},
        "roofline": {"bound": dom["bound"], "kernel": dom["kernel"], "achieved": dom["achieved"], "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": dom["frac"], "traffic": dom["traffic"],
                     "algorithmic_bytes_per_launch": dom["algorithmic_bytes_per_launch"],
                     "bytes_per_unit": dom["bytes_per_unit"], "avg_launch_ms": dom["avg_launch_ms"],
                     "launches": dom["launches"], "share_of_step": dom["share_of_step"]},
        "roofline_kernels": r1["kernels"],
        "path_roofline": r1["path"],
        "clocks": r1["clocks"],
        "gpu_launches": r1["d"]["launches"],
        "counters": {k: r1["d"][k] for k in ["pairs", "map_inserts", "relabels", "edges"]},
    }
    del r1, timed

    # ---- M2: the whole path (CLIP distinctiveness + pooling + Q as well), next frames ----
    if not args.no_m2:
        r2 = measure("M2", True)
        line["m2"] = {"value": r2["value"], "unit": "frames/s", "ms_per_step": r2["ms"] / args.steps,
                      "mode": "M2 = all §8(a) rows", "path_roofline": r2["path"], "roofline_kernels": r2["kernels"],
                      "dominant": r2["dominant"], "clocks": r2["clocks"], "gpu_launches": r2["d"]["launches"]}
        del r2

    # ---- e2e: the public API with pinned HOST inputs (M1), copies inside the timed region ----
    if not args.no_e2e:
        probe = gen(F, False)   # one window: its bytes bound how many windows fit in 4 GB pinned
        wbytes = sum(frame_bytes(fr) for fr in probe)
        E = args.e2e_steps if args.e2e_steps is not None else args.steps
        E = max(1, min(E, args.steps, int(4e9 // max(wbytes, 1)) - 1))
        host = [{k: (v.cpu().pin_memory() if isinstance(v, torch.Tensor) else v) for k, v in fr.items()}
                for fr in probe + gen(E * F, False)]
        del probe
        m.integrate_frames_host(host[:Fr], report=True)   # warm-up step
        h2d = sum(frame_bytes(fr) for fr in host[Fr:]) / E
        barrier(ws)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # the E steps in one call: libdisc pipelines them over two staging buffers (step w+1's H2D
        # overlaps step w's kernels) and reads every step's reports back before returning
        reps = m.integrate_frames_host(host[Fr:(E + 1) * Fr], report=True)
        max_u = max(r["unique_pairs"] for r in reps)
        torch.cuda.synchronize()
        te = max_over_ranks(time.perf_counter() - t0, ws)
        from paper_2603_03935_b200.disc import disc_frame_report
        import ctypes
        line["e2e"] = {"value": (1 if sharded else ws) * E * F / te, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                       "d2h_bytes_per_step": Fr * ctypes.sizeof(disc_frame_report), "steps": E, "mode": "M1",
                       "api": "disc_integrate_frames_host (pinned host buffers; E steps per call, "
                              "H2D of step w+1 overlapping step w's kernels, all reports read back)",
                       "max_unique_pairs_per_frame": int(max_u), "max_pairs_per_frame": caps["max_pairs_per_frame"],
                       "live_memberships_after": int(reps[-1]["live_memberships"])}
        del host
    line["gen_seconds"] = round(t_gen, 1)

    # ---- CPU baseline: the oracle as it stands, 1 thread, bounded prefix of the stream (M1) ----
    if rank == 0 and ws == 1 and not args.no_cpu:
        g0 = Generator(args.config, seed=par.stream_seed(seed_of(args.config), rank), device=dev)
        frames_np = (frame_to_numpy(m1(g0.frame(f, with_feats=False))) for f in range(10 ** 6))
        n, dt = run_oracle_frames(frames_np, cfg_kw, args.oracle_seconds)
        line["cpu_baseline"] = {"value": n / dt, "unit": "frames/s", "cores": 1, "host_cores": os.cpu_count(),
                                "kind": "oracle",
                                "sample": f"first {n} frames of the same stream (M1 path), map starting empty, {dt:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    par.teardown(RANK)


if __name__ == "__main__":
    main()
