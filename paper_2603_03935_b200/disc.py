"""ctypes binding of libdisc (include/disc.h).  Argument marshalling only: every step of the
DISC hot path runs in libdisc's sm_100a kernels.  There is no CPU fallback: if libdisc.so
is missing or cannot load, every entry point raises.

Device inputs are torch CUDA tensors (PyTorch provides device memory and streams); the pose
is a host 4x4 float32 array.  Names follow include/disc.h.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DISC_LIB_VARIANT: path of an alternative in-tree libdisc build (kernel-tuning experiments)
LIB_PATH = os.environ.get("DISC_LIB_VARIANT") or os.path.join(_HERE, "libdisc.so")

DISC_OK, DISC_ERR_INVALID, DISC_ERR_INTERNAL, DISC_ERR_CAPACITY, DISC_ERR_CUDA = 0, 2, 4, 5, 6
STATUS_NAMES = {0: "kept", 1: "area", 2: "conf", 3: "aspect", 4: "nodepth", 5: "nofeat"}


class DiscError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libdisc error {code}: {msg}")
        self.code = code


class disc_config(C.Structure):
    _fields_ = [
        ("voxel_size", C.c_float), ("tau_geo", C.c_float), ("tau_vis", C.c_float),
        ("depth_min", C.c_float), ("depth_max", C.c_float), ("mask_min_conf", C.c_float),
        ("mask_max_aspect", C.c_float), ("mask_min_area", C.c_int32), ("cover_min", C.c_float),
        ("lambda_size", C.c_float), ("eps_distinct", C.c_float), ("dbscan_eps", C.c_float),
        ("dbscan_min_pts", C.c_int32), ("refine_active", C.c_int32), ("feat_dim", C.c_int32),
        ("track_dim", C.c_int32), ("max_memberships", C.c_int64), ("max_instances", C.c_int32),
        ("max_masks", C.c_int32), ("max_pixels", C.c_int32), ("max_patches", C.c_int32),
        ("max_pairs_per_frame", C.c_int32), ("window", C.c_int32), ("device", C.c_int32),
        ("world_size", C.c_int32), ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p),
    ]


class disc_frame(C.Structure):
    _fields_ = [
        ("frame_id", C.c_int64), ("height", C.c_int32), ("width", C.c_int32),
        ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
        ("pose", C.c_float * 16), ("depth", C.c_void_p), ("num_masks", C.c_int32),
        ("masks", C.c_void_p), ("mask_conf", C.c_void_p), ("patch_h", C.c_int32),
        ("patch_w", C.c_int32), ("patch_feats", C.c_void_p), ("global_embed", C.c_void_p),
        ("track_feats", C.c_void_p), ("mask_bits", C.c_void_p),
    ]


REPORT_FIELDS = [
    ("kept", C.c_int32), ("drop_area", C.c_int32), ("drop_conf", C.c_int32),
    ("drop_aspect", C.c_int32), ("drop_nodepth", C.c_int32), ("drop_nofeat", C.c_int32),
    ("key_out_of_range", C.c_int64), ("unique_pairs", C.c_int64), ("edges", C.c_int64),
    ("created", C.c_int64), ("merged_away", C.c_int64), ("new_memberships", C.c_int64),
    ("relabeled", C.c_int64), ("live_instances", C.c_int64), ("live_memberships", C.c_int64),
    ("refine_rounds", C.c_int64), ("refine_merged", C.c_int64),
]


class disc_frame_report(C.Structure):
    _fields_ = REPORT_FIELDS

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in REPORT_FIELDS}


class disc_instance(C.Structure):
    _fields_ = [("id", C.c_int64), ("voxel_count", C.c_int64), ("last_seen", C.c_int64),
                ("obs_count", C.c_int32), ("q", C.c_float), ("aabb_min", C.c_int32 * 3),
                ("aabb_max", C.c_int32 * 3)]


class disc_frame_debug(C.Structure):
    _fields_ = [
        ("num_masks", C.c_int32), ("status", C.c_void_p), ("area", C.c_void_p), ("bbox", C.c_void_p),
        ("vs", C.c_void_p), ("target", C.c_void_p), ("factors", C.c_void_p), ("embed", C.c_void_p),
        ("track", C.c_void_p), ("pair_cap", C.c_int64), ("pair_s", C.c_void_p),
        ("pair_key", C.c_void_p), ("n_pairs", C.c_int64), ("trip_cap", C.c_int64),
        ("trip_s", C.c_void_p), ("trip_j", C.c_void_p), ("trip_c", C.c_void_p),
        ("trip_edge", C.c_void_p), ("n_trip", C.c_int64),
    ]


class disc_stats(C.Structure):
    _fields_ = [("frames", C.c_int64), ("k1_ms", C.c_double), ("k1_launches", C.c_int64),
                ("stage1_ms", C.c_double), ("stage2_ms", C.c_double), ("mask_bytes", C.c_int64),
                ("depth_bytes", C.c_int64), ("track_bytes", C.c_int64), ("feat_bytes", C.c_int64),
                ("pairs", C.c_int64), ("map_inserts", C.c_int64), ("relabels", C.c_int64),
                ("edges", C.c_int64), ("launches", C.c_int64), ("shard_memberships", C.c_int64 * 16)]


class disc_final_report(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ["rounds", "edges", "merged_away", "relabeled", "removed", "live_instances",
                                          "live_memberships"]]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


EXPORTS = {
    "disc_config_init": (C.c_int, [C.c_void_p]),
    "disc_map_create": (C.c_int, [C.c_void_p, C.c_void_p]),
    "disc_map_destroy": (None, [C.c_void_p]),
    "disc_integrate_frame": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "disc_integrate_frames": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "disc_integrate_frames_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "disc_query": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "disc_get_instances": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "disc_get_memberships": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "disc_debug_last_frame": (C.c_int, [C.c_void_p, C.c_void_p]),
    "disc_set_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "disc_finalize": (C.c_int, [C.c_void_p, C.c_float, C.c_float, C.c_int64, C.c_void_p]),
    "disc_classify": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_int64, C.c_void_p]),
    "disc_dense_transfer": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_float, C.c_void_p]),
    "disc_get_stats": (C.c_int, [C.c_void_p, C.c_void_p]),
    "disc_wait": (C.c_int, [C.c_void_p, C.c_void_p]),
    "disc_sync": (C.c_int, [C.c_void_p]),
    "disc_last_error": (C.c_char_p, [C.c_void_p]),
    "disc_version": (C.c_char_p, []),
    "disc_nccl_unique_id": (C.c_int, [C.c_void_p]),
}

_lib = None


def lib():
    """Load libdisc.so (in-tree).  Raises if it is missing: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def default_config(**kw) -> disc_config:
    c = disc_config()
    lib().disc_config_init(C.byref(c))
    for k, v in kw.items():
        if not hasattr(c, k):
            raise KeyError(k)
        setattr(c, k, v)
    return c


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (disc_nccl_unique_id), for disc_config.nccl_unique_id."""
    buf = (C.c_uint8 * 128)()
    rc = lib().disc_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc != DISC_OK:
        raise DiscError(rc, "disc_nccl_unique_id failed (libnccl.so.2 missing?)")
    return bytes(buf)


class DiscMap:
    """A GPU-resident DISC map (libdisc).  Single writer per map."""

    def __init__(self, **cfg):
        """cfg: disc_config fields.  world_size = G > 1 makes a key-hash-sharded map:
        with nccl_unique_id = None all G shards live in this process (one device); with the 128-byte
        id of nccl_unique_id() (rank 0's, broadcast) this process is shard `rank` of G (NCCL)."""
        import torch
        uid = cfg.pop("nccl_unique_id", None)
        self._uid = None
        if uid is not None:
            self._uid = (C.c_uint8 * 128)(*bytes(uid))
            cfg["nccl_unique_id"] = C.cast(self._uid, C.c_void_p)
        self.cfg = default_config(**cfg)
        h = C.c_void_p()
        rc = lib().disc_map_create(C.byref(self.cfg), C.byref(h))
        if rc != DISC_OK:
            raise DiscError(rc, "disc_map_create failed")
        self.h = h
        self.Df = self.cfg.feat_dim
        self.Dt = self.cfg.track_dim
        self.device = torch.device("cuda", self.cfg.device)
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            lib().disc_map_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != DISC_OK:
            raise DiscError(rc, lib().disc_last_error(self.h).decode())

    # ---- marshalling ------------------------------------------------------------------
    @staticmethod
    def make_frame(fr: dict, keep: list) -> disc_frame:
        """fr: dict with torch CUDA tensors (depth, masks [S,H,W] u8 -- or mask_bits [S, ceil(H*W/32)]
        int32, the bit-packed planes of disc_frame::mask_bits --, mask_conf, patch_feats, global_embed,
        track_feats [bf16]) and host scalars / pose."""
        import torch
        tf = fr.get("track_feats")
        if tf is not None and tf.dtype == torch.bfloat16:
            tf = tf.view(torch.int16)
        mk, mb = fr.get("masks"), fr.get("mask_bits")
        ts = [fr["depth"], mk, mb, fr.get("mask_conf"), fr.get("patch_feats"), fr.get("global_embed"), tf]
        for t in ts:
            if t is not None and not t.is_contiguous():
                raise ValueError("inputs must be contiguous")
        keep.extend(t for t in ts if t is not None)
        H, W = fr["depth"].shape
        pose = (C.c_float * 16)(*[float(x) for x in np.asarray(fr["pose"], np.float32).reshape(16)])
        return disc_frame(frame_id=int(fr["frame_id"]), height=H, width=W, fx=fr["fx"], fy=fr["fy"],
                          cx=fr["cx"], cy=fr["cy"], pose=pose, depth=_ptr(fr["depth"]),
                          num_masks=int(fr["num_masks"] if "num_masks" in fr else
                                        (mk if mk is not None else mb).shape[0]), masks=_ptr(mk),
                          mask_bits=_ptr(mb),
                          mask_conf=_ptr(fr.get("mask_conf")), patch_h=int(fr["patch_h"]),
                          patch_w=int(fr["patch_w"]), patch_feats=_ptr(fr.get("patch_feats")),
                          global_embed=_ptr(fr.get("global_embed")), track_feats=_ptr(tf))

    @staticmethod
    def _stream(stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    # ---- hot path ---------------------------------------------------------------------
    def integrate_frame(self, fr: dict, stream=None, report: bool = True):
        keep = []
        f = self.make_frame(fr, keep)
        rep = disc_frame_report()
        rc = lib().disc_integrate_frame(self.h, C.byref(f), self._stream(stream),
                                        C.byref(rep) if report else None)
        self._check(rc)
        return rep.as_dict() if report else None

    def integrate_frames(self, frames: list, stream=None, report: bool = False):
        keep = []
        arr = (disc_frame * len(frames))(*[self.make_frame(fr, keep) for fr in frames])
        reps = (disc_frame_report * len(frames))() if report else None
        rc = lib().disc_integrate_frames(self.h, arr, len(frames), self._stream(stream), reps)
        self._check(rc)
        return [r.as_dict() for r in reps] if report else None

    def integrate_frames_host(self, frames: list, stream=None, report: bool = True):
        """frames hold HOST tensors (pinned for full speed); the library copies them."""
        keep = []
        arr = (disc_frame * len(frames))(*[self.make_frame(fr, keep) for fr in frames])
        reps = (disc_frame_report * len(frames))() if report else None
        rc = lib().disc_integrate_frames_host(self.h, arr, len(frames), self._stream(stream), reps)
        self._check(rc)
        return [r.as_dict() for r in reps] if report else None

    # ---- readers ----------------------------------------------------------------------
    def query(self, q, k: int):
        q = np.ascontiguousarray(q, np.float32)
        ids = np.zeros(max(k, 1), np.int64)
        sc = np.zeros(max(k, 1), np.float32)
        n = C.c_int32()
        self._check(lib().disc_query(self.h, q.ctypes.data_as(C.c_void_p), k, ids.ctypes.data_as(C.c_void_p),
                                     sc.ctypes.data_as(C.c_void_p), C.byref(n)))
        return ids[: n.value], sc[: n.value]

    def instances(self, embeds=True, track=True) -> dict:
        n = C.c_int32()
        self._check(lib().disc_get_instances(self.h, None, None, None, 0, C.byref(n)))
        cnt = n.value
        arr = (disc_instance * max(cnt, 1))()
        E = np.zeros((cnt, self.Df), np.float32) if embeds else None
        T = np.zeros((cnt, max(self.Dt, 0)), np.float64) if (track and self.Dt > 0) else None
        self._check(lib().disc_get_instances(
            self.h, arr, None if E is None else E.ctypes.data_as(C.c_void_p),
            None if T is None else T.ctypes.data_as(C.c_void_p), cnt, C.byref(n)))
        out = dict(id=np.array([arr[i].id for i in range(cnt)], np.int64),
                   vcount=np.array([arr[i].voxel_count for i in range(cnt)], np.int64),
                   obs=np.array([arr[i].obs_count for i in range(cnt)], np.int32),
                   last_seen=np.array([arr[i].last_seen for i in range(cnt)], np.int64),
                   q=np.array([arr[i].q for i in range(cnt)], np.float32),
                   aabb=np.array([list(arr[i].aabb_min) + list(arr[i].aabb_max) for i in range(cnt)],
                                 np.int32).reshape(cnt, 6))
        if E is not None:
            out["e"] = E
        if T is not None:
            out["T"] = T
        return out

    def memberships(self):
        n = C.c_int64()
        self._check(lib().disc_get_memberships(self.h, None, None, 0, C.byref(n)))
        keys = np.zeros(max(n.value, 1), np.uint64)
        ids = np.zeros(max(n.value, 1), np.int64)
        self._check(lib().disc_get_memberships(self.h, keys.ctypes.data_as(C.c_void_p),
                                               ids.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
        keys, ids = keys[: n.value], ids[: n.value]
        o = np.lexsort((ids, keys))
        return keys[o], ids[o]

    def last_frame(self, pair_cap: int = 1 << 22, trip_cap: int = 1 << 17) -> dict:
        d = disc_frame_debug()
        self._check(lib().disc_debug_last_frame(self.h, C.byref(d)))
        S = d.num_masks
        out = dict(status=np.zeros(S, np.int32), area=np.zeros(S, np.int64), bbox=np.zeros((S, 4), np.int32),
                   vs=np.zeros(S, np.int64), target=np.zeros(S, np.int64), factors=np.zeros((S, 6), np.float32),
                   e=np.zeros((S, self.Df), np.float32), t=np.zeros((S, max(self.Dt, 0)), np.float64))
        ps = np.zeros(pair_cap, np.int32)
        pk = np.zeros(pair_cap, np.uint64)
        ts = np.zeros(trip_cap, np.int32)
        tj = np.zeros(trip_cap, np.int64)
        tc = np.zeros(trip_cap, np.int64)
        te = np.zeros(trip_cap, np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        d.status, d.area, d.bbox, d.vs, d.target = p(out["status"]), p(out["area"]), p(out["bbox"]), p(out["vs"]), p(out["target"])
        d.factors, d.embed = p(out["factors"]), p(out["e"])
        d.track = p(out["t"]) if self.Dt > 0 else None
        d.pair_cap, d.pair_s, d.pair_key = pair_cap, p(ps), p(pk)
        d.trip_cap, d.trip_s, d.trip_j, d.trip_c, d.trip_edge = trip_cap, p(ts), p(tj), p(tc), p(te)
        self._check(lib().disc_debug_last_frame(self.h, C.byref(d)))
        n, nt = d.n_pairs, d.n_trip
        o = np.lexsort((pk[:n], ps[:n]))
        out.update(pair_s=ps[:n][o], pair_key=pk[:n][o])
        o = np.lexsort((tj[:nt], ts[:nt]))
        out.update(trip_s=ts[:nt][o], trip_j=tj[:nt][o], trip_c=tc[:nt][o], trip_edge=te[:nt][o])
        return out

    def classify(self, table, k: int):
        """Top-k classes (rows of table [C][Df]) of every live instance with an embedding (disc_classify)."""
        table = np.ascontiguousarray(table, np.float32)
        C_ = table.shape[0]
        n = C.c_int64()
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._check(lib().disc_classify(self.h, p(table), C_, k, None, None, None, 0, C.byref(n)))
        kk = min(k, C_)
        ids = np.zeros(max(n.value, 1), np.int64)
        cls = np.zeros((max(n.value, 1), kk), np.int32)
        sc = np.zeros((max(n.value, 1), kk), np.float32)
        self._check(lib().disc_classify(self.h, p(table), C_, k, p(ids), p(cls), p(sc), n.value, C.byref(n)))
        return ids[: n.value], cls[: n.value], sc[: n.value]

    def dense_transfer(self, points, d_assign: float):
        """Nearest-voxel-centre instance per point, -1 = unassigned (disc_dense_transfer)."""
        pts = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
        out = np.zeros(max(pts.shape[0], 1), np.int64)
        self._check(lib().disc_dense_transfer(self.h, pts.ctypes.data_as(C.c_void_p), pts.shape[0], d_assign,
                                              out.ctypes.data_as(C.c_void_p)))
        return out[: pts.shape[0]]

    def finalize(self, tau_geo=None, tau_vis=None, min_voxels: int = 0) -> dict:
        """End-of-trajectory orphan merge + minimum-size filter (disc_finalize)."""
        rep = disc_final_report()
        tg = self.cfg.tau_geo if tau_geo is None else tau_geo
        tv = self.cfg.tau_vis if tau_vis is None else tau_vis
        self._check(lib().disc_finalize(self.h, tg, tv, int(min_voxels), C.byref(rep)))
        return rep.as_dict()

    def set_timing(self, on: bool):
        self._check(lib().disc_set_timing(self.h, 1 if on else 0))

    def stats(self) -> dict:
        s = disc_stats()
        self._check(lib().disc_get_stats(self.h, C.byref(s)))
        out = {k: getattr(s, k) for k, _ in disc_stats._fields_}
        out["shard_memberships"] = list(out["shard_memberships"])
        return out

    def sync(self):
        self._check(lib().disc_sync(self.h))

    def wait(self, stream=None):
        """Order `stream` (default: torch's current stream) after all queued map work."""
        self._check(lib().disc_wait(self.h, self._stream(stream)))
