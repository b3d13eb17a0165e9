"""ctypes wrapper of the CPU oracle (oracle/libdisc_oracle.so).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs; never by the product package
``paper_2603_03935_b200``.  The oracle itself is oracle/disc_oracle.cpp (definitional, fp64
semantics, pinned fp32 keys); this file only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DISC_ORACLE_LIB: an alternative build of the same source (the ASan/UBSan build, tools/sanitize_oracle.sh)
_LIB_PATH = os.environ.get("DISC_ORACLE_LIB") or os.path.join(_HERE, "libdisc_oracle.so")

KEPT, DROP_AREA, DROP_CONF, DROP_ASPECT, DROP_NODEPTH, DROP_NOFEAT = range(6)


class OraConfig(C.Structure):
    _fields_ = [
        ("voxel_size", C.c_float), ("tau_geo", C.c_float), ("tau_vis", C.c_float),
        ("depth_min", C.c_float), ("depth_max", C.c_float),
        ("mask_min_conf", C.c_float), ("mask_max_aspect", C.c_float), ("mask_min_area", C.c_int32),
        ("cover_min", C.c_float), ("lambda_size", C.c_float), ("eps_distinct", C.c_float),
        ("dbscan_eps", C.c_float), ("dbscan_min_pts", C.c_int32), ("refine_active", C.c_int32),
        ("feat_dim", C.c_int32), ("track_dim", C.c_int32),
    ]


class OraFrame(C.Structure):
    _fields_ = [
        ("frame_id", C.c_int64), ("height", C.c_int32), ("width", C.c_int32),
        ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
        ("pose", C.c_float * 16),
        ("depth", C.c_void_p), ("num_masks", C.c_int32), ("masks", C.c_void_p),
        ("mask_conf", C.c_void_p), ("patch_h", C.c_int32), ("patch_w", C.c_int32),
        ("patch_feats", C.c_void_p), ("global_embed", C.c_void_p), ("track_feats", C.c_void_p),
    ]


REPORT_FIELDS = [
    ("kept", C.c_int32), ("drop_area", C.c_int32), ("drop_conf", C.c_int32),
    ("drop_aspect", C.c_int32), ("drop_nodepth", C.c_int32), ("drop_nofeat", C.c_int32),
    ("key_out_of_range", C.c_int64), ("unique_pairs", C.c_int64), ("edges", C.c_int64),
    ("created", C.c_int64), ("merged_away", C.c_int64), ("new_memberships", C.c_int64),
    ("relabeled", C.c_int64), ("live_instances", C.c_int64), ("live_memberships", C.c_int64),
    ("refine_rounds", C.c_int64), ("refine_merged", C.c_int64),
]


class OraReport(C.Structure):
    _fields_ = REPORT_FIELDS

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in REPORT_FIELDS}


class OraFinalReport(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ["rounds", "edges", "merged_away", "relabeled", "removed", "live_instances",
                                          "live_memberships"]]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.environ.get("DISC_ORACLE_LIB") and (not os.path.exists(_LIB_PATH) or os.path.getmtime(
                _LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "disc_oracle.cpp"))):
            build()
        L = C.CDLL(_LIB_PATH)
        P, I32, I64, U64, D, F = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float
        sig = {
            "ora_create": (P, [P]), "ora_destroy": (None, [P]), "ora_set_selfcheck": (None, [P, I32]),
            "ora_integrate": (I32, [P, P, P]), "ora_last_error": (C.c_char_p, [P]),
            "ora_num_instances": (I64, [P]),
            "ora_get_instances": (I64, [P, P, P, P, P, P, P, P, P, I64]),
            "ora_num_memberships": (I64, [P]), "ora_get_memberships": (I64, [P, P, P, I64]),
            "ora_get_accept": (I64, [P, I64, P, P, I64]), "ora_next_id": (I64, [P]),
            "ora_last_num_masks": (I32, [P]), "ora_last_masks": (None, [P, P, P, P, P, P]),
            "ora_last_pairs": (I64, [P, P, P, I64]), "ora_last_triples": (I64, [P, P, P, P, P, I64]),
            "ora_last_quality": (None, [P, P, P, P, P]),
            "ora_pixel_world": (I32, [P, P, I32, I32, P]), "ora_point_key": (I32, [P, F, P]),
            "ora_pack_key": (U64, [I32, I32, I32]), "ora_pose_rigid": (I32, [P]),
            "ora_distinctiveness": (None, [I64, I32, P, D, P]),
            "ora_pool": (I32, [I64, I32, P, P, P, P, D, P, P]),
            "ora_s_size": (D, [I64, I32, I32, D]), "ora_s_angle": (D, [I64, P, P]),
            "ora_s_sem": (D, [I32, P, P]), "ora_s_dist": (D, [D]), "ora_quality": (D, [D, D, D, D]),
            "ora_dot_pin": (D, [I32, P, P]), "ora_query": (I64, [P, P, I32, P, P]),
            "ora_finalize": (I32, [P, F, F, I64, P]),
            "ora_classify": (I64, [P, P, I32, I32, P, P, P, I64]),
            "ora_dense_transfer": (None, [P, P, I64, F, P]),
            "ora_dbscan": (I32, [I64, P, F, I32, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


DEFAULTS = dict(voxel_size=0.05, tau_geo=0.3, tau_vis=0.8, depth_min=0.1, depth_max=10.0,
                mask_min_conf=0.5, mask_max_aspect=10.0, mask_min_area=400, cover_min=0.25,
                lambda_size=3.3, eps_distinct=1e-6, dbscan_eps=0.0, dbscan_min_pts=8, refine_active=0, feat_dim=64, track_dim=0)


def make_config(**kw) -> OraConfig:
    d = dict(DEFAULTS)
    d.update({k: v for k, v in kw.items() if k in DEFAULTS})
    return OraConfig(**d)


def make_frame(fr: dict, keep: list) -> OraFrame:
    """fr: dict of numpy arrays / scalars (see synth.frames).  `keep` holds references."""
    depth = _c(fr["depth"], np.float32)
    masks = _c(fr["masks"], np.uint8)
    conf = _c(fr.get("mask_conf"), np.float32)
    pf = _c(fr.get("patch_feats"), np.float32)
    ge = _c(fr.get("global_embed"), np.float32)
    tf = _c(fr.get("track_feats"), np.uint16)
    keep += [depth, masks, conf, pf, ge, tf]
    H, W = depth.shape
    S = masks.shape[0]
    pose = (C.c_float * 16)(*[float(x) for x in np.asarray(fr["pose"], np.float32).reshape(16)])
    return OraFrame(frame_id=int(fr["frame_id"]), height=H, width=W, fx=fr["fx"], fy=fr["fy"],
                    cx=fr["cx"], cy=fr["cy"], pose=pose, depth=_p(depth), num_masks=S,
                    masks=_p(masks), mask_conf=_p(conf), patch_h=int(fr["patch_h"]),
                    patch_w=int(fr["patch_w"]), patch_feats=_p(pf), global_embed=_p(ge),
                    track_feats=_p(tf))


class OracleMap:
    """Definitional CPU map (C.1/C.2).  Thin marshalling over libdisc_oracle.so."""

    def __init__(self, selfcheck: bool = False, **cfg):
        self.cfg = make_config(**cfg)
        self.Df = self.cfg.feat_dim
        self.Dt = self.cfg.track_dim
        self.h = lib().ora_create(C.byref(self.cfg))
        if not self.h:
            raise ValueError("invalid oracle config")
        lib().ora_set_selfcheck(self.h, 1 if selfcheck else 0)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_destroy(self.h)
            self.h = None

    def integrate(self, fr: dict) -> dict:
        keep = []
        f = make_frame(fr, keep)
        rep = OraReport()
        rc = lib().ora_integrate(self.h, C.byref(f), C.byref(rep))
        if rc != 0:
            raise RuntimeError(f"oracle integrate rc={rc}: {lib().ora_last_error(self.h).decode()}")
        return rep.as_dict()

    def try_integrate(self, fr: dict):
        keep = []
        f = make_frame(fr, keep)
        rep = OraReport()
        return lib().ora_integrate(self.h, C.byref(f), C.byref(rep))

    def instances(self) -> dict:
        n = lib().ora_num_instances(self.h)
        out = dict(id=np.zeros(n, np.int64), vcount=np.zeros(n, np.int64), obs=np.zeros(n, np.int32),
                   last_seen=np.zeros(n, np.int64), q=np.zeros(n, np.float64),
                   aabb=np.zeros((n, 6), np.int32), e=np.zeros((n, self.Df), np.float64),
                   T=np.zeros((n, max(self.Dt, 0)), np.float64))
        lib().ora_get_instances(self.h, _p(out["id"]), _p(out["vcount"]), _p(out["obs"]),
                                _p(out["last_seen"]), _p(out["q"]), _p(out["aabb"]), _p(out["e"]),
                                _p(out["T"]) if self.Dt > 0 else None, n)
        return out

    def memberships(self):
        n = lib().ora_num_memberships(self.h)
        keys = np.zeros(n, np.uint64)
        ids = np.zeros(n, np.int64)
        lib().ora_get_memberships(self.h, _p(keys), _p(ids), n)
        return keys, ids

    def accept(self, inst_id: int):
        n = lib().ora_get_accept(self.h, inst_id, None, None, 0)
        q = np.zeros(max(n, 0), np.float64)
        e = np.zeros((max(n, 0), self.Df), np.float64)
        if n > 0:
            lib().ora_get_accept(self.h, inst_id, _p(q), _p(e), n)
        return q, e

    def next_id(self) -> int:
        return lib().ora_next_id(self.h)

    def last_frame(self) -> dict:
        S = lib().ora_last_num_masks(self.h)
        st = np.zeros(S, np.int32)
        area = np.zeros(S, np.int64)
        bbox = np.zeros((S, 4), np.int32)
        vs = np.zeros(S, np.int64)
        tgt = np.zeros(S, np.int64)
        lib().ora_last_masks(self.h, _p(st), _p(area), _p(bbox), _p(vs), _p(tgt))
        n = lib().ora_last_pairs(self.h, None, None, 0)
        ps = np.zeros(n, np.int32)
        pk = np.zeros(n, np.uint64)
        lib().ora_last_pairs(self.h, _p(ps), _p(pk), n)
        nt = lib().ora_last_triples(self.h, None, None, None, None, 0)
        ts = np.zeros(nt, np.int32)
        tj = np.zeros(nt, np.int64)
        tc = np.zeros(nt, np.int64)
        te = np.zeros(nt, np.int32)
        lib().ora_last_triples(self.h, _p(ts), _p(tj), _p(tc), _p(te), nt)
        f6 = np.zeros((S, 6), np.float64)
        e = np.zeros((S, self.Df), np.float64)
        Dt = max(self.Dt, 0)
        u = np.zeros((S, Dt), np.float64)
        t = np.zeros((S, Dt), np.float64)
        lib().ora_last_quality(self.h, _p(f6), _p(e), _p(u) if Dt else None, _p(t) if Dt else None)
        return dict(status=st, area=area, bbox=bbox, vs=vs, target=tgt, pair_s=ps, pair_key=pk,
                    trip_s=ts, trip_j=tj, trip_c=tc, trip_edge=te, factors=f6, e=e, u=u, t=t)

    def finalize(self, tau_geo=None, tau_vis=None, min_voxels=0) -> dict:
        """Orphan merge to a fixpoint + minimum-size filter (R35-R38)."""
        rep = OraFinalReport()
        tg = self.cfg.tau_geo if tau_geo is None else tau_geo
        tv = self.cfg.tau_vis if tau_vis is None else tau_vis
        rc = lib().ora_finalize(self.h, tg, tv, int(min_voxels), C.byref(rep))
        if rc != 0:
            raise RuntimeError(f"oracle finalize rc={rc}: {lib().ora_last_error(self.h).decode()}")
        return rep.as_dict()

    def classify(self, table, k: int):
        """Top-k classes (table rows) of every live instance with an embedding."""
        table = np.ascontiguousarray(table, np.float32)
        C = table.shape[0]
        n = lib().ora_classify(self.h, _p(table), C, k, None, None, None, 0)
        kk = min(k, C)
        ids = np.zeros(n, np.int64)
        cls = np.zeros((n, kk), np.int32)
        sc = np.zeros((n, kk), np.float64)
        lib().ora_classify(self.h, _p(table), C, k, _p(ids), _p(cls), _p(sc), n)
        return ids, cls, sc

    def dense_transfer(self, points, d_assign: float):
        """Nearest-voxel-centre instance per point, -1 = unassigned."""
        pts = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
        out = np.zeros(pts.shape[0], np.int64)
        lib().ora_dense_transfer(self.h, _p(pts), pts.shape[0], d_assign, _p(out))
        return out

    def query(self, q, k: int):
        q = np.ascontiguousarray(q, np.float32)
        ids = np.zeros(k, np.int64)
        sc = np.zeros(k, np.float64)
        n = lib().ora_query(self.h, _p(q), k, _p(ids), _p(sc))
        return ids[:n], sc[:n]


# ---- single steps (pins) ----------------------------------------------------------------

def pixel_world(cfg: OraConfig, fr: dict, u: int, v: int):
    keep = []
    f = make_frame(fr, keep)
    out = np.zeros(3, np.float32)
    ok = lib().ora_pixel_world(C.byref(cfg), C.byref(f), u, v, _p(out))
    return bool(ok), out


def point_key(p, r: float):
    p = np.ascontiguousarray(p, np.float32)
    out = np.zeros(3, np.int32)
    ok = lib().ora_point_key(_p(p), C.c_float(r), _p(out))
    return bool(ok), out


def pack_key(ix, iy, iz) -> int:
    return int(lib().ora_pack_key(int(ix), int(iy), int(iz)))


def pose_rigid(pose) -> bool:
    p = np.ascontiguousarray(pose, np.float32).reshape(16)
    return bool(lib().ora_pose_rigid(_p(p)))


def distinctiveness(feats, eps=1e-6):
    F = np.ascontiguousarray(feats, np.float32)
    P, Df = F.reshape(-1, F.shape[-1]).shape
    D = np.zeros(P, np.float64)
    lib().ora_distinctiveness(P, Df, _p(F), eps, _p(D))
    return D


def pool(cnt, npix, D, feats, cover_min=0.25):
    cnt = np.ascontiguousarray(cnt, np.int64)
    npix = np.ascontiguousarray(npix, np.int64)
    D = np.ascontiguousarray(D, np.float64)
    F = np.ascontiguousarray(feats, np.float32)
    P = cnt.shape[0]
    Df = F.shape[-1]
    e = np.zeros(Df, np.float64)
    dbar = C.c_double(0)
    rc = lib().ora_pool(P, Df, _p(cnt), _p(npix), _p(D), _p(F), cover_min, _p(e), C.byref(dbar))
    return rc, e, dbar.value


def s_size(area, H, W, lam=3.3):
    return lib().ora_s_size(area, H, W, lam)


def s_angle(normals, rays):
    N = np.ascontiguousarray(normals, np.float64)
    Rr = np.ascontiguousarray(rays, np.float64)
    return lib().ora_s_angle(N.shape[0], _p(N), _p(Rr))


def s_sem(e, g):
    e = np.ascontiguousarray(e, np.float64)
    g = None if g is None else np.ascontiguousarray(g, np.float32)
    return lib().ora_s_sem(e.shape[0], _p(e), _p(g))


def s_dist(dbar):
    return lib().ora_s_dist(dbar)


def quality(a, b, c, d):
    return lib().ora_quality(a, b, c, d)


def dot_pin(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return lib().ora_dot_pin(a.shape[0], _p(a), _p(b))


def dbscan(points, eps: float, min_pts: int):
    """Classic sequential DBSCAN labels (R42): cluster number in creation order or -1."""
    pts = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
    lab = np.zeros(pts.shape[0], np.int32)
    n = lib().ora_dbscan(pts.shape[0], _p(pts), eps, min_pts, _p(lab))
    return lab, n
