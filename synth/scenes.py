"""Synthetic scene streams shaped like the paper's workloads (BASELINE.json configs).

Harness only (see synth/__init__.py).  Every random draw is a counter-based hash of
(seed, stream, index), so a frame's bytes depend only on (config, seed, frame index) and
every rank / device can regenerate any frame independently.  The recipe per config is
stated in DESIGN.md §4 (after SURVEY.md §8(d) "Synthetic inputs").

Geometry: axis-aligned boxes ray-cast forward from a pinhole camera with OpenCV axes
(x right, y down, z forward), pose camera->world row-major 4x4.  Depth is z-depth (the ray
parameter t of a camera ray with z = 1).  Masks: one per visible object; large room
surfaces are split into 2-4 frame-varying Voronoi pieces (SAM-like over-segmentation).
Tokens: per-object unit prototypes mixed by pixel share per 14x14-style patch + noise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

MASK32 = 0xFFFFFFFF
PIECES = 64   # segment id = object id * PIECES + piece


# ----------------------------------------------------------------------------------------
# counter-based randomness (device independent: int64 arithmetic, low 32 bits kept)
# ----------------------------------------------------------------------------------------

def _mix32(x: torch.Tensor) -> torch.Tensor:
    x = x & MASK32
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & MASK32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & MASK32
    x = x ^ (x >> 16)
    return x


def hash_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    s = _mix32(torch.tensor([(seed * 0x9E3779B1 + stream * 0x85EBCA77) & MASK32], dtype=torch.int64,
                            device=idx.device))
    return _mix32(_mix32(idx.to(torch.int64) ^ s) + s)


def hash_uniform(seed: int, stream: int, n: int, device) -> torch.Tensor:
    idx = torch.arange(n, dtype=torch.int64, device=device)
    h = hash_u32(seed, stream, idx)
    return ((h >> 8).to(torch.float32) + 0.5) * (1.0 / 16777216.0)


def hash_normal(seed: int, stream: int, n: int, device) -> torch.Tensor:
    u1 = hash_uniform(seed, stream * 2 + 1, n, device)
    u2 = hash_uniform(seed, stream * 2 + 2, n, device)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def np_rng(seed: int, stream: int) -> np.random.Generator:
    """Counter-based (Philox) host generator for small scene parameters."""
    return np.random.Generator(np.random.Philox(key=[seed & MASK32, stream & MASK32]))


# ----------------------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------------------

@dataclass
class SceneConfig:
    name: str
    H: int
    W: int
    fx: float
    fy: float
    cx: float
    cy: float
    voxel: float
    n_masks: int
    Hp: int
    Wp: int
    Df: int
    Dt: int
    frames: int
    scene: str = "room"                 # "tiny" | "room" | "building"
    room: tuple = (6.5, 5.0, 3.0)
    n_objects: int = 60
    noise: bool = False
    valid_max: float = 10.0             # depth beyond this is reported as 0 (invalid)
    min_area: int = 400
    overlap_masks: bool = False         # X: SAM-"everything" hierarchical masks
    traj: str = "orbit"
    pieces: tuple = (2, 4)              # Voronoi pieces per large room surface per frame
    split_frac: float = 0.04            # objects covering more of the image are split 1-3x
    fill_masks: bool = False            # refine segments up to ~n_masks per frame (mean n_masks, +-20 %)
    extra: dict = field(default_factory=dict)


def _hp(H):
    return H // 14


CONFIGS = {
    "T": SceneConfig("T", 48, 64, 32.0, 32.0, 32.0, 24.0, 0.05, 4, 16, 16, 64, 32, 3,
                     scene="tiny", n_objects=3, min_area=8, traj="tiny"),
    "R": SceneConfig("R", 680, 1200, 600.0, 600.0, 599.5, 339.5, 0.02, 40, _hp(680), _hp(1200),
                     1024, 384, 2000, room=(6.5, 5.0, 3.0), n_objects=140, traj="orbit", pieces=(4, 8),
                     split_frac=0.02, fill_masks=True),
    "N": SceneConfig("N", 480, 640, 577.6, 578.7, 318.9, 242.7, 0.05, 30, _hp(480), _hp(640),
                     1024, 384, 5000, room=(7.0, 6.0, 3.0), n_objects=90, noise=True,
                     valid_max=4.5, traj="handheld", pieces=(3, 6), split_frac=0.03,
                     fill_masks=True),
    "H": SceneConfig("H", 480, 640, 320.0, 320.0, 320.0, 240.0, 0.02, 60, _hp(480), _hp(640),
                     1024, 384, 20000, scene="building", n_objects=2400, traj="tour", pieces=(3, 6),
                     split_frac=0.02, fill_masks=True),
    "X": SceneConfig("X", 480, 640, 577.6, 578.7, 318.9, 242.7, 0.05, 50, _hp(480), _hp(640),
                     1024, 384, 300, room=(7.0, 6.0, 3.0), n_objects=40, overlap_masks=True,
                     traj="handheld"),
}

CONFIG_INDEX = {"T": 0, "R": 1, "N": 2, "H": 3, "X": 4}


def seed_of(name: str) -> int:
    return 0xD15C0000 + CONFIG_INDEX.get(name[0], 9)


def disc_config_kwargs(cfg: SceneConfig) -> dict:
    """disc_config / ora_config fields for a scene config (defaults of R8, R11, R16)."""
    return dict(voxel_size=cfg.voxel, tau_geo=0.3, tau_vis=0.8, depth_min=0.1, depth_max=10.0,
                mask_min_conf=0.5, mask_max_aspect=10.0, mask_min_area=cfg.min_area,
                cover_min=0.25, lambda_size=3.3, eps_distinct=1e-6, feat_dim=cfg.Df,
                track_dim=cfg.Dt)


# ----------------------------------------------------------------------------------------
# scene construction (host, small)
# ----------------------------------------------------------------------------------------

@dataclass
class Scene:
    lo: np.ndarray            # [B,3] box mins (world)
    hi: np.ndarray            # [B,3]
    obj: np.ndarray           # [B] object id of each box
    room_lo: np.ndarray | None
    room_hi: np.ndarray | None
    n_obj: int                # total object ids (room surfaces 0..5 first when a room exists)
    splittable: np.ndarray    # [n_obj] bool: large surfaces split SAM-like
    floors: list = field(default_factory=list)   # building: list of (z0, z1)
    nav: list = field(default_factory=list)      # building: navigable waypoints


def _room_scene(cfg: SceneConfig, seed: int) -> Scene:
    rng = np_rng(seed, 1)
    L = np.array(cfg.room, np.float64)
    lo, hi = [], []
    n = cfg.n_objects
    for i in range(n):
        kind = rng.uniform()
        if kind < 0.6:      # floor object
            sz = rng.uniform([0.25, 0.25, 0.2], [1.0, 1.0, 1.1])
            p = rng.uniform([0.2, 0.2], L[:2] - 0.2 - sz[:2])
            lo.append([p[0], p[1], 0.0]); hi.append([p[0] + sz[0], p[1] + sz[1], sz[2]])
        else:               # wall-mounted thin object (picture, shelf)
            w, h, dpt = rng.uniform(0.3, 1.2), rng.uniform(0.3, 0.9), rng.uniform(0.03, 0.25)
            z0 = rng.uniform(0.6, L[2] - h - 0.2)
            side = int(rng.integers(0, 4))
            if side < 2:
                y0 = rng.uniform(0.1, L[1] - w - 0.1)
                x0 = 0.0 if side == 0 else L[0] - dpt
                lo.append([x0, y0, z0]); hi.append([x0 + dpt, y0 + w, z0 + h])
            else:
                x0 = rng.uniform(0.1, L[0] - w - 0.1)
                y0 = 0.0 if side == 2 else L[1] - dpt
                lo.append([x0, y0, z0]); hi.append([x0 + w, y0 + dpt, z0 + h])
    lo = np.array(lo, np.float64).reshape(-1, 3)
    hi = np.array(hi, np.float64).reshape(-1, 3)
    obj = np.arange(n) + 6
    split = np.zeros(n + 6, bool)
    split[:6] = True
    return Scene(lo, hi, obj, np.zeros(3), L, n + 6, split)


def _tiny_scene(cfg: SceneConfig) -> Scene:
    # T: a wall at z in [1.62, 1.70] and three boxes before it with front faces at z-depths
    # that are multiples of 2 cm (1.50, 1.54, 1.58): keys stay >= 0.0125 voxel from
    # boundaries.
    lo = np.array([[-2.0, -2.0, 1.62], [-0.60, -0.45, 1.50], [-0.10, -0.30, 1.54], [0.35, 0.0, 1.58]])
    hi = np.array([[2.0, 2.0, 1.70], [-0.25, 0.10, 1.60], [0.25, 0.30, 1.60], [0.70, 0.45, 1.60]])
    obj = np.arange(4)
    return Scene(lo, hi, obj, None, None, 4, np.zeros(4, bool))


def _building_scene(cfg: SceneConfig, seed: int) -> Scene:
    """H: 3 stories of 40 x 30 m, 4.5-6 m rooms off a central corridor, objects per room."""
    rng = np_rng(seed, 1)
    lo, hi, obj = [], [], []
    oid = 0
    FL, FW, FH, WT = 40.0, 30.0, 3.0, 0.12
    floors = []
    nav = []
    per_room = max(1, cfg.n_objects // (3 * 2 * 7))
    for k in range(3):
        z0 = k * (FH + 0.3)
        floors.append((z0, z0 + FH))
        # slab (floor) and ceiling slab
        lo.append([0, 0, z0 - 0.3]); hi.append([FL, FW, z0]); obj.append(oid); oid += 1
        lo.append([0, 0, z0 + FH]); hi.append([FL, FW, z0 + FH + 0.01]); obj.append(oid); oid += 1
        # outer walls
        for (a, b) in [([0, 0, z0], [FL, WT, z0 + FH]), ([0, FW - WT, z0], [FL, FW, z0 + FH]),
                       ([0, 0, z0], [WT, FW, z0 + FH]), ([FL - WT, 0, z0], [FL, FW, z0 + FH])]:
            lo.append(a); hi.append(b); obj.append(oid); oid += 1
        # corridor along x at y in [13.5, 16.5]; rooms on both sides, 7 per side
        cy0, cy1 = 13.5, 16.5
        xs = np.linspace(0, FL, 8)
        for side in range(2):
            ya, yb = (WT, cy0) if side == 0 else (cy1, FW - WT)
            wall_y = cy0 if side == 0 else cy1
            for r in range(7):
                x0, x1 = xs[r], xs[r + 1]
                # corridor wall with a 1 m door gap in the middle
                xm = 0.5 * (x0 + x1)
                lo.append([x0, wall_y - WT / 2, z0]); hi.append([xm - 0.5, wall_y + WT / 2, z0 + FH])
                obj.append(oid); oid += 1
                lo.append([xm + 0.5, wall_y - WT / 2, z0]); hi.append([x1, wall_y + WT / 2, z0 + FH])
                obj.append(oid); oid += 1
                # partition wall between rooms
                if r < 6:
                    lo.append([x1 - WT / 2, ya, z0]); hi.append([x1 + WT / 2, yb, z0 + FH])
                    obj.append(oid); oid += 1
                # furniture
                for _ in range(per_room):
                    sz = rng.uniform([0.3, 0.3, 0.3], [1.2, 1.2, 1.2])
                    px = rng.uniform(x0 + 0.3, x1 - 0.3 - sz[0])
                    py = rng.uniform(ya + 0.3, yb - 0.3 - sz[1])
                    lo.append([px, py, z0]); hi.append([px + sz[0], py + sz[1], z0 + sz[2]])
                    obj.append(oid); oid += 1
                # navigable room centre and door
                nav.append((k, xm, 0.5 * (ya + yb)))
                nav.append((k, xm, wall_y + (-0.6 if side == 0 else 0.6)))
        for x in np.linspace(2, FL - 2, 10):
            nav.append((k, x, 0.5 * (cy0 + cy1)))
    lo = np.array(lo, np.float64)
    hi = np.array(hi, np.float64)
    obj = np.array(obj)
    split = np.zeros(oid, bool)
    ext = hi - lo
    big = (np.sort(ext, axis=1)[:, 1] > 2.5)  # walls / slabs: split SAM-like
    split[obj[big]] = True
    return Scene(lo, hi, obj, None, None, oid, split, floors, nav)


# ----------------------------------------------------------------------------------------
# trajectories -> camera->world pose (float32, row-major)
# ----------------------------------------------------------------------------------------

def look_pose(pos, yaw: float, pitch: float, roll: float = 0.0) -> np.ndarray:
    """OpenCV camera (x right, y down, z forward) in a z-up world."""
    f = np.array([math.cos(yaw) * math.cos(pitch), math.sin(yaw) * math.cos(pitch), math.sin(pitch)])
    up = np.array([0.0, 0.0, 1.0])
    r = np.cross(f, up)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    if roll != 0.0:
        c, s = math.cos(roll), math.sin(roll)
        r, d = c * r + s * d, -s * r + c * d
    M = np.eye(4)
    M[:3, 0], M[:3, 1], M[:3, 2], M[:3, 3] = r, d, f, pos
    return M.astype(np.float32)


def trajectory_pose(cfg: SceneConfig, scene: Scene, seed: int, f: int) -> np.ndarray:
    if cfg.traj == "tiny":
        M = np.eye(4, dtype=np.float32)
        M[:3, 3] = [[0.0, 0.0, 0.0], [0.04, 0.0, 0.0], [0.04, 0.02, 0.0]][f % 3]
        return M
    if cfg.traj == "orbit":   # R: smooth orbit + walk, looking outward at the walls
        L = np.array(cfg.room)
        w = 2 * math.pi / 400.0
        ctr = L / 2
        pos = np.array([ctr[0] + 0.28 * L[0] * math.cos(w * f), ctr[1] + 0.28 * L[1] * math.sin(w * f),
                        1.35 + 0.15 * math.sin(f / 53.0)])
        yaw = w * f + 0.7 * math.sin(f / 61.0)
        pitch = -0.30 + 0.15 * math.sin(f / 47.0)
        return look_pose(pos, yaw, pitch)
    if cfg.traj == "handheld":   # N / X: Lissajous walk with per-frame jitter
        L = np.array(cfg.room)
        rng = np_rng(seed, 1_000_000 + f)
        j = rng.normal(0, 1, 5)
        pos = np.array([L[0] / 2 + 0.3 * L[0] * math.sin(f / 180.0) + 0.004 * j[0],
                        L[1] / 2 + 0.3 * L[1] * math.sin(f / 130.0 + 1.0) + 0.004 * j[1],
                        1.4 + 0.1 * math.sin(f / 70.0) + 0.003 * j[2]])
        yaw = f / 95.0 + 0.5 * math.sin(f / 41.0) + 0.004 * j[3]
        pitch = -0.25 + 0.12 * math.sin(f / 33.0) + 0.004 * j[4]
        return look_pose(pos, yaw, pitch, roll=0.01 * math.sin(f / 20.0))
    if cfg.traj == "tour":       # H: discrete agent, 0.25 m steps / 15 deg turns, sensor 1.2 m
        return _tour_pose(cfg, scene, seed, f)
    raise ValueError(cfg.traj)


_TOUR_CACHE: dict = {}


def _tour_pose(cfg: SceneConfig, scene: Scene, seed: int, f: int) -> np.ndarray:
    key = (cfg.name, seed)
    if key not in _TOUR_CACHE:
        # visit waypoints floor by floor (stairs teleport between floors: the tour's
        # stairwell segments are not modelled), discretised into forward 0.25 m / turn 15 deg
        rng = np_rng(seed, 7)
        poses = []
        pts = scene.nav
        pos = None
        yaw = 0.0
        order = sorted(range(len(pts)), key=lambda i: (pts[i][0], pts[i][1] if pts[i][0] % 2 == 0 else -pts[i][1]))
        for i in order:
            k, x, y = pts[i]
            z = scene.floors[k][0] + 1.2
            tgt = np.array([x, y, z])
            if pos is None or abs(pos[2] - z) > 0.5:
                pos = tgt.copy()
            while True:
                d = tgt - pos
                dist = math.hypot(d[0], d[1])
                if dist < 0.25:
                    break
                want = math.atan2(d[1], d[0])
                dy = (want - yaw + math.pi) % (2 * math.pi) - math.pi
                if abs(dy) > math.radians(7.5):
                    yaw += math.copysign(math.radians(15), dy)
                else:
                    pos = pos + 0.25 * np.array([math.cos(yaw), math.sin(yaw), 0.0])
                poses.append((pos.copy(), yaw))
            # look around: a full turn in 15 degree steps at each room centre
            for _ in range(int(rng.integers(6, 24))):
                yaw += math.radians(15)
                poses.append((pos.copy(), yaw))
        _TOUR_CACHE[key] = poses
    poses = _TOUR_CACHE[key]
    pos, yaw = poses[f % len(poses)]
    return look_pose(pos, yaw, -0.15)


# ----------------------------------------------------------------------------------------
# generator
# ----------------------------------------------------------------------------------------

class Generator:
    """Deterministic frame source: frame(f) depends only on (cfg, seed, f)."""

    def __init__(self, cfg: SceneConfig | str, seed: int | None = None, device="cpu", **overrides):
        if isinstance(cfg, str):
            cfg = CONFIGS[cfg]
        if overrides:
            cfg = replace(cfg, **overrides)
        self.cfg = cfg
        self.seed = seed_of(cfg.name) if seed is None else seed
        self.device = torch.device(device)
        if cfg.scene == "tiny":
            self.scene = _tiny_scene(cfg)
        elif cfg.scene == "building":
            self.scene = _building_scene(cfg, self.seed)
        else:
            self.scene = _room_scene(cfg, self.seed)
        dev = self.device
        sc = self.scene
        self.lo = torch.tensor(sc.lo, dtype=torch.float32, device=dev)
        self.hi = torch.tensor(sc.hi, dtype=torch.float32, device=dev)
        self.box_obj = torch.tensor(sc.obj, dtype=torch.int64, device=dev)
        # per-object prototypes (unit, Df) and tracking identities (unit, Dt)
        n = sc.n_obj
        self.proto = self._unit_rows(101, n, cfg.Df)
        self.ident = self._unit_rows(202, n, cfg.Dt) if cfg.Dt > 0 else None
        # pixel grid -> camera rays and patch index (input synthesis only)
        v, u = torch.meshgrid(torch.arange(cfg.H, device=dev), torch.arange(cfg.W, device=dev), indexing="ij")
        self.rays_cam = torch.stack([(u.float() - cfg.cx) / cfg.fx, (v.float() - cfg.cy) / cfg.fy,
                                     torch.ones_like(u, dtype=torch.float32)], -1).reshape(-1, 3)
        self.patch_of = ((v * cfg.Hp // cfg.H) * cfg.Wp + (u * cfg.Wp // cfg.W)).reshape(-1)
        self.u = u.reshape(-1)
        self.v = v.reshape(-1)

    def _unit_rows(self, stream: int, n: int, d: int) -> torch.Tensor:
        x = hash_normal(self.seed, stream, n * d, self.device).reshape(n, d)
        return x / x.norm(dim=1, keepdim=True)

    def pose(self, f: int) -> np.ndarray:
        return trajectory_pose(self.cfg, self.scene, self.seed, f)

    # ---- ray casting ----
    def _raycast(self, pose: np.ndarray):
        cfg, dev = self.cfg, self.device
        Rm = torch.tensor(pose[:3, :3], dtype=torch.float32, device=dev)
        o = torch.tensor(pose[:3, 3], dtype=torch.float32, device=dev)
        d = self.rays_cam @ Rm.T
        d = torch.where(d.abs() < 1e-9, torch.full_like(d, 1e-9), d)
        inv = 1.0 / d
        N = d.shape[0]
        t_best = torch.full((N,), float("inf"), device=dev)
        obj = torch.full((N,), -1, dtype=torch.int64, device=dev)
        sc = self.scene
        if sc.room_lo is not None:
            rl = torch.tensor(sc.room_lo, dtype=torch.float32, device=dev)
            rh = torch.tensor(sc.room_hi, dtype=torch.float32, device=dev)
            t1 = (rl - o) * inv
            t2 = (rh - o) * inv
            tfar = torch.maximum(t1, t2)
            t_room, ax = tfar.min(dim=1)
            side = (d.gather(1, ax[:, None])[:, 0] > 0).long()
            t_best = t_room
            obj = ax * 2 + side
        # boxes, culled to those near the camera
        lo, hi, bobj = self.lo, self.hi, self.box_obj
        if lo.shape[0] > 64:   # cull boxes farther than the valid depth range (closest point)
            closest = torch.minimum(torch.maximum(o, lo), hi)
            near = ((closest - o).norm(dim=1) < cfg.valid_max + 0.5)
            lo, hi, bobj = lo[near], hi[near], bobj[near]
        B = lo.shape[0]
        chunk = max(1, (1 << 24) // max(B, 1))
        for s0 in range(0, N, chunk):
            dd = inv[s0:s0 + chunk]
            t1 = (lo[None] - o) * dd[:, None, :]
            t2 = (hi[None] - o) * dd[:, None, :]
            tn = torch.minimum(t1, t2).amax(-1)
            tf = torch.maximum(t1, t2).amin(-1)
            hit = (tn <= tf) & (tn > 1e-4)
            tb = torch.where(hit, tn, torch.full_like(tn, float("inf")))
            tmin, bi = tb.min(dim=1)
            better = tmin < t_best[s0:s0 + chunk]
            t_best[s0:s0 + chunk] = torch.where(better, tmin, t_best[s0:s0 + chunk])
            obj[s0:s0 + chunk] = torch.where(better, bobj[bi], obj[s0:s0 + chunk])
        pts = o + t_best[:, None] * d
        return t_best, obj, pts

    # ---- one frame ----
    def frame(self, f: int, with_feats: bool = True) -> dict:
        cfg, dev, sc = self.cfg, self.device, self.scene
        pose = self.pose(f)
        t, obj, pts = self._raycast(pose)
        HW = cfg.H * cfg.W
        depth = t.clone()
        hitmask = torch.isfinite(depth) & (obj >= 0)
        depth = torch.where(hitmask, depth, torch.zeros_like(depth))
        if cfg.noise:   # N: axial noise sigma(z) = 0.0012 + 0.0019 (z - 0.4)^2, 5% holes
            z = depth
            sig = 0.0012 + 0.0019 * (z - 0.4) ** 2
            depth = z + sig * hash_normal(self.seed, 10_000 + f, HW, dev)
            holes = hash_uniform(self.seed, 20_000_000 + f, HW, dev) < 0.05
            depth = torch.where(holes, torch.zeros_like(depth), depth)
        depth = torch.where(depth > cfg.valid_max, torch.zeros_like(depth), depth)
        obj = torch.where(hitmask, obj, torch.full_like(obj, -1))
        # SAM-like segments: split large surfaces into 2-4 frame-varying Voronoi pieces
        seg = obj * PIECES
        vis = torch.unique(obj[obj >= 0])
        rng = np_rng(self.seed, 3_000_000 + f)
        npix_obj = torch.bincount(obj[obj >= 0], minlength=sc.n_obj)
        for oi in vis.tolist():
            big = int(npix_obj[oi]) > cfg.split_frac * HW
            if not (sc.splittable[oi] or big):
                continue
            k = int(rng.integers(cfg.pieces[0], cfg.pieces[1] + 1)) if sc.splittable[oi] else int(rng.integers(1, 4))
            if k <= 1:
                continue
            sel = obj == oi
            p = pts[sel]
            lo_, hi_ = p.min(0).values, p.max(0).values
            seeds = lo_ + (hi_ - lo_) * torch.tensor(rng.uniform(0, 1, (k, 3)), dtype=torch.float32, device=dev)
            piece = torch.cdist(p, seeds).argmin(1)
            seg[sel] = oi * PIECES + piece
        seg = torch.where(obj >= 0, seg, torch.full_like(seg, -1))
        n_target = cfg.n_masks
        if cfg.fill_masks:   # finer SAM-like over-segmentation up to this frame's mask count
            n_target = int(round(cfg.n_masks * rng.uniform(0.8, 1.2)))
            seg = self._refine(seg, pts, rng, n_target)
        ids, counts = torch.unique(seg[seg >= 0], return_counts=True)
        order = torch.argsort(counts, descending=True, stable=True)
        ids = ids[order][: n_target]
        S_part = ids.shape[0]
        masks = (seg[None, :] == ids[:, None]).to(torch.uint8)
        if cfg.overlap_masks and S_part < cfg.n_masks:
            masks = self._hierarchical(masks, obj, ids, cfg.n_masks)
        S = masks.shape[0]
        conf = 0.4 + 0.6 * hash_uniform(self.seed, 4_000_000 + f, max(S, 1), dev)[:S]
        out = dict(frame_id=f, H=cfg.H, W=cfg.W, fx=cfg.fx, fy=cfg.fy, cx=cfg.cx, cy=cfg.cy,
                   pose=pose, depth=depth.reshape(cfg.H, cfg.W).contiguous(),
                   masks=masks.reshape(S, cfg.H, cfg.W).contiguous(), mask_conf=conf.contiguous(),
                   patch_h=cfg.Hp, patch_w=cfg.Wp, patch_feats=None, global_embed=None,
                   track_feats=None)
        # token grids: pixel share of each visible object per patch
        P = cfg.Hp * cfg.Wp
        vis_obj, inv = torch.unique(obj.clamp_min(0), return_inverse=True)
        share = torch.zeros(P, vis_obj.shape[0], device=dev)
        share.index_put_((self.patch_of, inv), torch.ones(HW, device=dev), accumulate=True)
        share = share / share.sum(1, keepdim=True).clamp_min(1.0)
        if with_feats:
            feats = share @ self.proto[vis_obj]
            feats = feats + 0.05 * hash_normal(self.seed, 5_000_000 + f, P * cfg.Df, dev).reshape(P, cfg.Df)
            scale = 5.0 + 10.0 * hash_uniform(self.seed, 6_000_000 + f, P, dev)
            feats = feats / feats.norm(dim=1, keepdim=True).clamp_min(1e-6) * scale[:, None]
            w = torch.bincount(inv, minlength=vis_obj.shape[0]).float()
            g = (w / w.sum()) @ self.proto[vis_obj]
            out["patch_feats"] = feats.reshape(cfg.Hp, cfg.Wp, cfg.Df).contiguous()
            out["global_embed"] = g.contiguous()
        if cfg.Dt > 0:
            tr = 4.0 * (share @ self.ident[vis_obj])
            tr = tr + 0.02 * hash_normal(self.seed, 7_000_000 + f, P * cfg.Dt, dev).reshape(P, cfg.Dt)
            out["track_feats"] = snap_bf16(tr).reshape(cfg.Hp, cfg.Wp, cfg.Dt).contiguous()
        return out

    def _refine(self, seg, pts, rng, n_target):
        """R/N/H: SAM-like over-segmentation finer than the per-surface split -- while the frame has
        fewer than n_target segments, the largest segment (at least 4 x min_area pixels) is cut in
        two along the Voronoi boundary of two of its own 3-D points (a partition: masks stay
        disjoint, every pixel keeps one segment)."""
        cfg = self.cfg
        ids, counts = torch.unique(seg[seg >= 0], return_counts=True)
        cnt = dict(zip(ids.tolist(), counts.tolist()))
        used = {}
        for i in cnt:
            used[i // PIECES] = max(used.get(i // PIECES, -1), i % PIECES)
        while len(cnt) < n_target:
            L = max(cnt, key=lambda k: (cnt[k], -k))
            o = L // PIECES
            if cnt[L] < 4 * cfg.min_area or used[o] + 1 >= PIECES:
                break
            sel = seg == L
            p = pts[sel]
            a, b = rng.integers(0, p.shape[0], 2)
            if a == b:
                b = (a + p.shape[0] // 2) % p.shape[0]
            second = (p - p[int(b)]).square().sum(1) < (p - p[int(a)]).square().sum(1)
            n2 = int(second.sum())
            if n2 == 0 or n2 == p.shape[0]:
                break
            new = o * PIECES + used[o] + 1
            used[o] += 1
            idx = sel.nonzero()[:, 0]
            seg[idx[second]] = new
            cnt[new] = n2
            cnt[L] -= n2
        return seg

    def _hierarchical(self, masks, obj, ids, n_target):
        """X: add overlapping whole-object and half-segment masks (SAM 'everything')."""
        cfg = self.cfg
        extra = []
        objs = torch.unique(ids // PIECES)
        for oi in objs.tolist():          # whole-object masks (unions of pieces)
            if len(extra) + masks.shape[0] >= n_target:
                break
            if int((ids // PIECES == oi).sum()) > 1:
                extra.append((obj == oi).to(torch.uint8))
        level = 0
        while len(extra) + masks.shape[0] < n_target and level < 4:
            base = torch.cat([masks] + ([torch.stack(extra)] if extra else []), 0)
            added = False
            for m in base:
                if len(extra) + masks.shape[0] >= n_target:
                    break
                sel = m.bool()
                cnt = int(sel.sum())
                if cnt < 800:
                    continue
                us = self.u[sel] if level % 2 == 0 else self.v[sel]
                med = us.float().median()
                coord = self.u if level % 2 == 0 else self.v
                extra.append((sel & (coord.float() <= med)).to(torch.uint8))
                added = True
            level += 1
            if not added:
                break
        if extra:
            masks = torch.cat([masks, torch.stack(extra)[: n_target - masks.shape[0]]], 0)
        return masks


def snap_bf16(x: torch.Tensor) -> torch.Tensor:
    """bf16 values that are multiples of 2^-12 with |x| <= 8 (reading R15): every product
    cnt * g and every sum of them is exact in fp64, so the tracking pooling has one correct
    fp64 result in any summation order."""
    x = x.clamp(-8.0, 8.0).to(torch.bfloat16).float()
    x = torch.round(x * 4096.0) / 4096.0
    y = x.to(torch.bfloat16)
    assert torch.equal(y.float(), x), "snapped value not representable in bf16"
    return y


def frame_to_numpy(fr: dict) -> dict:
    """Host copy of a generated frame in the oracle's layout (bf16 -> uint16 bit patterns)."""
    out = {}
    for k, v in fr.items():
        if isinstance(v, torch.Tensor):
            if v.dtype == torch.bfloat16:
                out[k] = v.view(torch.int16).cpu().numpy().view(np.uint16)
            else:
                out[k] = v.cpu().numpy()
        else:
            out[k] = v
    return out


def pack_mask_bits(masks: torch.Tensor) -> torch.Tensor:
    """[S, H, W] masks (nonzero = in mask) -> [S, ceil(H*W/32)] int32 words in the layout of
    disc_frame::mask_bits: pixel p = v*W + u of plane s is bit p % 32 of word p / 32 (little-endian
    words; bits past H*W zero).  A layout change only: the same binary masks, 1/8 of the bytes."""
    S = masks.shape[0]
    flat = (masks.reshape(S, -1) != 0)
    n = flat.shape[1]
    pad = (-n) % 32
    if pad:
        flat = torch.cat([flat, flat.new_zeros((S, pad))], dim=1)
    w = flat.reshape(S, -1, 32).to(torch.int64) << torch.arange(32, device=masks.device, dtype=torch.int64)
    words = w.sum(dim=2)                                    # < 2^32: every bit once
    return (words - ((words >> 31) << 32)).to(torch.int32)  # the same 32 bits as int32
