"""Hand-worked fixture T0.

64x48 image, fx = fy = 32, cx = 32, cy = 24, a fronto-parallel wall at z-depth 1.62 m,
voxel r = 0.05 m.  Frame 0 (pose I): masks A = {u < 32}, B = {u >= 32}.  Frame 1 (pose
translated by (0.05, 0, 0)): mask C = {16 <= u < 48}.  Frame 2 = frame 1.  Expected values
are in tests/golden/t0.json; they are derived by hand there, not computed by any code here.
"""
from __future__ import annotations

import numpy as np

T0_H, T0_W = 48, 64
T0_INTR = dict(fx=32.0, fy=32.0, cx=32.0, cy=24.0)
T0_DEPTH = 1.62
T0_VOXEL = 0.05


def t0_frame(index: int, with_tokens: bool = False, Df: int = 16, Dt: int = 0) -> dict:
    H, W = T0_H, T0_W
    depth = np.full((H, W), T0_DEPTH, np.float32)
    u = np.arange(W)[None, :].repeat(H, 0)
    pose = np.eye(4, dtype=np.float32)
    if index == 0:
        masks = np.stack([(u < 32), (u >= 32)]).astype(np.uint8)
    else:
        pose[0, 3] = 0.05
        masks = ((u >= 16) & (u < 48))[None].astype(np.uint8)
    fr = dict(frame_id=index, depth=depth, masks=masks, mask_conf=None, pose=pose,
              patch_h=16, patch_w=16, patch_feats=None, global_embed=None, track_feats=None,
              **T0_INTR)
    if with_tokens:
        rng = np.random.default_rng(1234)  # fixed tokens: every frame sees the same wall
        fr["patch_feats"] = rng.standard_normal((16, 16, Df)).astype(np.float32)
        fr["global_embed"] = rng.standard_normal(Df).astype(np.float32)
    if Dt > 0:
        # identical tracking tokens everywhere: every detection has the same t, gate passes
        g = np.zeros((16, 16, Dt), np.float32)
        g[..., 0] = 1.0
        fr["track_feats"] = (g.view(np.uint32) >> 16).astype(np.uint16)
    return fr
