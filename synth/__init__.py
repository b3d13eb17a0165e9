"""Seeded synthetic RGB-D + mask + token streams for the DISC hot path (harness only).

This package produces INPUTS.  It holds none of the method's arithmetic (no back-projection,
voxelisation, pooling, distinctiveness, quality or association): it ray-casts box scenes
forward (world -> image) and synthesises masks and token grids from the ray hits.  Both the
CUDA path and the CPU oracle consume the bytes it produces; neither imports the other.
"""
from .scenes import CONFIGS, SceneConfig, Generator, frame_to_numpy, disc_config_kwargs, pack_mask_bits  # noqa: F401
from .fixtures import t0_frame  # noqa: F401
