"""B200-native i-NOLF render path (NEPHELE, arXiv 2303.04086).

Drop-in for the reference package's one-query-per-ray hot path:
``render_rays`` / ``render_range`` / ``render_frame`` / ``compose`` with the
reference signatures, plus the fused multi-asset ``SceneRenderer``.  The
compute runs in libnolf_b200.so (hand-written CUDA for sm_100a, C ABI in
include/nolf.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from . import errors  # noqa: F401
from .model import (Aabb, Camera, Frame, LightFieldAsset, MarchParams, ModelWiring,  # noqa: F401
                    RayRange, RenderCounters, Tile, look_at, orbit_camera)
from .nolf_io import read_asset, write_asset  # noqa: F401


def __getattr__(name):
    # render entry points import torch lazily (first import can be slow)
    if name in ("render_rays", "render_ray", "render_range", "render_frame", "compose",
                "compose_device", "render_scene", "SceneRenderer", "frame_tiles", "device_asset",
                "invalidate", "unpack_index", "slot_xy", "load_device_asset"):
        from . import render
        return getattr(render, name)
    raise AttributeError(name)
