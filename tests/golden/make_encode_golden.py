"""Golden vectors for the frame encoder (protocol.encode_frame RAW).

Test infrastructure: imports the reference package from /root/reference (in
the build container only) and encodes the reference-composed scene frame of
``scene.npz`` plus a synthetic frame that exercises rounding ties, clipping,
the depth_far clamp and inf depths.  Output: ``encode.npz``.
Run: python tests/golden/make_encode_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from radfarm.core import Frame  # noqa: E402
from radfarm.protocol import ENC_DEFLATE, encode_frame  # noqa: E402


def enc(rgba, depth, far=10.0):
    h, w = depth.shape
    fd = encode_frame(Frame(width=w, height=h, rgba=rgba, depth=depth), depth_far=far)
    return (np.frombuffer(fd.rgba, np.uint8).reshape(h, w, 4).copy(),
            np.frombuffer(fd.depth, "<u2").reshape(h, w).copy())


def main():
    g = np.load(os.path.join(HERE, "scene.npz"))
    s8, s16 = enc(g["rgba"], g["depth"])
    rng = np.random.default_rng(7)
    rgba = rng.uniform(-0.1, 1.1, (16, 16, 4)).astype(np.float32)
    rgba.reshape(-1)[:64] = (np.arange(64, dtype=np.float32) + 0.5) / 255.0   # .5 ties
    depth = rng.uniform(0.0, 14.0, (16, 16)).astype(np.float32)
    depth[::5, ::3] = np.inf
    depth[1, :4] = [0.0, 10.0, 10.5, 5.0]
    r8, r16 = enc(rgba, depth)
    # ENC_DEFLATE (protocol.py:265-267): the zlib streams themselves
    h, w = g["depth"].shape
    fz = encode_frame(Frame(width=w, height=h, rgba=g["rgba"], depth=g["depth"]), ENC_DEFLATE)
    sz = encode_frame(Frame(width=16, height=16, rgba=rgba, depth=depth), ENC_DEFLATE, 7.5)
    np.savez_compressed(os.path.join(HERE, "encode.npz"), scene_rgba8=s8, scene_depth16=s16,
                        syn_rgba=rgba, syn_depth=depth, syn_rgba8=r8, syn_depth16=r16,
                        scene_deflate_rgba=np.frombuffer(fz.rgba, np.uint8),
                        scene_deflate_depth=np.frombuffer(fz.depth, np.uint8),
                        syn_deflate_rgba=np.frombuffer(sz.rgba, np.uint8),
                        syn_deflate_depth=np.frombuffer(sz.depth, np.uint8))
    print("done")


if __name__ == "__main__":
    main()
