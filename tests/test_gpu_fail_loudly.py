"""Device-side failures are reported, never blended into pixels.

Every case here is impossible for valid input (the host sizes hit queues
and compose layers from the instances' screen boxes); each one is forced
with an invalid tile list and must raise CapacityError (the reference's
class for "demand exceeds capacity", errors.py) instead of writing wrong or
out-of-bounds pixels.  The frames that are written stay memory-safe."""

import numpy as np
import pytest

from golden_util import asset, camera, load
from paper_2303_04086_b200 import errors
from paper_2303_04086_b200 import render as R
from paper_2303_04086_b200.model import orbit_camera

pytestmark = pytest.mark.gpu


def _scene():
    g = load("scene.npz")
    names = {"sphere": "toy_sphere", "box": "toy_box", "two": "toy_two"}
    return g, [(asset(names[str(n)]), tr) for n, tr in zip(g["names"], g["transforms"])]


def _render(scene, cam, tiles, stride=1024):
    import torch
    r = R.SceneRenderer(scene)
    t = torch.from_numpy(np.asarray(tiles, np.int32).reshape(-1, 5)).to(r.device)
    # frame-layout outputs hold the whole frame
    out = r.alloc(max(len(tiles), -(-cam.width * cam.height // stride)), stride, want_f32=False, want_u8=True)
    r.render([cam], t, len(tiles), stride, out, frame_layout=True)
    return r, out


def test_tile_outside_frame_raises():
    g, scene = _scene()
    cam = camera(g)
    r, _ = _render(scene, cam, [[0, 0, 0, 32, 32], [0, 48, 48, 80, 80]])   # 2nd tile past 64x64
    with pytest.raises(errors.CapacityError, match="tiles skipped"):
        r.check()
    r.check()                                       # reported once, then clean again


def test_tile_larger_than_slot_raises():
    g, scene = _scene()
    cam = camera(g)
    r, _ = _render(scene, cam, [[0, 0, 0, 40, 40]], stride=1024)        # 1600 px > 1024 slots
    with pytest.raises(errors.CapacityError):
        r.check()


def test_missing_camera_raises():
    g, scene = _scene()
    cam = camera(g)
    r, _ = _render(scene, cam, [[3, 0, 0, 32, 32]])                      # camera 3 of 1
    with pytest.raises(errors.CapacityError):
        r.check()


def test_duplicated_tiles_overflow_the_hit_queue():
    """Every tile listed 40 times: each pixel is marched 40 times, so the hit
    records exceed the queue the host sized from the screen box (at most the
    frame's 4096 pixels)."""
    a = asset("toy_sphere")
    cam = orbit_camera(0.8, 0.3, radius=1.2, size=64)
    tiles = np.concatenate([R.frame_tiles(64, 64, 32)] * 40)
    r, _ = _render([(a, np.eye(4))], cam, tiles)
    with pytest.raises(errors.CapacityError, match="hit queue"):
        r.check()


def test_error_also_fails_the_next_render_call():
    import torch
    g, scene = _scene()
    cam = camera(g)
    r, _ = _render(scene, cam, [[0, 60, 60, 92, 92]])
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)                                # the asynchronous read-back has landed
    t = torch.from_numpy(R.frame_tiles(64, 64, 32)).to(r.device)
    out = r.alloc(len(t), 1024, want_f32=False, want_u8=True)
    with pytest.raises(errors.CapacityError):
        r.render([cam], t, len(t), 1024, out, frame_layout=True)
    r.render([cam], t, len(t), 1024, out, frame_layout=True)        # then it works again
    r.check()


def test_valid_frames_report_nothing():
    g, scene = _scene()
    cam = camera(g)
    r, _ = _render(scene, cam, R.frame_tiles(64, 64, 32))
    r.check()


def test_empty_padding_tiles_are_valid():
    """Uneven shards pad their tile lists with empty rects: no pixels, no error."""
    g, scene = _scene()
    cam = camera(g)
    tiles = np.concatenate([R.frame_tiles(64, 64, 32), np.zeros((3, 5), np.int32)])
    r, _ = _render(scene, cam, tiles)
    r.check()
