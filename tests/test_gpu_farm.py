"""GPU farm workers with the real kernels (farm.GpuFarm, one GPU: every
worker on rank 0): the reference master's dispatch log replayed tick by
tick (tests/golden/dispatch.json) with every task rendered by the CUDA path
and every finished frame equal to compose(render_frame(scene, camera)) --
tile-partition invariance (test_renderer.py:38-48) plus farm.compose.
The 2-GPU run of the same check is tools/farm_check.py."""

import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN, asset
from paper_2303_04086_b200 import render as R
from paper_2303_04086_b200.farm import GpuFarm
from paper_2303_04086_b200.model import orbit_camera
from paper_2303_04086_b200.schedule import Thresholds

pytestmark = pytest.mark.gpu
CASES = json.load(open(os.path.join(GOLDEN, "dispatch.json")))
TOY = {"a": "toy_sphere", "b": "toy_box", "c": "toy_two", "d": "toy_sphere"}


def run_case(rec, world=1, rank=0):
    c = rec["case"]
    assets = {n: asset(TOY[n]) for n in c["assets"]}
    cam = orbit_camera(c["azimuth"], c["elevation"], radius=c["radius"], size=c["size"])
    farm = GpuFarm(assets, heavy_workers=c["heavy"], light_workers=c["light"],
                   light_rays_per_tick=c["rays_per_tick"], tile_size=c["tile"],
                   thresholds=Thresholds(**c["thresholds"]), world=world, rank=rank)
    farm.open(c["size"], c["size"], cam.fx, cam.fy, cam.cx, cam.cy, c["fps"])
    for name, tr in c["edits"]:
        farm.edit_add(name, tr)
    farm.set_pose(cam.pose)
    logs, frames = [], []
    for t in range(len(rec["ticks"])):
        log, fin = farm.tick(t * 0.005)
        logs.append([list(e) for e in log])
        frames += fin
    named = [(n, np.eye(4)) for n in sorted(c["assets"])]       # session scene order (farm.py SceneEdit)
    for name, tr in c["edits"]:
        named = [e for e in named if e[0] != name] + [(name, np.asarray(tr, np.float64))]
    return logs, frames, [(assets[n], tr) for n, tr in named], cam


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_gpu_farm_replays_dispatch_and_composes(idx):
    rec = CASES[idx]
    logs, frames, scene, cam = run_case(rec)
    assert logs == rec["ticks"]
    assert frames, "no frame finished"
    ref = R.compose(R.render_frame(scene, cam))
    for f in frames:
        assert f.timed_out_tiles == 0
        np.testing.assert_array_equal(f.frame.rgba, ref.rgba)
        np.testing.assert_array_equal(f.frame.depth, ref.depth)
