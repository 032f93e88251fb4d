"""Ray -> GPU assignment: FarmAssigner replays the reference MasterNode's
recorded dispatches bit for bit (tests/golden/dispatch.json, made by
tests/golden/make_dispatch_golden.py), plus the throughput-mode tile map."""

import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN
from paper_2303_04086_b200.model import Aabb, orbit_camera
from paper_2303_04086_b200.schedule import (FarmAssigner, Thresholds, gather_slots,
                                            tile_partition)

CASES = json.load(open(os.path.join(GOLDEN, "dispatch.json")))


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_assignment_matches_reference_master(idx):
    rec = CASES[idx]
    c = rec["case"]
    proxies = {n: Aabb(min=(0.0, 0.0, 0.0), max=(1.0, 1.0, 1.0)) for n in c["assets"]}
    fa = FarmAssigner(proxies, heavy_workers=c["heavy"], light_workers=c["light"],
                      light_rays_per_tick=c["rays_per_tick"], tick_s=0.005, tile_size=c["tile"],
                      thresholds=Thresholds(**c["thresholds"]))
    cam = orbit_camera(c["azimuth"], c["elevation"], radius=c["radius"], size=c["size"])
    assert np.array_equal(cam.pose, np.asarray(rec["pose"]))
    fa.open(c["size"], c["size"], cam.fx, cam.fy, cam.cx, cam.cy, c["fps"])
    for name, tr in c["edits"]:
        fa.edit_add(name, tr)
    fa.set_pose(cam.pose)
    for t, expected in enumerate(rec["ticks"]):
        got = [list(e) for e in fa.tick(t * 0.005)]
        assert got == expected, f"tick {t}"


@pytest.mark.parametrize("n_tiles,world", [(8160, 1), (8160, 2), (8160, 8), (17, 4), (3, 8)])
def test_tile_partition_covers_every_tile_once(n_tiles, world):
    parts = [tile_partition(n_tiles, world, r) for r in range(world)]
    allt = np.sort(np.concatenate(parts))
    assert np.array_equal(allt, np.arange(n_tiles))
    slots = gather_slots(n_tiles, world)
    assert len(np.unique(slots)) == n_tiles
    n_max = -(-n_tiles // world)
    for r, p in enumerate(parts):    # rank r's j-th tile lands in slot r*n_max + j
        assert np.array_equal(slots[p], r * n_max + np.arange(len(p)))
