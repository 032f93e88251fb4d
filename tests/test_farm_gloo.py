"""GPU farm workers (farm.GpuFarm) on world size 2, gloo on CPU: the
reference master's dispatches (tests/golden/dispatch.json) split over two
ranks (worker k on rank k mod 2), every rank's tiles exchanged to rank 0
and assembled into the composed frame.  The renderer and the compose are
replaced by host stand-ins here (no GPU); tests/test_gpu_farm.py runs the
real kernels."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import GOLDEN
from oracle import oracle as O
from paper_2303_04086_b200.farm import GpuFarm
from paper_2303_04086_b200.model import Aabb, orbit_camera
from paper_2303_04086_b200.schedule import Thresholds

CASES = json.load(open(os.path.join(GOLDEN, "dispatch.json")))


class _Stub:
    proxy = Aabb(min=(0.0, 0.0, 0.0), max=(1.0, 1.0, 1.0))


def fake_frame(name, W, H):
    """What a renderer would produce for asset `name` over the whole frame."""
    y, x = np.mgrid[0:H, 0:W]
    k = ord(name) - ord("a") + 1
    a = ((x * 3 + y * 5 + 7 * k) % 11) / 10.0
    rgba = np.stack([a * 0.3, a * 0.5, a * (k % 3) / 3, a], -1).astype(np.float32)
    depth = np.where(a > 0, 1.0 + ((x + 2 * y + k) % 7), np.inf).astype(np.float32)
    return rgba, depth


def make_farm(rec, world, rank):
    c = rec["case"]
    cam = orbit_camera(c["azimuth"], c["elevation"], radius=c["radius"], size=c["size"])
    full = {n: fake_frame(n, c["size"], c["size"]) for n in c["assets"]}

    def execute(task, camera, transform):
        x0, y0, x1, y1 = task.rect
        if task.skip:
            return (torch.zeros((y1 - y0, x1 - x0, 4)), torch.full((y1 - y0, x1 - x0), float("inf")))
        r, d = full[task.asset_id]
        return torch.from_numpy(r[y0:y1, x0:x1].copy()), torch.from_numpy(d[y0:y1, x0:x1].copy())

    def compose(rgba, depth):
        o, d = O.compose(rgba.numpy(), depth.numpy())
        return torch.from_numpy(o), torch.from_numpy(d)

    farm = GpuFarm({n: _Stub() for n in c["assets"]}, heavy_workers=c["heavy"], light_workers=c["light"],
                   light_rays_per_tick=c["rays_per_tick"], tile_size=c["tile"],
                   thresholds=Thresholds(**c["thresholds"]), world=world, rank=rank,
                   device=torch.device("cpu"), execute=execute, compose=compose)
    farm.open(c["size"], c["size"], cam.fx, cam.fy, cam.cx, cam.cy, c["fps"])
    for name, tr in c["edits"]:
        farm.edit_add(name, tr)
    farm.set_pose(cam.pose)
    return farm, full


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for rec in CASES:
            farm, full = make_farm(rec, world, rank)
            frames, logs = [], []
            for t in range(len(rec["ticks"])):
                log, fin = farm.tick(t * 0.005)
                logs.append([list(e) for e in log])
                frames += [(f.index, f.frame.rgba, f.frame.depth, f.timed_out_tiles) for f in fin]
            ranks = sorted({e[-1] for e in farm.log})
            res.append((logs, frames, ranks))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def two_rank_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_two_rank_farm_replays_reference_dispatch(two_rank_run, idx):
    rec = CASES[idx]
    for rank in (0, 1):
        logs, _, _ = two_rank_run[rank][idx]
        assert logs == rec["ticks"], f"rank {rank}: dispatch log differs from the reference master"


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_two_rank_farm_frames_equal_compose_of_full_frames(two_rank_run, idx):
    rec = CASES[idx]
    c = rec["case"]
    logs, frames, ranks = two_rank_run[0][idx]
    assert frames, "no frame finished"
    assert two_rank_run[1][idx][1] == []                 # only rank 0 assembles
    if any(e[5].startswith("light") for t in rec["ticks"] for e in t) and c["light"] > 1:
        assert ranks == [0, 1], "both ranks must render"
    # scene order: sorted assets, edits re-appended (farm.py: SceneEdit add)
    order = sorted(c["assets"])
    for name, _ in c["edits"]:
        order = [n for n in order if n != name] + [name]
    full = {n: fake_frame(n, c["size"], c["size"]) for n in c["assets"]}
    skip = {e[1] for t in rec["ticks"] for e in t if e[6]}
    rg = np.stack([np.zeros_like(full[n][0]) if n in skip else full[n][0] for n in order])
    dp = np.stack([np.full_like(full[n][1], np.inf) if n in skip else full[n][1] for n in order])
    want_rgba, want_depth = O.compose(rg, dp)
    for index, rgba, depth, timed_out in frames:
        if timed_out:
            continue
        np.testing.assert_array_equal(rgba, want_rgba)
        np.testing.assert_array_equal(depth, want_depth)
