"""World-size-2 (gloo, CPU) test of the multi-GPU frame composer's host
logic: tile sharding, the single gather of every rank's encoded tiles, and
the rank-major slot table rank 0 uses to assemble the frame."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_04086_b200.dist import (gather_to_root, partition, rank_buffer_bytes, row_bands,
                                        shard_tiles, slot_tile_table)
from paper_2303_04086_b200.render import frame_tiles, slot_xy

W, H, T = 70, 45, 16
STRIDE = T * T


def pixel_code(x, y):
    return ((x * 7 + y * 13) % 251).astype(np.uint8)


def worker(rank, world, port, q, by_rows):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tiles = frame_tiles(W, H, T)
        parts = partition(tiles, world, T, by_rows=by_rows)
        mine, n_max = shard_tiles(tiles, world, rank, parts)
        P = n_max * STRIDE
        buf = np.zeros(rank_buffer_bytes(n_max, STRIDE), np.uint8)
        rgba = buf[:P * 4].reshape(P, 4)
        depth = buf[P * 4:].view(np.uint16)
        for j, (c, x0, y0, x1, y1) in enumerate(mine):   # "render": encode pixel coordinates
            w, h = x1 - x0, y1 - y0
            for l in range(w * h):
                lx, ly = slot_xy(l, w, h)
                x, y = x0 + lx, y0 + ly
                rgba[j * STRIDE + l] = [pixel_code(np.int64(x), np.int64(y)), rank + 1, 0, 255]
                depth[j * STRIDE + l] = y * W + x
        t = torch.from_numpy(buf)
        gathered = torch.empty(world * t.numel(), dtype=torch.uint8) if rank == 0 else None
        out = gather_to_root(t, gathered, world, rank)
        if rank == 0:
            g = out.numpy()
            table = slot_tile_table(tiles, world, parts)
            frame = np.zeros((H * W, 4), np.uint8)
            fdepth = np.zeros(H * W, np.uint16)
            per = rank_buffer_bytes(n_max, STRIDE)
            for s, (c, x0, y0, x1, y1) in enumerate(table):   # what k_unpack does
                r, j = divmod(s, n_max)
                base = g[r * per:(r + 1) * per]
                w, h = x1 - x0, y1 - y0
                for l in range(w * h):
                    lx, ly = slot_xy(l, w, h)
                    dst = (y0 + ly) * W + x0 + lx
                    frame[dst] = base[(j * STRIDE + l) * 4:(j * STRIDE + l) * 4 + 4]
                    fdepth[dst] = base[P * 4:].view(np.uint16)[j * STRIDE + l]
            q.put((frame, fdepth))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("by_rows", [False, True])
def test_two_rank_gather_assembles_the_frame(by_rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, by_rows)) for r in range(2)]
    for p in procs:
        p.start()
    frame, fdepth = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ys, xs = np.mgrid[0:H, 0:W]
    assert np.array_equal(fdepth.reshape(H, W), (ys * W + xs).astype(np.uint16))
    assert np.array_equal(frame[:, 0].reshape(H, W), pixel_code(xs, ys))
    tiles = frame_tiles(W, H, T)
    owner = np.zeros((H, W), np.uint8)
    for r, p in enumerate(partition(tiles, 2, T, by_rows=by_rows)):
        for c, x0, y0, x1, y1 in tiles[p]:
            owner[y0:y1, x0:x1] = r + 1
    assert np.array_equal(frame[:, 1].reshape(H, W), owner)   # each tile rendered by its owner


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_row_bands_cover_every_pixel_once(world):
    for V, w, h, t in ((1, 3840, 2160, 32), (16, 216, 216, 32), (2, 64, 45, 16)):
        cnt = np.zeros(V * h * w, np.int32)
        for r in range(world):
            for first, wpx, ppx, hgt in row_bands(world, r, V, w, h, t):
                for k in range(hgt):
                    cnt[first + k * ppx:first + k * ppx + wpx] += 1
        assert cnt.min() == 1 and cnt.max() == 1


@pytest.mark.parametrize("world,w0", [(2, 0.8), (4, 0.85), (3, 0.5)])
def test_weighted_row_partition_and_bands(world, w0):
    """--rank0-weight: rank 0 gets ~w0/(w0 + N-1) of the tile rows; the row
    bands of the weighted owners still cover every pixel exactly once and
    agree with the tile partition."""
    from paper_2303_04086_b200.schedule import row_owners
    weights = [w0] + [1.0] * (world - 1)
    for V, w, h, t in ((1, 3840, 2160, 32), (3, 96, 70, 16)):
        tiles = frame_tiles(w, h, t)
        tiles = np.concatenate([frame_tiles(w, h, t, cam=c) for c in range(V)])
        parts = partition(tiles, world, t, by_rows=True, weights=weights)
        assert sorted(np.concatenate(parts).tolist()) == list(range(len(tiles)))
        cnt = np.zeros(V * h * w, np.int32)
        for r in range(world):
            own = np.zeros(V * h * w, bool)
            for first, wpx, ppx, hgt in row_bands(world, r, V, w, h, t, weights):
                for k in range(hgt):
                    cnt[first + k * ppx:first + k * ppx + wpx] += 1
                    own[first + k * ppx:first + k * ppx + wpx] = True
            for c, x0, y0, x1, y1 in tiles[parts[r]]:
                assert own[(c * h + y0) * w + x0] and own[(c * h + y1 - 1) * w + x1 - 1]
        assert cnt.min() == 1 and cnt.max() == 1
        owners = row_owners(1000, world, weights)
        share = (owners == 0).mean()
        assert abs(share - w0 / (w0 + world - 1)) < 0.01
