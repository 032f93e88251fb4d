"""Multi-GPU frame composition over ray tiles.

Every rank renders the tiles t with t mod N == rank (all assets replicated),
composes them locally, and the encoded tiles (rgba8 + u16 depth, 6 B/px,
protocol.encode_frame RAW) are gathered to rank 0 in ONE collective per
frame; rank 0 writes the row-major frame with nolf_unpack_gathered.
"""

from __future__ import annotations

import math

import numpy as np

from .schedule import gather_slots, row_owners, row_partition, tile_partition


def partition(tiles: np.ndarray, world: int, tile: int, by_rows: bool = True, weights=None):
    """Per-rank tile index lists (row-interleaved by default, optionally
    weighted per rank)."""
    if by_rows:
        return [row_partition(tiles, world, r, tile, weights) for r in range(world)]
    return [tile_partition(len(tiles), world, r) for r in range(world)]


def shard_tiles(tiles: np.ndarray, world: int, rank: int, parts=None):
    """(this rank's tiles padded with empty tiles to n_max, n_max)."""
    if parts is None:
        parts = [tile_partition(len(tiles), world, r) for r in range(world)]
    n_max = max(max(len(p) for p in parts), 1)
    mine = tiles[parts[rank]]
    pad = np.zeros((n_max - len(mine), 5), np.int32)      # x0 == x1: no pixels
    return np.concatenate([mine, pad]).astype(np.int32), n_max


def slot_tile_table(tiles: np.ndarray, world: int, parts=None) -> np.ndarray:
    """Tile of every gathered slot (rank-major), empty rows for padding."""
    if parts is None:
        parts = [tile_partition(len(tiles), world, r) for r in range(world)]
    n_max = max(max(len(p) for p in parts), 1)
    table = np.zeros((world * n_max, 5), np.int32)
    table[gather_slots(len(tiles), world, parts)] = tiles
    return table


def row_bands(world: int, rank: int, n_views: int, width: int, height: int, tile: int, weights=None):
    """2-D copy descriptors (in pixels) covering this rank's tile rows of a
    row-major frame stack (cameras concatenated): (first_pixel, width_px,
    pitch_px, height).  Plain round robin: full bands as one strided copy per
    camera, a partial last band as its own copy; weighted owners: one copy
    per run of consecutive owned rows."""
    rows_per_cam = -(-height // tile)
    owners = row_owners(n_views * rows_per_cam, world, weights)
    out = []
    if weights is not None and not all(w == weights[0] for w in weights):
        for c in range(n_views):
            ty = 0
            while ty < rows_per_cam:
                if owners[c * rows_per_cam + ty] != rank:
                    ty += 1
                    continue
                t0 = ty
                while ty < rows_per_cam and owners[c * rows_per_cam + ty] == rank:
                    ty += 1
                npx = (min(ty * tile, height) - t0 * tile) * width
                out.append(((c * height + t0 * tile) * width, npx, npx, 1))
        return out
    for c in range(n_views):
        mine = [ty for ty in range(rows_per_cam) if owners[c * rows_per_cam + ty] == rank]
        full = [ty for ty in mine if (ty + 1) * tile <= height]
        tail = [ty for ty in mine if (ty + 1) * tile > height]
        if full:
            out.append(((c * height + full[0] * tile) * width, tile * width, world * tile * width,
                        len(full)))
        for ty in tail:
            out.append(((c * height + ty * tile) * width, (height - ty * tile) * width,
                        (height - ty * tile) * width, 1))
    return out


def rank_buffer_bytes(n_max: int, tile_stride: int) -> int:
    """Per-rank gather payload: n_max slots of rgba8 then their depth16."""
    return n_max * tile_stride * 6


def gather_to_root(buf, gathered, world: int, rank: int):
    """One collective per frame: every rank's encoded tiles to rank 0."""
    import torch.distributed as dist
    if world == 1:
        return buf
    dist.gather(buf, list(gathered.chunk(world)) if rank == 0 else None, dst=0)
    return gathered
