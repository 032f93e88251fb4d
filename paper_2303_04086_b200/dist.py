"""Multi-GPU frame composition over ray tiles.

Every rank renders the tiles t with t mod N == rank (all assets replicated),
composes them locally, and the encoded tiles (rgba8 + u16 depth, 6 B/px,
protocol.encode_frame RAW) are gathered to rank 0 in ONE collective per
frame; rank 0 writes the row-major frame with nolf_unpack_gathered.
"""

from __future__ import annotations

import math

import numpy as np

from .schedule import gather_slots, tile_partition


def shard_tiles(tiles: np.ndarray, world: int, rank: int):
    """(this rank's tile rows padded with empty tiles to ceil(n/N), n_max)."""
    n_max = math.ceil(len(tiles) / world)
    mine = tiles[tile_partition(len(tiles), world, rank)]
    pad = np.zeros((n_max - len(mine), 5), np.int32)      # x0 == x1: no pixels
    return np.concatenate([mine, pad]).astype(np.int32), n_max


def slot_tile_table(tiles: np.ndarray, world: int) -> np.ndarray:
    """Tile of every gathered slot (rank-major), empty rows for padding."""
    n_max = math.ceil(len(tiles) / world)
    table = np.zeros((world * n_max, 5), np.int32)
    table[gather_slots(len(tiles), world)] = tiles
    return table


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
