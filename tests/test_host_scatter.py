"""nolf_host_scatter (the host half of the sparse frame delivery): packed
live chunks -> row-major encode_frame RAW frame, stale chunks reset to the
miss encoding.  Pure host code in libnolf_b200.so: runs without a GPU."""

import ctypes as C

import numpy as np
import pytest

from paper_2303_04086_b200 import _native as N
from paper_2303_04086_b200.render import frame_tiles, unpack_index


def _pack(frame8, frame16, tiles, stride, W, H, ids):
    """What the compose epilogue packs: each chunk's 128 slots in slot order."""
    idx = unpack_index(tiles, stride, W, H)               # packed slot of every pixel
    slot_px = np.full(len(tiles) * stride, -1, np.int64)
    slot_px[idx[idx >= 0]] = np.flatnonzero(idx >= 0)
    pack = np.zeros((len(ids), 768), np.uint8)
    for i, c in enumerate(ids):
        px = slot_px[c * 128:(c + 1) * 128]
        r8 = np.zeros((128, 4), np.uint8)
        d16 = np.full(128, 65535, np.uint16)
        ok = px >= 0
        r8[ok] = frame8.reshape(-1, 4)[px[ok]]
        d16[ok] = frame16.reshape(-1)[px[ok]]
        pack[i, :512] = r8.reshape(-1)
        pack[i, 512:] = d16.view(np.uint8)
    return pack


def _scatter(pack, ids, tiles, stride, W, H, f8, f16, prev, prev_n, threads=4):
    ids = np.ascontiguousarray(ids, np.uint32)
    rc = N.lib().nolf_host_scatter(pack.ctypes.data, ids.ctypes.data, len(ids), tiles.ctypes.data, len(tiles),
                                   stride, W, H, f8.ctypes.data, f16.ctypes.data, prev.ctypes.data,
                                   C.byref(prev_n), threads)
    N.check(rc)


@pytest.mark.parametrize("W,H", [(64, 40), (96, 64)])
def test_scatter_rebuilds_frame_and_clears_stale_chunks(W, H):
    rng = np.random.default_rng(W)
    stride = 1024
    tiles = np.ascontiguousarray(frame_tiles(W, H, 32), np.int32)
    n_chunks = len(tiles) * stride // 128
    f8 = np.zeros((H, W, 4), np.uint8)
    f16 = np.full((H, W), 65535, np.uint16)
    prev = np.zeros(n_chunks, np.uint32)
    prev_n = C.c_uint32(0)
    idx = unpack_index(tiles, stride, W, H)
    for step in range(3):
        want8 = rng.integers(0, 256, (H, W, 4), dtype=np.uint8)
        want16 = rng.integers(0, 65535, (H, W), dtype=np.uint16)
        live = np.sort(rng.choice(n_chunks, size=n_chunks // 3, replace=False)).astype(np.uint32)
        # pixels outside live chunks are misses in a real frame
        in_live = np.isin(idx // 128, live).reshape(H, W)
        want8[~in_live] = 0
        want16[~in_live] = 65535
        pack = _pack(want8, want16, tiles, stride, W, H, live)
        _scatter(pack, live, tiles, stride, W, H, f8, f16, prev, prev_n)
        np.testing.assert_array_equal(f8, want8)
        np.testing.assert_array_equal(f16, want16)
        assert prev_n.value == len(live) and np.array_equal(prev[:len(live)], live)


def test_scatter_rejects_bad_ids():
    tiles = np.ascontiguousarray(frame_tiles(32, 32, 32), np.int32)
    f8 = np.zeros((32, 32, 4), np.uint8)
    f16 = np.zeros((32, 32), np.uint16)
    prev = np.zeros(8, np.uint32)
    pack = np.zeros((1, 768), np.uint8)
    rc = N.lib().nolf_host_scatter(pack.ctypes.data, np.array([99], np.uint32).ctypes.data, 1, tiles.ctypes.data,
                                   1, 1024, 32, 32, f8.ctypes.data, f16.ctypes.data, prev.ctypes.data,
                                   C.byref(C.c_uint32(0)), 1)
    assert rc == N.NOLF_EDATA
