"""nolf_host_scatter (the host half of the sparse frame delivery): packed
non-miss 8-pixel runs of the live chunks -> row-major encode_frame RAW
frame, runs that were written before and are misses now reset.  Pure host
code in libnolf_b200.so: runs without a GPU."""

import ctypes as C

import numpy as np
import pytest

from paper_2303_04086_b200 import _native as N
from paper_2303_04086_b200.render import frame_tiles, unpack_index


def _pack(frame8, frame16, tiles, stride, W, H, live):
    """What the compose epilogue packs: per live chunk its non-miss runs."""
    idx = unpack_index(tiles, stride, W, H)               # packed slot of every pixel
    slot_px = np.full(len(tiles) * stride, -1, np.int64)
    slot_px[idx[idx >= 0]] = np.flatnonzero(idx >= 0)
    heads, runs = [], []
    for c in live:
        mask, first = 0, len(runs)
        for r in range(16):
            px = slot_px[c * 128 + 8 * r:c * 128 + 8 * r + 8]
            r8 = np.zeros((8, 4), np.uint8)
            d16 = np.full(8, 65535, np.uint16)
            ok = px >= 0
            r8[ok] = frame8.reshape(-1, 4)[px[ok]]
            d16[ok] = frame16.reshape(-1)[px[ok]]
            if r8.any() or (d16 != 65535).any():
                mask |= 1 << r
                runs.append(np.concatenate([r8.reshape(-1), d16.view(np.uint8)]))
        heads.append((c, mask, first))
    return (np.ascontiguousarray(np.array(runs, np.uint8).reshape(-1, 48)) if runs else np.zeros((1, 48), np.uint8),
            np.ascontiguousarray(np.array(heads, np.uint32).reshape(-1, 3)))


def _scatter(runs, heads, tiles, stride, W, H, f8, f16, dirty, threads=4):
    rc = N.lib().nolf_host_scatter(runs.ctypes.data, heads.ctypes.data, len(heads), tiles.ctypes.data, len(tiles),
                                   stride, W, H, f8.ctypes.data, f16.ctypes.data, dirty.ctypes.data, threads)
    N.check(rc)


@pytest.mark.parametrize("W,H", [(64, 40), (96, 64)])
def test_scatter_rebuilds_frame_and_resets_stale_runs(W, H):
    rng = np.random.default_rng(W)
    stride = 1024
    tiles = np.ascontiguousarray(frame_tiles(W, H, 32), np.int32)
    n_chunks = len(tiles) * stride // 128
    f8 = np.zeros((H, W, 4), np.uint8)
    f16 = np.full((H, W), 65535, np.uint16)
    dirty = np.zeros(n_chunks, np.uint16)
    idx = unpack_index(tiles, stride, W, H)
    for step in range(4):
        want8 = rng.integers(0, 256, (H, W, 4), dtype=np.uint8)
        want16 = rng.integers(0, 65535, (H, W), dtype=np.uint16)
        hit = rng.uniform(size=(H, W)) < 0.15                 # sparse hits, many all-miss runs
        live = np.sort(rng.choice(n_chunks, size=n_chunks // 3, replace=False)).astype(np.uint32)
        keep = hit & np.isin(idx // 128, live).reshape(H, W)
        want8[~keep] = 0
        want16[~keep] = 65535
        runs, heads = _pack(want8, want16, tiles, stride, W, H, live)
        _scatter(runs, heads, tiles, stride, W, H, f8, f16, dirty)
        np.testing.assert_array_equal(f8, want8)
        np.testing.assert_array_equal(f16, want16)
        assert int((dirty != 0).sum()) > 0


def test_scatter_rejects_bad_headers():
    tiles = np.ascontiguousarray(frame_tiles(32, 32, 32), np.int32)
    f8 = np.zeros((32, 32, 4), np.uint8)
    f16 = np.zeros((32, 32), np.uint16)
    dirty = np.zeros(8, np.uint16)
    runs = np.zeros((1, 48), np.uint8)
    heads = np.array([[99, 1, 0]], np.uint32)
    rc = N.lib().nolf_host_scatter(runs.ctypes.data, heads.ctypes.data, 1, tiles.ctypes.data, 1, 1024, 32, 32,
                                   f8.ctypes.data, f16.ctypes.data, dirty.ctypes.data, 1)
    assert rc == N.NOLF_EDATA
