"""Packed tile-slot layout (nolf_kernels.cuh:slot_xy) and its host mirror."""

import numpy as np
import pytest

from paper_2303_04086_b200.render import frame_tiles, slot_xy, unpack_index


@pytest.mark.parametrize("W,H,T", [(70, 45, 16), (64, 64, 32), (3840, 2160, 32), (33, 7, 8)])
def test_unpack_index_is_the_inverse_of_slot_xy(W, H, T):
    tiles = frame_tiles(W, H, T)
    idx = unpack_index(tiles, T * T, W, H)
    assert (idx >= 0).all()
    assert len(np.unique(idx)) == W * H
    for t in (0, len(tiles) // 2, len(tiles) - 1):
        c, x0, y0, x1, y1 = tiles[t]
        w, h = x1 - x0, y1 - y0
        lx, ly = slot_xy(np.arange(w * h), w, h)
        assert sorted(zip(lx.tolist(), ly.tolist())) == [(x, y) for x in range(w) for y in range(h)]
        np.testing.assert_array_equal(idx[(y0 + ly) * W + x0 + lx], t * T * T + np.arange(w * h))


def test_full_tiles_use_8x4_warp_blocks():
    lx, ly = slot_xy(np.arange(32), 32, 32)
    assert set(lx.tolist()) == set(range(8)) and set(ly.tolist()) == set(range(4))
    lx, ly = slot_xy(np.arange(20), 20, 1)          # ragged edge tile: row-major
    np.testing.assert_array_equal(lx, np.arange(20))
