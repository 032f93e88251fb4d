"""The package's own .nolf reader/writer on the reference-written fixtures."""

import gzip
import os

import numpy as np
import pytest

from golden_util import GOLDEN
from paper_2303_04086_b200 import errors, nolf_io


def raw(name="toy_sphere"):
    return gzip.decompress(open(os.path.join(GOLDEN, "assets", f"{name}.nolf.gz"), "rb").read())


@pytest.mark.parametrize("name", ["toy_sphere", "toy_box", "toy_two", "toy_live", "toy_norefine"])
def test_round_trip_preserves_every_array(name):
    a = nolf_io.read_asset(raw(name))
    b = nolf_io.read_asset(nolf_io.write_asset(a))
    for attr in ("density_atlas", "diffuse_atlas"):
        x, y = getattr(a, attr), getattr(b, attr)
        if x is None:
            assert y is None
            continue
        assert np.array_equal(x.index, y.index) and np.array_equal(x.cubes, y.cubes)
    assert np.array_equal(a.psh.offsets, b.psh.offsets)
    assert np.array_equal(a.psh_features, b.psh_features)
    for m1, m2 in ((a.specular_mlp, b.specular_mlp), (a.diffuse_mlp, b.diffuse_mlp)):
        for w1, w2 in zip(m1.weights + m1.biases, m2.weights + m2.biases):
            assert np.array_equal(w1, w2)
    assert a.wiring == b.wiring and a.march == b.march


def test_sections_byte_identical_to_reference_writer():
    data = raw()
    a = nolf_io.read_asset(data)
    s1 = nolf_io.unpack_sections(data)
    s2 = nolf_io.unpack_sections(nolf_io.write_asset(a))
    assert set(s1) == set(s2)
    for k in s1:
        if k != "meta":
            assert s1[k] == s2[k], k


def test_corruption_is_a_data_error():
    data = bytearray(raw())
    data[-5] ^= 0xFF
    with pytest.raises(errors.DataError):
        nolf_io.read_asset(bytes(data))
    with pytest.raises(errors.DataError):
        nolf_io.read_asset(b"XXXX" + bytes(data[4:]))
    with pytest.raises(errors.DataError):
        nolf_io.read_asset(bytes(data[:60]))
