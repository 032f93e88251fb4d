"""Native .nolf reader (nolf_asset_load / _mem, csrc/nolf_load.h), the C
counterpart of assetio.read_asset (assetio.py:48-66, 174-255).  Corrupt input
is rejected with NOLF_EDATA before any device call, so those cases run on
CPU; the GPU half checks a natively loaded asset renders bit-identically to
the Python-loaded one."""

import ctypes as C
import gzip
import struct
import zlib

import numpy as np
import pytest

from golden_util import GOLDEN
from paper_2303_04086_b200 import _native as N
from paper_2303_04086_b200 import nolf_io

ASSET = f"{GOLDEN}/assets/toy_sphere.nolf.gz"


def _raw():
    return gzip.decompress(open(ASSET, "rb").read())


def _load_mem(buf):
    h = C.c_void_p()
    o2w = (C.c_double * 16)()
    rc = N.lib().nolf_asset_load_mem(bytes(buf), len(buf), 0, C.byref(h), o2w)
    return rc, N.lib().nolf_last_error().decode()


def _table(raw):
    count = struct.unpack_from("<H", raw, 6)[0]
    out = {}
    for i in range(count):
        pos = 8 + i * 36
        name = raw[pos:pos + 16].rstrip(b"\0").decode()
        out[name] = (pos,) + struct.unpack_from("<QQI", raw, pos + 16)
    return out


@pytest.mark.parametrize("mutate,msg", [
    (lambda r: b"NOPE" + r[4:], "bad magic"),
    (lambda r: r[:6], "truncated"),
    (lambda r: r[:4] + struct.pack("<H", 7) + r[6:], "unsupported asset version"),
    (lambda r: r[:40], "section table truncated"),
])
def test_corrupt_container_is_a_data_error(mutate, msg):
    rc, err = _load_mem(mutate(_raw()))
    assert rc == N.NOLF_EDATA and msg in err, err


def test_checksum_mismatch_is_a_data_error():
    raw = bytearray(_raw())
    pos, off, length, crc = _table(bytes(raw))["den_cubes"]
    raw[off + length // 2] ^= 0x40
    rc, err = _load_mem(raw)
    assert rc == N.NOLF_EDATA and "den_cubes failed its checksum" in err


def test_bad_meta_and_sizes_are_data_errors():
    asset = nolf_io.read_asset(ASSET)
    sections = nolf_io.unpack_sections(_raw())
    bad = dict(sections)
    bad["meta"] = b"{not json"
    rc, err = _load_mem(nolf_io.pack_sections(bad))
    assert rc == N.NOLF_EDATA and "meta" in err
    bad = dict(sections)
    bad["psh_features"] = bad["psh_features"][:-4]
    rc, err = _load_mem(nolf_io.pack_sections(bad))
    assert rc == N.NOLF_EDATA and "psh_features" in err
    bad = dict(sections)
    del bad["fs_w1"]
    rc, err = _load_mem(nolf_io.pack_sections(bad))
    assert rc == N.NOLF_EDATA and "missing section fs_w1" in err
    assert asset.psh.offset_size > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["toy_sphere", "toy_box", "toy_live", "toy_norefine"])
def test_native_load_renders_like_python_load(name):
    import torch
    from paper_2303_04086_b200 import render as R
    path = f"{GOLDEN}/assets/{name}.nolf.gz"
    a_py = nolf_io.read_asset(path)
    a_c = R.load_device_asset(path)
    np.testing.assert_array_equal(a_c.object_to_world, a_py.object_to_world)
    assert a_c.bf16_ok == R.bf16_capable(a_py)
    from paper_2303_04086_b200.model import orbit_camera
    cam = orbit_camera(0.5, 0.4, radius=2.0, size=64)
    outs = []
    for a in (a_py, a_c):
        r = R.SceneRenderer([(a, None)])
        tiles = R.frame_tiles(cam.width, cam.height, 32)
        out = r.alloc(len(tiles), 1024, want_f32=True, want_u8=False)
        r.render([cam], torch.from_numpy(tiles).to(r.device), len(tiles), 1024, out, frame_layout=True)
        outs.append((out["rgba"].cpu().numpy(), out["depth"].cpu().numpy(), out["counters"].cpu().numpy()))
    for x, y in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(x, y)
    assert outs[0][2][3] > 0                      # samples were marched
    if name == "toy_sphere":
        assert np.isfinite(outs[0][1]).sum() > 0


@pytest.mark.parametrize("path,value", [
    (("density_atlas", "b"), 1 << 20),          # b^3 overflows the cell count
    (("density_atlas", "r"), 100000),
    (("density_atlas", "cubes"), 1 << 40),
    (("psh", "table_size"), 1 << 40),
    (("psh", "features"), 1 << 33),
    (("diffuse_encoder", "base_resolution"), 1 << 40),
    (("specular_mlp", "widths"), [19, 1 << 40, 64, 4]),
])
def test_hostile_meta_sizes_are_data_errors(path, value):
    """Untrusted meta sizes are bounded before any multiplication or
    allocation: NOLF_EDATA, never an overflowed size or an exception across
    the C ABI."""
    import json
    sec = nolf_io.unpack_sections(_raw())
    meta = json.loads(sec["meta"])
    meta[path[0]][path[1]] = value
    sec["meta"] = json.dumps(meta).encode()
    rc, err = _load_mem(nolf_io.pack_sections(sec))
    assert rc == N.NOLF_EDATA, err


def test_deeply_nested_meta_is_a_data_error():
    sec = nolf_io.unpack_sections(_raw())
    sec["meta"] = b"[" * 100000 + b"]" * 100000
    rc, err = _load_mem(nolf_io.pack_sections(sec))
    assert rc == N.NOLF_EDATA, err
