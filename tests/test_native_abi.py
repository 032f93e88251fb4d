"""The C-ABI library loads without a GPU and exports every entry point that
include/nolf.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2303_04086_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "nolf.h")).read()
    return sorted(set(re.findall(r"\b(nolf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for n in ("nolf_asset_create", "nolf_render_rays", "nolf_render_rect", "nolf_render_scene",
              "nolf_compose", "nolf_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.nolf_abi_version() == _native.ABI_VERSION == 4


def test_workspace_size_is_monotone():
    lib = _native.lib()
    assert lib.nolf_workspace_bytes(1, 1000) < lib.nolf_workspace_bytes(2, 1000)
    assert lib.nolf_workspace_bytes(1, 1000) < lib.nolf_workspace_bytes(1, 2000)


def test_invalid_arguments_fail_loudly_without_gpu():
    lib = _native.lib()
    rc = lib.nolf_compose(0, 10, None, None, 0.5, None, None, None)
    assert rc == _native.NOLF_EINVAL
    assert b"at least one frame" in lib.nolf_last_error()


def test_deflate_matches_python_zlib():
    """nolf_deflate (ENC_DEFLATE, protocol.py:265-267) == zlib.compress(x, 6)
    byte for byte when the library's zlib is the interpreter's."""
    import zlib
    import numpy as np
    from paper_2303_04086_b200 import render
    from golden_util import load
    lib = _native.lib()
    if lib.nolf_zlib_version().decode() != zlib.ZLIB_RUNTIME_VERSION:
        import pytest
        pytest.skip("different zlib builds")
    g = load("encode.npz")
    for key in ("scene_rgba8", "scene_depth16", "syn_rgba8"):
        raw = np.ascontiguousarray(g[key]).tobytes()
        assert render.deflate(raw) == zlib.compress(raw, 6)
    assert render.deflate(np.ascontiguousarray(g["scene_rgba8"]).tobytes()) == g["scene_deflate_rgba"].tobytes()
    assert render.deflate(np.ascontiguousarray(g["scene_depth16"]).astype("<u2").tobytes()) == \
        g["scene_deflate_depth"].tobytes()


def test_launch_options_are_validated_without_gpu():
    lib = _native.lib()
    for key, good, bad in ((_native.OPT_MARCH_ORDER, 2, 3), (_native.OPT_COMPOSE_SLOTS, 8, 5),
                           (_native.OPT_MARCH_SPLIT, 2, 3), (_native.OPT_CHUNK_COST, 0, 2),
                           (_native.OPT_HEAVY_WAVES, 3, -1)):
        assert lib.nolf_set_option(key, good) == 0
        assert lib.nolf_set_option(key, bad) == _native.NOLF_EINVAL
    assert lib.nolf_set_option(99, 0) == _native.NOLF_EINVAL
    # back to the defaults (options are per thread)
    for key, v in ((_native.OPT_MARCH_ORDER, 0), (_native.OPT_COMPOSE_SLOTS, 0), (_native.OPT_MARCH_SPLIT, 1),
                   (_native.OPT_CHUNK_COST, 1), (_native.OPT_HEAVY_WAVES, 3)):
        assert lib.nolf_set_option(key, v) == 0
