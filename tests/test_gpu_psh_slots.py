"""The CUDA path's PSH addresses, read back from the shading kernels
themselves (nolf_debug_psh_slots), against the reference's integers.

north_star: PSH addresses must be bit-exact.  The rgba tolerance cannot pin
them (features are U(+-1e-4), so one wrong corner moves rgba by ~1e-6), and
the shaders do not run the reference's u64 ``(h0 + Phi[h1]) % m``
(encoding.py:130-140): k_shade uses per-axis residue tables in u32
(nolf_device.cuh:psh_slot), k_shade_tc the same tables staged in shared
memory with Phi narrowed to u16 (nolf_shade_tc.cuh:tc_gather_inputs).  So
each variant's slots are compared with the golden ``psh_slots`` of every
render case (tests/golden/make_golden.py dumps them from the reference's
PshTable.corner_slots), in both MLP modes, and through the fused scene path."""

import numpy as np
import pytest

from golden_util import asset, camera, case_asset, load, render_cases
from oracle import oracle as O
from paper_2303_04086_b200 import render as R
from paper_2303_04086_b200.model import RayRange

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["fp32", "bf16"])
def mlp_mode(request):
    R.set_mlp_mode(request.param)
    yield request.param
    R.set_mlp_mode("fp32")


@pytest.mark.parametrize("case", render_cases())
def test_render_range_psh_slots_equal_reference(case, mlp_mode):
    g = load(f"render_{case}.npz")
    if "psh_slots" not in g:
        pytest.skip("case has no shaded hits")
    a = case_asset(case, g)
    x0, y0, x1, y1 = (int(v) for v in g["rect"])
    n = (x1 - x0) * (y1 - y0)
    with R.debug_psh_slots(n) as dbg:
        R.render_range(a, RayRange(camera(g), x0, y0, x1, y1))
    got = dbg.slots()
    hr = g["hit_rows"]
    assert len(hr) > 0
    assert np.array_equal(got[hr], g["psh_slots"]), f"{case} ({mlp_mode}): PSH addresses differ"
    miss = np.ones(n, bool)
    miss[hr] = False
    assert np.all(got[miss] == -1), "a non-hit row was shaded"


@pytest.mark.parametrize("name", ["rays_sphere", "rays_sphere_xform"])
def test_render_rays_psh_slots_equal_reference(name, mlp_mode):
    g = load(f"{name}.npz")
    a = case_asset("sphere", g)
    with R.debug_psh_slots(len(g["dirs"])) as dbg:
        R.render_rays(a, g["origins"], g["dirs"])
    got = dbg.slots()
    assert np.array_equal(got[g["hit_rows"]], g["psh_slots"])


@pytest.mark.parametrize("tile", [32, 17])
def test_fused_scene_psh_slots_equal_oracle(tile, mlp_mode):
    """render_scene (chunk cull + march + k_shade(_tc) + compose): the slots
    of every compose layer equal the oracle's for that (asset, pixel); the
    oracle's slots are pinned to the reference in test_oracle.py."""
    g = load("scene.npz")
    names = {"sphere": "toy_sphere", "box": "toy_box", "two": "toy_two"}
    scene = [(asset(names[str(n)]), tr) for n, tr in zip(g["names"], g["transforms"])]
    cam = camera(g)
    W, H = cam.width, cam.height
    tiles = R.frame_tiles(W, H, tile)
    stride = tile * tile
    P = len(tiles) * stride
    with R.debug_psh_slots(len(scene) * P) as dbg:
        R.render_scene(scene, cam, tile=tile)
    got = dbg.slots().reshape(len(scene), P, 8)
    # oracle per asset: hit flags and slots of every pixel (row-major)
    px, py = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    dirs = O.camera_dirs(cam, px.reshape(-1), py.reshape(-1))
    origins = np.broadcast_to(np.asarray(cam.pose)[:3, 3], dirs.shape)
    hits, slots = [], []
    for a, tr in scene:
        import dataclasses
        placed = dataclasses.replace(a, object_to_world=np.asarray(tr, np.float64))
        _, _, D = O.render_rays(placed, origins, dirs, debug=True)
        hits.append(D["hit"])
        slots.append(D["slots"])
    idx = R.unpack_index(tiles, stride, W, H)          # packed slot of every pixel
    n_checked = 0
    layer = np.zeros(W * H, np.int64)                  # next compose layer per pixel
    for k in range(len(scene)):
        rows = np.flatnonzero(hits[k])
        lay = layer[rows]
        np.testing.assert_array_equal(got[lay, idx[rows]], slots[k][rows],
                                      err_msg=f"asset {k}: PSH addresses differ from the oracle")
        layer[rows] += 1
        n_checked += len(rows)
    assert n_checked > 0
