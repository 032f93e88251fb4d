"""synth.py's restatement of the reference asset pipeline vs the reference's
toy assets (tests/golden/assets/*.nolf.gz, built by make_golden.py with the
reference's bake_density_cubes / init_light_field / bake_diffuse_cubes)."""

import numpy as np
import pytest

from golden_util import asset, load
from tools import synth

SEEDS = {"sphere": 3, "box": 1, "two": 2}
TOY = dict(b=16, r=4, psh_resolution=16, diffuse_levels=3, diffuse_table=2 ** 10)


@pytest.mark.parametrize("kind", ["sphere", "box", "two"])
def test_cpu_stages_equal_reference(kind):
    ref = asset(f"toy_{kind}")
    sh = load("shells.npz")
    a = synth.make_asset(kind, SEEDS[kind], shell_points=sh[f"{kind}_psh"], bake_diffuse=False,
                         **TOY)
    # bake_density_cubes
    assert np.array_equal(a.density_atlas.index, ref.density_atlas.index)
    assert np.array_equal(a.density_atlas.cubes, ref.density_atlas.cubes)
    # psh_construct over the voxelised hit shell
    assert (a.psh.table_size, a.psh.offset_size) == (ref.psh.table_size, ref.psh.offset_size)
    assert np.array_equal(a.psh.offsets, ref.psh.offsets)
    # init_light_field rng draw order
    assert np.array_equal(a.psh_features, ref.psh_features)
    for m1, m2 in ((a.specular_mlp, ref.specular_mlp), (a.diffuse_mlp, ref.diffuse_mlp)):
        assert m1.heads == m2.heads
        for x, y in zip(m1.weights + m1.biases, m2.weights + m2.biases):
            assert np.array_equal(x, y)
    for x, y in zip(a.diffuse_features, ref.diffuse_features):
        assert np.array_equal(x, y)
    # the diffuse-shell mask gives the reference's diffuse index grid
    mask = synth.voxelize(sh[f"{kind}_dif"], 16, 1)
    cells, pts = synth.masked_sample_points(mask, 4)
    idx = np.full((16, 16, 16), -1, np.int32)
    for cid, (i, j, k) in enumerate(cells):
        idx[i, j, k] = cid
    assert np.array_equal(idx, ref.diffuse_atlas.index)
    assert len(pts) == len(cells) * 125


def test_psh_is_perfect_on_random_sets():
    rng = np.random.default_rng(0)
    for n in (8, 16):
        occ = rng.uniform(size=(n, n, n)) < 0.2
        v = synth.occupied_vertices(occ)
        t = synth.build_psh(v, n)
        u = v.astype(np.uint64)
        h0 = (u @ synth.P0) % np.uint64(t.table_size)
        h1 = (u @ synth.P1) % np.uint64(t.offset_size)
        slots = (h0 + t.offsets.astype(np.uint64)[h1]) % np.uint64(t.table_size)
        assert len(np.unique(slots)) == len(v)


def test_zodiac_layout():
    tr = synth.zodiac_transforms()
    assert len(tr) == 12
    centres = [m[:3, :3] @ np.full(3, 0.5) + m[:3, 3] for m in tr]
    np.testing.assert_allclose([np.hypot(c[0], c[1]) for c in centres], 2.0)
    cam = synth.zodiac_camera()
    assert (cam.width, cam.height) == (3840, 2160)
    np.testing.assert_allclose(np.linalg.norm(cam.position), 4.0)
