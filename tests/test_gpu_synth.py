"""GPU halves of the asset pipeline: hit-shell march (nolf_march_rays) and the
diffuse bake (nolf_eval_diffuse) against the reference's outputs."""

import numpy as np
import pytest

from golden_util import asset, load
from tools import synth

pytestmark = pytest.mark.gpu
SEEDS = {"sphere": 3, "box": 1, "two": 2}


@pytest.mark.parametrize("kind", ["sphere", "box", "two"])
def test_shell_points_bit_exact(kind):
    ref = asset(f"toy_{kind}")
    sh = load("shells.npz")
    p = synth.collect_hit_points_gpu(ref.density_atlas, ref.march, 12, 16)
    assert p.shape == sh[f"{kind}_psh"].shape
    assert np.array_equal(p, sh[f"{kind}_psh"]), "collect_hit_points bits differ"
    p = synth.collect_hit_points_gpu(ref.density_atlas, ref.march, 8, 8)
    assert np.array_equal(p, sh[f"{kind}_dif"])


@pytest.mark.parametrize("kind", ["sphere", "box", "two"])
def test_full_pipeline_reproduces_reference_asset(kind):
    ref = asset(f"toy_{kind}")
    a = synth.make_asset(kind, SEEDS[kind], b=16, r=4, psh_resolution=16, diffuse_levels=3,
                         diffuse_table=2 ** 10, shell_cameras_n=12, shell_image_size=16,
                         diffuse_shell_cameras=8, diffuse_shell_image=8)
    assert np.array_equal(a.psh.offsets, ref.psh.offsets)
    assert np.array_equal(a.diffuse_atlas.index, ref.diffuse_atlas.index)
    err = np.abs(a.diffuse_atlas.cubes - ref.diffuse_atlas.cubes).max()
    assert err <= 2e-6, err     # fp32 MLP (sequential FMA) vs OpenBLAS sgemm
