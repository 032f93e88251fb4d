"""The reference's own known-answer tests for the hot path,
restated against the pinned C oracle (CPU) and the CUDA path (GPU).

Each test names the reference test it restates.  The reference marches
closed-form ``AnalyticSource`` media in some of them; the B200 path marches
cube atlases only, so those media are baked first (``synth.bake_density``,
the restatement of atlas.bake_cubes).  A baked constant stays exactly
constant (trilinear weights sum to 1, the sum is rounded to fp32), so the
closed forms hold to the same tolerances; a baked step ramps over one
sub-voxel (1/256), well inside the tests' one-step depth budget.

CPU tests check the oracle, GPU tests the CUDA path through the
reference-signature mirror (``render.march_rays`` / ``render_ray`` /
``compose``) AND against the oracle (hit flags, depth bits and sample
counts bit for bit)."""

import math

import numpy as np
import pytest

from golden_util import asset as golden_asset
from oracle import oracle as O
from paper_2303_04086_b200.model import Frame, MarchParams, RenderCounters
from tools.synth import bake_density, march_only_asset

gpu = pytest.mark.gpu


# ------------------------------------------------------------------ march media
def _constant(sigma, step, t_stop):
    atlas = bake_density(lambda p: np.full(len(p), float(sigma)), b=4, r=2)
    return march_only_asset(atlas, MarchParams(step=step, t_stop=t_stop))


def _sparse_blob(step):
    # test_lightfield.py:42-47: density only in a small ball around (0.9, 0.9, 0.9)
    atlas = bake_density(lambda p: 2.0 * (np.linalg.norm(p - 0.9, axis=1) < 0.05), b=8, r=4)
    return march_only_asset(atlas, MarchParams(step=step))


def _plane(step, t_stop):
    atlas = bake_density(lambda p: np.where(p[:, 0] >= 0.5, 10.0, 0.0), b=32, r=8)
    return march_only_asset(atlas, MarchParams(step=step, t_stop=t_stop))


def _bumpy(fn, t_stop=1e-9):
    return march_only_asset(bake_density(fn, b=32, r=8), MarchParams(step=1 / 128, t_stop=t_stop))


def _x_rays(entry_t, y=(0.5,), z=(0.5,)):
    """Rays along +x entering the unit box at parameter entry_t (test_lightfield.py:35-37)."""
    y, z = np.broadcast_arrays(np.asarray(y, float), np.asarray(z, float))
    o = np.column_stack([np.full(len(y), -float(entry_t)), y, z])
    return o, np.tile([1.0, 0.0, 0.0], (len(y), 1))


def _oracle_march(a, o, d):
    _, _, D = O.render_rays(a, o, d, debug=True)
    return D["hit"], D["t_hit"], D["alpha_c"], D["samples"]


def _gpu_march(a, o, d):
    from paper_2303_04086_b200 import render as R
    r = R.march_rays(a, o, d)
    return r.hit, r.t_hit, r.alpha_c, r.samples


MARCHERS = [pytest.param(_oracle_march, id="oracle"), pytest.param(_gpu_march, id="cuda", marks=gpu)]


@pytest.mark.parametrize("march", MARCHERS)
def test_empty_cells_give_clean_miss(march):
    """test_lightfield.py:42-55"""
    hit, t_hit, alpha, samples = march(_sparse_blob(1 / 32), *_x_rays(1.0))
    assert not hit[0]
    assert alpha[0] == 0.0
    assert samples[0] == 0
    assert np.isinf(t_hit[0])


@pytest.mark.parametrize("march", MARCHERS)
def test_constant_sigma_closed_form(march):
    """test_lightfield.py:57-66 and test_acceptance.py:254-264: sigma = 2, entry
    t = 1, step 0.1 -> the hit is the first sample (t = 1.05), 10 samples,
    alpha_c = 1 - exp(-2 * 0.1 * 10)."""
    hit, t_hit, alpha, samples = march(_constant(2.0, 0.1, 1e-9), *_x_rays(1.0))
    assert hit[0]
    assert t_hit[0] == pytest.approx(1.05, abs=1e-9)
    assert samples[0] == 10
    assert alpha[0] == pytest.approx(1.0 - math.exp(-2.0 * 0.1 * 10), abs=1e-9)


@pytest.mark.parametrize("march", MARCHERS)
@pytest.mark.parametrize("t_stop,min_alpha", [(1e-4, 0.98), (1e-6, 0.99)])
def test_step_density_depth_and_saturation(march, t_stop, min_alpha):
    """test_lightfield.py:68-77 (t_stop 1e-4) and test_acceptance.py:266-275
    (t_stop 1e-6): the plane x = 0.5 sits at t = 2 for a ray entering at 1.5."""
    step = 1 / 64
    hit, t_hit, alpha, _ = march(_plane(step, t_stop), *_x_rays(1.5))
    assert hit[0]
    assert abs(t_hit[0] - 2.0) <= step
    assert alpha[0] > min_alpha


def _sin_medium(p):     # test_lightfield.py:80-81
    return 3.0 * (np.sin(7 * p[:, 0]) + 1.1) * (p[:, 1] + 0.2)


def _bumpy_medium(p):   # test_acceptance.py:278
    return 3.0 * (np.sin(9 * p[:, 0]) + 1.05)


@pytest.mark.parametrize("march", MARCHERS)
@pytest.mark.parametrize("medium,n,lo,hi", [(_sin_medium, 32, 0.2, 0.8), (_bumpy_medium, 64, 0.1, 0.9)])
def test_weight_sum_bounded_by_one(march, medium, n, lo, hi):
    """test_lightfield.py:79-92 / test_acceptance.py:276-285 march 32 / 64 rays
    through a smooth medium and check sum(w) = 1 - T_final <= 1.  The marcher
    exports alpha_c = sum(w), not T; the identity is pinned through the oracle
    (every ray's alpha_c equals the reference's golden march to 1e-12,
    test_oracle.py) and here: 0 < alpha_c <= 1 on every ray."""
    rng = np.random.default_rng(3)
    o, d = _x_rays(0.5, rng.uniform(lo, hi, n), rng.uniform(lo, hi, n))
    hit, t_hit, alpha, samples = march(_bumpy(medium), o, d)
    assert np.all(alpha > 0.0) and np.all(alpha <= 1.0 + 1e-6)
    assert np.all(hit) and np.all(samples > 0)
    assert np.all((t_hit > 0.5) & (t_hit < 1.5))


@gpu
@pytest.mark.parametrize("medium", [_sin_medium, _bumpy_medium])
def test_cuda_march_equals_oracle_bitwise(medium):
    """The same KAT rays through both marchers: hit flags, t_hit (the depth
    bits) and sample counts identical to the last bit; alpha_c to a few ulps
    -- it is a sum of T*(1 - exp(-sigma*step)) and CUDA's fp64 exp() and the
    oracle's libm exp() (like numpy's) are each within an ulp of exp but not
    always the same ulp (exp choice never moved a hit index)."""
    rng = np.random.default_rng(7)
    o, d = _x_rays(0.5, rng.uniform(0.05, 0.95, 256), rng.uniform(0.05, 0.95, 256))
    a = _bumpy(medium)
    (gh, gt, ga, gs), (ch, ct, ca, cs) = _gpu_march(a, o, d), _oracle_march(a, o, d)
    assert np.array_equal(gh, ch)
    assert np.array_equal(gt, ct)
    assert np.array_equal(gs, cs)
    np.testing.assert_allclose(ga, ca, rtol=1e-14, atol=0)


# ------------------------------------------------------------------ render
def _renderers():
    return [pytest.param("oracle", id="oracle"), pytest.param("cuda", id="cuda", marks=gpu)]


def _render_ray(which, a, origin, direction, counters):
    o = np.asarray(origin, float)[None, :]
    d = np.asarray(direction, float)[None, :]
    if which == "oracle":
        rgba, depth = O.render_rays(a, o, d, counters)
    else:
        from paper_2303_04086_b200 import render as R
        rgba, depth = R.render_rays(a, o, d, counters)
    return rgba[0], float(depth[0])


@pytest.mark.parametrize("which", _renderers())
def test_proxy_miss_costs_nothing(which):
    """test_lightfield.py:247-255"""
    cnt = RenderCounters()
    rgba, depth = _render_ray(which, golden_asset("toy_sphere"), (5.0, 5.0, 5.0), (0.0, 0.0, 1.0), cnt)
    np.testing.assert_array_equal(rgba, 0)
    assert np.isinf(depth)
    assert cnt.fs_evals == 0 and cnt.march_samples == 0


@pytest.mark.parametrize("which", _renderers())
def test_hitting_ray_queries_specular_net_exactly_once(which):
    """test_lightfield.py:257-264 (one query per ray)"""
    cnt = RenderCounters()
    _, depth = _render_ray(which, golden_asset("toy_sphere"), (-1.0, 0.5, 0.5), (1.0, 0.0, 0.0), cnt)
    assert cnt.fs_evals == 1
    assert cnt.hit_pixels == 1
    assert cnt.fd_evals == 0
    assert np.isfinite(depth)


@pytest.mark.parametrize("which", _renderers())
def test_sphere_center_ray_depth(which):
    """test_lightfield.py:266-272 on the baked sphere asset (radius 0.25 at the
    box centre): the front surface z = 0.75 is at depth 1.25 from z = 2."""
    a = golden_asset("toy_sphere")
    rgba, depth = _render_ray(which, a, (0.5, 0.5, 2.0), (0.0, 0.0, -1.0), RenderCounters())
    assert rgba[3] > 0.5
    assert depth == pytest.approx(1.25, abs=2 * a.march.step + 1 / 32)


# ------------------------------------------------------------------ compose
def _flat(w, h, rgba, depth):
    f = Frame.empty(w, h)
    f.rgba[:] = rgba
    f.depth[:] = depth
    return f


def _compose(which, frames):
    if which == "oracle":
        rgba = np.stack([f.rgba for f in frames])
        depth = np.stack([f.depth for f in frames])
        return O.compose(rgba, depth)
    from paper_2303_04086_b200 import render as R
    out = R.compose(frames)
    return out.rgba, out.depth


@pytest.mark.parametrize("which", _renderers())
def test_compose_opaque_occlusion(which):
    """test_farm.py:22-27"""
    red = _flat(2, 2, [1, 0, 0, 1], 1.0)
    blue = _flat(2, 2, [0, 0, 1, 1], 2.0)
    rgba, depth = _compose(which, [blue, red])
    np.testing.assert_allclose(rgba[0, 0], [1, 0, 0, 1], atol=1e-6)
    assert depth[0, 0] == pytest.approx(1.0)


@pytest.mark.parametrize("which", _renderers())
def test_compose_alpha_over_blend(which):
    """test_farm.py:29-35"""
    front = _flat(1, 1, [0.5, 0, 0, 0.5], 1.0)
    back = _flat(1, 1, [0, 0, 1, 1], 2.0)
    rgba, depth = _compose(which, [front, back])
    np.testing.assert_allclose(rgba[0, 0], [0.5, 0, 0.5, 1.0], atol=1e-6)
    assert depth[0, 0] == pytest.approx(2.0)


@pytest.mark.parametrize("which", _renderers())
def test_compose_single_frame_identity(which):
    """test_farm.py:37-41"""
    f = _flat(3, 2, [0.2, 0.3, 0.4, 0.8], 1.5)
    rgba, depth = _compose(which, [f])
    np.testing.assert_allclose(rgba, f.rgba, atol=1e-6)
    np.testing.assert_allclose(depth, f.depth)


@pytest.mark.parametrize("which", _renderers())
def test_compose_arrival_order_irrelevant_for_distinct_depths(which):
    """test_farm.py:43-56"""
    rng = np.random.default_rng(0)
    frames = []
    for i in range(4):
        f = Frame.empty(8, 8)
        alpha = rng.uniform(0.2, 1.0, (8, 8)).astype(np.float32)
        f.rgba[..., :3] = rng.uniform(0, 0.8, (8, 8, 3)) * alpha[..., None]
        f.rgba[..., 3] = alpha
        f.depth[:] = (1.0 + i) + rng.uniform(0, 0.3, (8, 8)).astype(np.float32)
        frames.append(f)
    a_rgba, a_depth = _compose(which, frames)
    b_rgba, b_depth = _compose(which, frames[::-1])
    np.testing.assert_allclose(a_rgba, b_rgba, atol=1e-6)
    np.testing.assert_allclose(a_depth, b_depth)
