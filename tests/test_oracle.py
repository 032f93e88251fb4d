"""The C oracle (oracle/nolf_oracle.c) against the reference's own outputs.

This pins the checker: every integer the north star requires bit-exact (box
hit, march hit, hit sample index i*, active sample counts, PSH slot
addresses) and the f64 ray setup must equal the reference's golden vectors
exactly; pixels must agree to 1e-6 (fp32 MLP vs OpenBLAS sgemm ordering)."""

import numpy as np
import pytest

from golden_util import camera, case_asset, load, render_cases
from oracle import oracle as O
from paper_2303_04086_b200.model import RenderCounters

CASES = render_cases()


@pytest.mark.parametrize("case", CASES)
def test_render_case_matches_reference(case):
    g = load(f"render_{case}.npz")
    a = case_asset(case, g)
    cam = camera(g)
    dirs = O.camera_dirs(cam, *_pixels(g))
    assert np.array_equal(dirs, g["dirs"]), "camera_dirs bits differ from core.camera_dirs"
    origins = np.broadcast_to(np.asarray(g["origin"]), dirs.shape)
    cnt = RenderCounters()
    rgba, depth, D = O.render_rays(a, origins, dirs, cnt, debug=True)
    _check(g, rgba, depth, D, cnt)
    # fused rect path (renderer.render_range) gives the same pixels
    x0, y0, x1, y1 = g["rect"]
    r2, d2 = O.render_rect(a, cam, (x0, y0, x1, y1))
    assert np.array_equal(r2.reshape(-1, 4), rgba)
    assert np.array_equal(d2.reshape(-1), depth)


@pytest.mark.parametrize("name", ["rays_sphere", "rays_sphere_xform"])
def test_arbitrary_rays_match_reference(name):
    g = load(f"{name}.npz")
    a = case_asset("sphere", g)
    cnt = RenderCounters()
    rgba, depth, D = O.render_rays(a, g["origins"], g["dirs"], cnt, debug=True)
    _check(g, rgba, depth, D, cnt)


def _pixels(g):
    x0, y0, x1, y1 = g["rect"]
    px, py = np.meshgrid(np.arange(x0, x1), np.arange(y0, y1))
    return px.reshape(-1).astype(np.float64), py.reshape(-1).astype(np.float64)


def _check(g, rgba, depth, D, cnt):
    assert np.array_equal(D["o_obj"], g["o_obj"])
    assert np.array_equal(D["d_obj"], g["d_obj"])
    assert np.array_equal(D["boxhit"], g["boxhit"])
    bh = g["boxhit"]
    assert np.array_equal(D["t_near"][bh], g["t_near"][bh])
    assert np.array_equal(D["t_far"][bh], g["t_far"][bh])
    assert np.array_equal(D["hit"], g["hit"])
    assert np.array_equal(D["istar"], g["istar"])
    assert np.array_equal(D["samples"], g["samples"])
    assert np.array_equal(D["t_hit"], g["t_hit"])
    np.testing.assert_allclose(D["alpha_c"], g["alpha_c"], rtol=0, atol=1e-12)
    hr = g["hit_rows"]
    assert np.array_equal(D["p_h"][hr], g["p_h"][hr])
    if "psh_slots" in g:
        assert np.array_equal(D["slots"][hr], g["psh_slots"]), "PSH addresses differ"
        np.testing.assert_allclose(D["es"][hr], g["es"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(D["fs_out"][hr], g["fs_out"], rtol=0, atol=2e-6)
        if g["wiring"][4]:  # use_diffuse_color: the diffuse stage actually runs
            np.testing.assert_allclose(D["diffuse"][hr], g["diffuse"], rtol=0, atol=2e-6)
    np.testing.assert_allclose(rgba, g["rgba"], rtol=0, atol=1e-6)
    fin = np.isfinite(g["depth"])
    assert np.array_equal(np.isfinite(depth), fin)
    np.testing.assert_array_equal(depth[fin], g["depth"][fin])
    assert [cnt.fs_evals, cnt.fd_evals, cnt.hit_pixels, cnt.march_samples] == g["counters"].tolist()


def test_compose_matches_reference():
    g = load("compose.npz")
    n = len([k for k in g if k.startswith("in_rgba_")])
    for i in range(n):
        rgba, depth = O.compose(g[f"in_rgba_{i}"], g[f"in_depth_{i}"])
        np.testing.assert_array_equal(rgba, g[f"out_rgba_{i}"])
        np.testing.assert_array_equal(depth, g[f"out_depth_{i}"])


def test_scene_compose_matches_reference():
    g = load("scene.npz")
    rgba, depth = O.compose(g["frame_rgba"], g["frame_depth"])
    np.testing.assert_array_equal(rgba, g["rgba"])
    np.testing.assert_array_equal(depth, g["depth"])


def test_scene_frames_match_reference():
    from golden_util import asset
    g = load("scene.npz")
    cam = camera(g)
    names = {"sphere": "toy_sphere", "box": "toy_box", "two": "toy_two"}
    for k, (nm, tr) in enumerate(zip(g["names"], g["transforms"])):
        rgba, depth = O.render_rect(asset(names[str(nm)]), cam, transform=tr)
        np.testing.assert_allclose(rgba, g["frame_rgba"][k], rtol=0, atol=1e-6)
        fin = np.isfinite(g["frame_depth"][k])
        assert np.array_equal(np.isfinite(depth), fin)
        np.testing.assert_array_equal(depth[fin], g["frame_depth"][k][fin])


def test_encode_frame_restatement_matches_reference():
    """protocol.encode_frame RAW (protocol.py:256-266) goldens, incl. .5 ties,
    clipping, the depth_far clamp and inf depths."""
    g = load("encode.npz")
    r8, d16 = O.encode_frame(g["syn_rgba"], g["syn_depth"])
    np.testing.assert_array_equal(r8, g["syn_rgba8"])
    np.testing.assert_array_equal(d16, g["syn_depth16"])
    s = load("scene.npz")
    r8, d16 = O.encode_frame(s["rgba"], s["depth"])
    np.testing.assert_array_equal(r8, g["scene_rgba8"])
    np.testing.assert_array_equal(d16, g["scene_depth16"])


def test_compose_any_number_of_frames():
    """farm.compose takes any K (farm.py:129-172): 100 frames with depth
    ties and inf / zero-alpha layers vs a direct numpy restatement."""
    rng = np.random.default_rng(9)
    K, P = 100, 64
    a = rng.uniform(0, 1, (K, P)).astype(np.float32)
    a[rng.uniform(size=(K, P)) < 0.3] = 0
    rgba = np.concatenate([rng.uniform(0, 1, (K, P, 3)).astype(np.float32) * a[..., None], a[..., None]], -1)
    depth = np.where(a > 0, rng.choice([1.0, 1.5, 2.0], (K, P)), np.inf).astype(np.float32)
    o, d = O.compose(rgba, depth)
    for p in range(P):
        order = np.argsort(depth[:, p], kind="stable")
        oc, T, od = np.zeros(3), 1.0, np.float32(np.inf)
        for k in order:
            oc += T * rgba[k, p, :3].astype(np.float64)
            if np.isinf(od) and rgba[k, p, 3] > np.float32(0.5):
                od = depth[k, p]
            T *= np.float64(np.float32(1.0) - rgba[k, p, 3])
        want = np.concatenate([np.clip(oc, 0, 1), [np.clip(1 - T, 0, 1)]]).astype(np.float32)
        if want[3] <= 0:
            want[:] = 0
            od = np.float32(np.inf)
        np.testing.assert_array_equal(o[p], want)
        assert d[p] == od
