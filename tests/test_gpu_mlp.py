"""Specular MLP kernels vs a plain PyTorch fp32 reference of the same op
(neural.py:89-108 forward with heads sigmoid x3 + identity), and full renders
with the tcgen05 bf16 MLP vs the reference goldens at the north-star bf16
tolerance (2/255)."""

import numpy as np
import pytest

from golden_util import asset, camera, case_asset, load
from paper_2303_04086_b200 import render as R
from paper_2303_04086_b200.model import RayRange

pytestmark = pytest.mark.gpu
BF16_TOL = 2.0 / 255.0


def torch_mlp(m, x):
    import torch
    h = torch.as_tensor(x, dtype=torch.float32)
    n = len(m.weights)
    for i, (w, b) in enumerate(zip(m.weights, m.biases)):
        h = h @ torch.as_tensor(w).T + torch.as_tensor(b)
        if i < n - 1:
            h = torch.relu(h)
    out = h.clone()
    out[:, :3] = torch.sigmoid(h[:, :3])
    return out.numpy()


def inputs(n, rng, scale=1.0):
    es = rng.uniform(-1e-4, 1e-4, (n, 2)) * scale
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    from oracle.oracle import lib  # noqa: F401  (oracle only for SH below)
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    sh = np.stack([np.full(n, 0.28209479177387814), -0.4886025119029199 * y, 0.4886025119029199 * z,
                   -0.4886025119029199 * x, 1.0925484305920792 * x * y, -1.0925484305920792 * y * z,
                   0.31539156525252005 * (2 * z * z - x * x - y * y), -1.0925484305920792 * x * z,
                   0.5462742152960396 * (x * x - y * y), -0.5900435899266435 * y * (3 * x * x - y * y),
                   2.890611442640554 * x * y * z, -0.4570457994644658 * y * (4 * z * z - x * x - y * y),
                   0.3731763325901154 * z * (2 * z * z - 3 * x * x - 3 * y * y),
                   -0.4570457994644658 * x * (4 * z * z - x * x - y * y), 1.445305721320277 * z * (x * x - y * y),
                   -0.5900435899266435 * x * (x * x - 3 * y * y)], axis=1)
    ac = rng.uniform(1e-4, 1 - 1e-4, (n, 1))
    return np.concatenate([es, sh, ac], axis=1).astype(np.float32)


@pytest.mark.parametrize("n", [1, 127, 128, 1000, 20000])
def test_mlp_fp32_and_bf16_vs_torch(n):
    a = asset("toy_sphere")
    x = inputs(n, np.random.default_rng(n))
    ref = torch_mlp(a.specular_mlp, x)
    f32 = R.mlp_eval(a, x, "fp32")
    assert np.abs(f32 - ref).max() <= 1e-5
    bf = R.mlp_eval(a, x, "bf16")
    assert np.abs(bf[:, :3] - ref[:, :3]).max() <= BF16_TOL
    assert np.abs(bf[:, 3] - ref[:, 3]).max() <= 0.02 * (1 + np.abs(ref[:, 3]).max())


def test_mlp_bf16_scaled_features():
    """Features x1e3 (SURVEY.md 8(d) bf16 stress fixture)."""
    a = asset("toy_sphere")
    x = inputs(4096, np.random.default_rng(7), scale=1e3)
    ref = torch_mlp(a.specular_mlp, x)
    bf = R.mlp_eval(a, x, "bf16")
    assert np.abs(bf[:, :3] - ref[:, :3]).max() <= BF16_TOL


@pytest.mark.parametrize("case", ["sphere_far", "sphere_close", "sphere_inside", "box_far", "two_far",
                                  "sphere_xform", "abl_opacity", "abl_tint", "abl_hit_point",
                                  "abl_diffuse_color", "norefine_far"])
def test_render_bf16_vs_reference(case):
    g = load(f"render_{case}.npz")
    a = case_asset(case, g)
    cam = camera(g)
    x0, y0, x1, y1 = (int(v) for v in g["rect"])
    R.set_mlp_mode("bf16")
    try:
        tile, _ = R.render_range(a, RayRange(cam, x0, y0, x1, y1))
    finally:
        R.set_mlp_mode("fp32")
    rgba, depth = tile.rgba.reshape(-1, 4), tile.depth.reshape(-1)
    fin = np.isfinite(g["depth"])
    assert np.array_equal(np.isfinite(depth), fin)
    assert np.array_equal(depth[fin], g["depth"][fin])
    err = np.abs(rgba - g["rgba"]).max()
    assert err <= BF16_TOL, err
    print(case, "bf16 max err", err)


def test_fused_scene_bf16_vs_reference():
    g = load("scene.npz")
    names = {"sphere": "toy_sphere", "box": "toy_box", "two": "toy_two"}
    scene = [(asset(names[str(n)]), tr) for n, tr in zip(g["names"], g["transforms"])]
    R.set_mlp_mode("bf16")
    try:
        out = R.render_scene(scene, camera(g))
    finally:
        R.set_mlp_mode("fp32")
    fin = np.isfinite(g["depth"])
    assert np.array_equal(np.isfinite(out.depth), fin)
    assert np.abs(out.rgba - g["rgba"]).max() <= BF16_TOL
