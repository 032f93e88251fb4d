"""Stage-2 training on the GPU (train.py: k_train_shade + k_adam) against
the reference (tests/golden/train.npz, made by make_train_golden.py).

Bars: the forward (prediction, per-ray loss) to fp32-MLP rounding; every
gradient of shade_backward (lightfield.py:358-397: specular / diffuse MLP
weights and biases, psh_backward and hashgrid_backward scatters) within
1e-4 of its scale (fp32 GEMM order vs OpenBLAS sgemm); three steps of
train_light_field (lightfield.py:654-749, same rng) give the reference's
losses and trained arrays (Adam's first steps move each weight by ~lr, so
a gradient whose sign differs between summation orders may land 2 lr away:
those elements are bounded and counted)."""

import copy

import numpy as np
import pytest

from golden_util import asset, load
from paper_2303_04086_b200 import render as R
from paper_2303_04086_b200.model import orbit_camera

pytestmark = pytest.mark.gpu


def _close(got, want, rel=1e-4, what=""):
    scale = max(float(np.abs(want).max()), 1e-30)
    err = float(np.abs(np.asarray(got, np.float64) - want).max())
    assert err <= rel * scale, f"{what}: max |err| {err:.3g} vs scale {scale:.3g}"


def test_shade_backward_gradients_match_reference():
    from paper_2303_04086_b200.train import GpuTrainer
    g = load("train.npz")
    a = copy.deepcopy(asset("toy_sphere"))
    tr = GpuTrainer(a)
    pred, loss = tr.shade_step(g["grad_p_h"], g["grad_alpha_c"], g["grad_dirs"], g["grad_rgb"], g["grad_alpha"],
                               int(g["grad_b"]))
    _close(pred[:, :3], g["grad_pred_c"], 1e-5, "pred c")
    _close(pred[:, 3], g["grad_pred_a"], 1e-5, "pred alpha")
    _close(loss, g["grad_loss"], 1e-5, "loss")
    gr = tr.gradients()
    names = ["psh"] + [f"fs_{k}{i}" for i in range(3) for k in ("w", "b")] + \
            [f"fd_{k}{i}" for i in range(2) for k in ("w", "b")]
    order = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10]   # tensors in GpuTrainer order: psh, fs w0 b0 w1 b1 w2 b2, fd w0 b0 w1 b1
    keys = ["grad_psh", "grad_fs_w0", "grad_fs_b0", "grad_fs_w1", "grad_fs_b1", "grad_fs_w2", "grad_fs_b2",
            "grad_fd_w0", "grad_fd_b0", "grad_fd_w1", "grad_fd_b1"]
    for i, k in zip(order, keys):
        _close(gr[i], g[k], 1e-4, k)
    levels = len([k for k in g if k.startswith("grad_ed_")])
    for l in range(levels):
        _close(gr[11 + l], g[f"grad_ed_{l}"], 1e-4, f"grad_ed_{l}")
    assert np.abs(g["grad_psh"]).max() > 0 and np.abs(g["grad_fs_w0"]).max() > 0


def test_train_light_field_matches_reference():
    from paper_2303_04086_b200.train import train_light_field
    from paper_2303_04086_b200.model import Aabb  # noqa: F401
    g = load("train.npz")
    a = copy.deepcopy(asset("toy_sphere"))
    cams = [orbit_camera(0.8, 0.3, radius=2.0, size=32), orbit_camera(2.2, -0.2, radius=1.8, size=32)]
    for c, p in zip(cams, g["train_poses"]):
        assert np.array_equal(c.pose, p)            # the golden's training views

    class Cfg:
        steps, batch_rays, lr_features, lr_mlp = 3, 512, 1e-2, 1e-3
        error_cell, error_floor, error_rho = 8, 1e-3, 0.1
    losses = train_light_field(a, g["train_images"], g["train_alphas"], cams, Cfg, np.random.default_rng(11))
    np.testing.assert_allclose(losses, g["train_losses"], rtol=1e-5)
    pairs = [(a.psh_features, g["train_psh"], 1e-2)]
    pairs += [(p, g[f"train_fs_{i}"], 1e-3) for i, p in enumerate(a.specular_mlp.parameters())]
    pairs += [(p, g[f"train_fd_{i}"], 1e-3) for i, p in enumerate(a.diffuse_mlp.parameters())]
    pairs += [(f, g[f"train_ed_{i}"], 1e-2) for i, f in enumerate(a.diffuse_features)]
    moved = 0
    for got, want, lr in pairs:
        d = np.abs(np.asarray(got, np.float64) - want)
        assert d.max() <= 2 * 3 * lr + 1e-6, d.max()          # never more than a full sign flip per step
        off = d > 1e-5 * max(float(np.abs(want).max()), 1e-6)
        assert off.mean() <= 0.01, f"{off.mean():.3%} of the elements differ"
        moved += int(off.sum())
    print("elements off by a sign flip:", moved)
