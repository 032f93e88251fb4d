"""Golden vectors for the stage-2 training step, made by running the REFERENCE.

Test infrastructure (like make_golden.py; needs /root/reference).  Writes
``tests/golden/train.npz``:

* ``grad_*``: one exact backward (lightfield.shade_batch(..., want_cache,
  force_live_diffuse) + shade_backward, lightfield.py:267-397) on a fixed
  batch of hit rays of the toy sphere (the march run by the reference),
  with the batch's targets, losses and predictions;
* ``train_*``: three steps of lightfield.train_light_field (lightfield.py:
  654-749: sample_rays -> march -> shade -> loss -> shade_backward ->
  adam_step -> update_error_map) from toy_sphere on two 32x32 training
  views, default_rng(11), batch 512: the per-step losses and every trained
  array afterwards.

Run: python tests/golden/make_train_golden.py
"""

from __future__ import annotations

import copy
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (puts the reference on sys.path)

from radfarm import assetio  # noqa: E402
from radfarm.core import aabb_intersect_batch, camera_dirs  # noqa: E402
from radfarm.lightfield import (LightFieldTrainConfig, march_rays, shade_backward, shade_batch,  # noqa: E402
                                train_light_field)
from radfarm.scenes import orbit_camera  # noqa: E402


def load_toy():
    import gzip
    import tempfile
    raw = gzip.decompress(open(os.path.join(HERE, "assets", "toy_sphere.nolf.gz"), "rb").read())
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.nolf")
        open(p, "wb").write(raw)
        return assetio.read_asset(p)


def views():
    cams = [orbit_camera(0.8, 0.3, radius=2.0, size=32), orbit_camera(2.2, -0.2, radius=1.8, size=32)]
    rng = np.random.default_rng(5)
    images = rng.uniform(0.0, 1.0, (2, 32, 32, 3)).astype(np.float32)
    alphas = rng.uniform(0.0, 1.0, (2, 32, 32)).astype(np.float32)
    return cams, images, alphas


def main():
    asset = load_toy()
    out = {}
    # ---- one backward on a fixed batch of hit rays
    cam = orbit_camera(1.1, 0.4, radius=2.0, size=48)
    px, py = np.meshgrid(np.arange(48), np.arange(48))
    dirs = camera_dirs(cam, px.reshape(-1), py.reshape(-1))
    origins = np.broadcast_to(cam.position, dirs.shape).copy()
    tn, tf, bh = aabb_intersect_batch(origins, dirs, asset.proxy, 0.0, np.inf)
    res = march_rays(asset.density_source(), origins, dirs, np.where(bh, tn, 1.0), np.where(bh, tf, 0.0),
                     asset.march)
    hit = res.hit
    rng = np.random.default_rng(3)
    rgb = rng.uniform(0, 1, (len(dirs), 3)).astype(np.float32)
    alpha = rng.uniform(0, 1, len(dirs)).astype(np.float32)
    b = len(dirs)
    c, a, extras = shade_batch(asset, res.p_h[hit], res.alpha_c[hit], dirs[hit], want_cache=True,
                               force_live_diffuse=True)
    err_c = c - rgb[hit]
    err_a = a - alpha[hit]
    grads = shade_backward(asset, extras["cache"], 2.0 * err_c / b, 2.0 * err_a / b)
    out.update(grad_p_h=res.p_h[hit], grad_alpha_c=res.alpha_c[hit], grad_dirs=dirs[hit],
               grad_rgb=rgb[hit], grad_alpha=alpha[hit], grad_b=np.array(b), grad_pred_c=c, grad_pred_a=a,
               grad_loss=(err_c ** 2).sum(axis=1) + err_a ** 2, grad_psh=grads["psh_features"])
    for i, (w, bb) in enumerate(zip(*grads["fs"])):
        out[f"grad_fs_w{i}"], out[f"grad_fs_b{i}"] = w, bb
    for i, (w, bb) in enumerate(zip(*grads["fd"])):
        out[f"grad_fd_w{i}"], out[f"grad_fd_b{i}"] = w, bb
    for i, g in enumerate(grads["diffuse_features"]):
        out[f"grad_ed_{i}"] = g
    print("backward batch: hits", int(hit.sum()))
    # ---- three steps of train_light_field
    cams, images, alphas = views()
    tasset = copy.deepcopy(asset)
    cfg = LightFieldTrainConfig(steps=3, batch_rays=512)
    losses = train_light_field(tasset, images, alphas, cams, cfg, np.random.default_rng(11))
    out.update(train_losses=np.array(losses), train_images=images, train_alphas=alphas,
               train_poses=np.stack([c.pose for c in cams]), train_psh=tasset.psh_features)
    for i, p in enumerate(tasset.specular_mlp.parameters()):
        out[f"train_fs_{i}"] = p
    for i, p in enumerate(tasset.diffuse_mlp.parameters()):
        out[f"train_fd_{i}"] = p
    for i, f in enumerate(tasset.diffuse_features):
        out[f"train_ed_{i}"] = f
    print("train losses", losses)
    MG.savez("train.npz", out)
    print("written", os.path.getsize(os.path.join(HERE, "train.npz")), "bytes")


if __name__ == "__main__":
    main()
