"""Stage-2 training of an i-NOLF asset on the GPU.

``train_light_field`` keeps the reference's signature and loop
(lightfield.py:654-749) with every per-ray stage on the B200:

  sample_rays / ErrorMap / update_error_map   neural.py:180-272 (host: the
                                              batch draw must consume the
                                              caller's rng exactly as the
                                              reference does)
  aabb + march_rays (frozen density)          nolf_march_rays
  shade_batch(force_live_diffuse) + loss +    nolf_train_shade (k_train_shade:
  shade_backward                              forward + backward fused, MLP
                                              grads reduced per CTA, feature
                                              grads scattered)
  adam_step per parameter group               nolf_adam (k_adam: the
                                              reference's f32 update)

``GpuTrainer`` owns the trainable tensors on the device in the reference's
layouts (one flat f32 buffer + an f64 gradient buffer + Adam moments) and
writes them back into the asset's arrays with ``export()``.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C
import numpy as np

from . import _native as N
from . import errors

N_OFFSETS = 27            # NOLF_TRAIN_OFFSETS
_TP_PSH, _TP_FS, _TP_FD, _TP_HG = 0, 1, 7, 11


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------ host side of the loop (neural.py:180-272)
@dataclass
class TrainBatch:
    origins: np.ndarray
    dirs: np.ndarray
    rgb: np.ndarray
    alpha: np.ndarray
    cells: np.ndarray

    def __len__(self):
        return len(self.origins)


@dataclass
class ErrorMap:
    """Per-image low-resolution sampling weights (neural.py:194-215)."""
    weights: np.ndarray
    cell_size: int = 8
    floor: float = 1e-3
    rho: float = 0.1

    @classmethod
    def uniform(cls, n_images, height, width, cell_size=8, floor=1e-3, rho=0.1):
        cy = (height + cell_size - 1) // cell_size
        cx = (width + cell_size - 1) // cell_size
        return cls(np.ones((n_images, cy, cx), dtype=np.float64), cell_size, floor, rho)


def sample_rays(error_map, images, alphas, cameras, n, rng) -> TrainBatch:
    """neural.py:218-254: cell by weighted choice, pixel uniform in the cell."""
    from .model import Camera  # noqa: F401  (cameras are reference-compatible objects)
    if n < 1:
        raise errors.DomainError("batch size must be >= 1")
    if len(cameras) == 0:
        raise errors.DomainError("empty training set")
    w = error_map.weights.reshape(-1)
    p = w / w.sum()
    cells = rng.choice(len(w), size=n, p=p)
    n_img, cy, cx = error_map.weights.shape
    img = cells // (cy * cx)
    rest = cells % (cy * cx)
    cell_y, cell_x = rest // cx, rest % cx
    height, width = images.shape[1:3]
    cs = error_map.cell_size
    py = np.minimum(cell_y * cs + rng.integers(0, cs, size=n), height - 1)
    px = np.minimum(cell_x * cs + rng.integers(0, cs, size=n), width - 1)
    origins = np.empty((n, 3))
    dirs = np.empty((n, 3))
    for i in np.unique(img):
        sel = img == i
        cam = cameras[i]
        dirs[sel] = _camera_dirs(cam, px[sel], py[sel])
        origins[sel] = cam.position
    return TrainBatch(origins, dirs, images[img, py, px].astype(np.float32),
                      alphas[img, py, px].astype(np.float32), cells)


def _camera_dirs(cam, px, py):
    """core.camera_dirs (core.py:162-170)."""
    u = (np.asarray(px, np.float64) + 0.5 - cam.cx) / cam.fx
    v = -(np.asarray(py, np.float64) + 0.5 - cam.cy) / cam.fy
    d = np.stack([u, v, -np.ones_like(u)], axis=-1) @ np.asarray(cam.pose)[:3, :3].T
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def update_error_map(error_map, cells, losses) -> None:
    """neural.py:257-272: EMA of the mean per-cell ray loss, floored."""
    losses = np.asarray(losses, dtype=np.float64)
    if np.any(losses < 0):
        raise errors.DomainError("ray losses must be non-negative")
    sums = np.zeros(error_map.weights.size)
    counts = np.zeros(error_map.weights.size)
    np.add.at(sums, cells, losses)
    np.add.at(counts, cells, 1.0)
    touched = counts > 0
    flat = error_map.weights.reshape(-1)
    rho = error_map.rho
    flat[touched] = (1.0 - rho) * flat[touched] + rho * (sums[touched] / counts[touched])
    np.maximum(flat, error_map.floor, out=flat)


# ------------------------------------------------------------------ device side
class GpuTrainer:
    """The trainable tensors of an asset on the GPU plus their Adam state."""

    def __init__(self, asset, lr_features=1e-2, lr_mlp=1e-3, beta1=0.9, beta2=0.99, eps=1e-15):
        torch = _torch()
        from . import render as R
        self.asset = asset
        self.dev = R._device()
        self.handle = R.device_asset(asset).handle          # fixed tables (PSH addressing, hash grid)
        fs, fd = asset.specular_mlp, asset.diffuse_mlp
        if len(fs.weights) != 3 or fd is None or len(fd.weights) != 2:
            raise errors.ConfigError("GPU training needs a 3-layer specular and a 2-layer diffuse network")
        tensors = [asset.psh_features] + [fs.weights[0], fs.biases[0], fs.weights[1], fs.biases[1],
                                          fs.weights[2], fs.biases[2]] + \
                  [fd.weights[0], fd.biases[0], fd.weights[1], fd.biases[1]] + list(asset.diffuse_features)
        self.arrays = tensors
        offs, o = [], 0
        for a in tensors:
            offs.append(o)
            o += int(np.asarray(a).size)
        self.offsets = np.zeros(N_OFFSETS, np.int64)
        self.offsets[:len(offs)] = offs
        flat = np.concatenate([np.ascontiguousarray(a, np.float32).reshape(-1) for a in tensors])
        self.params = torch.from_numpy(flat).to(self.dev)
        self.grads = torch.zeros(o, dtype=torch.float64, device=self.dev)
        self.m = torch.zeros(o, dtype=torch.float32, device=self.dev)
        self.v = torch.zeros(o, dtype=torch.float32, device=self.dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # AdamState per group (lightfield.py:677-688): [first, last) float ranges, lr
        end = lambda i: offs[i + 1] if i + 1 < len(offs) else o   # noqa: E731
        self.groups = {"psh_features": (offs[_TP_PSH], end(_TP_PSH), lr_features),
                       "fs": (offs[_TP_FS], end(_TP_FS + 5), lr_mlp)}
        if asset.wiring.use_diffuse_color:
            self.groups["fd"] = (offs[_TP_FD], end(_TP_FD + 3), lr_mlp)
            self.groups["diffuse_features"] = (offs[_TP_HG], o, lr_features)
        self.steps = {k: 0 for k in self.groups}
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    def shade_step(self, p_h, alpha_c, dirs, rgb, alpha, batch: int):
        """Forward + loss + backward for the hit rays; grads are reset first.
        Returns (pred (n,4) f32, per-ray loss (n,) f64) host arrays."""
        torch = _torch()
        from . import render as R
        n = len(p_h)
        self.grads.zero_()
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(self.dev)   # noqa: E731
        ph, ac, dv = t(p_h, np.float64), t(alpha_c, np.float64), t(dirs, np.float64)
        tr, ta = t(rgb, np.float32), t(alpha, np.float32)
        pred = torch.empty((n, 4), dtype=torch.float32, device=self.dev)
        loss = torch.empty(n, dtype=torch.float64, device=self.dev)
        offs = (C.c_int64 * N_OFFSETS)(*self.offsets.tolist())
        N.check(N.lib().nolf_train_shade(self.handle, self.params.data_ptr(), offs, self.grads.data_ptr(), n,
                                         ph.data_ptr(), ac.data_ptr(), dv.data_ptr(), tr.data_ptr(), ta.data_ptr(),
                                         float(batch), pred.data_ptr(), loss.data_ptr(), self.flag.data_ptr(),
                                         R._stream_ptr()))
        return pred.cpu().numpy(), loss.cpu().numpy()

    def gradients(self) -> list:
        """The last step's gradients, as f32 arrays in the reference layouts."""
        g = self.grads.cpu().numpy().astype(np.float32)
        out, o = [], 0
        for a in self.arrays:
            n = int(np.asarray(a).size)
            out.append(g[o:o + n].reshape(np.asarray(a).shape))
            o += n
        return out

    def adam(self, groups=None):
        """adam_step (neural.py:162-177) on the named groups (all by default)."""
        from . import render as R
        for name in groups or list(self.groups):
            a, b, lr = self.groups[name]
            self.steps[name] += 1
            N.check(N.lib().nolf_adam(self.params.data_ptr() + 4 * a, self.grads.data_ptr() + 8 * a,
                                      self.m.data_ptr() + 4 * a, self.v.data_ptr() + 4 * a, b - a, lr,
                                      self.beta1, self.beta2, self.eps, self.steps[name], self.flag.data_ptr(),
                                      R._stream_ptr()))
        f = int(self.flag.item())
        if f & 2:
            raise errors.TrainingError("non-finite gradient")

    def export(self) -> None:
        """Write the trained tensors back into the asset's arrays (in place,
        like the reference) and drop the stale device copy."""
        from . import render as R
        flat = self.params.cpu().numpy()
        o = 0
        for a in self.arrays:
            n = int(a.size)
            a[...] = flat[o:o + n].reshape(a.shape)
            o += n
        R.invalidate()


def train_light_field(asset, images, alphas, cameras, config, rng, log=None):
    """lightfield.train_light_field (lightfield.py:654-749) with the per-ray
    work on the GPU; returns the per-step loss log and trains ``asset`` in
    place."""
    from . import render as R
    if config.steps == 0:
        return []
    n_img, height, width = images.shape[:3]
    emap = ErrorMap.uniform(n_img, height, width, cell_size=config.error_cell, floor=config.error_floor,
                            rho=config.error_rho)
    tr = GpuTrainer(asset, lr_features=config.lr_features, lr_mlp=config.lr_mlp)
    losses, initial, bad = [], None, 0
    for step in range(config.steps):
        batch = sample_rays(emap, images, alphas, cameras, config.batch_rays, rng)
        res = R.march_rays(asset, batch.origins, batch.dirs)          # slab vs the proxy + frozen march
        b = len(batch)
        pred_c = np.zeros((b, 3))
        pred_a = np.zeros(b)
        hit = res.hit
        ray_losses = None
        if np.any(hit):
            if asset.wiring.use_hit_point:
                p_h = res.p_h[hit]
            else:
                raise errors.ConfigError("GPU training needs use_hit_point wiring")
            pred, lh = tr.shade_step(p_h, res.alpha_c[hit], batch.dirs[hit], batch.rgb[hit], batch.alpha[hit], b)
            pred_c[hit] = pred[:, :3]
            pred_a[hit] = pred[:, 3]
        err_c = pred_c - batch.rgb
        err_a = pred_a - batch.alpha
        ray_losses = (err_c ** 2).sum(axis=1) + err_a ** 2
        if np.any(hit):
            ray_losses[hit] = lh                 # the f64 loss of the exact (not f32-rounded) prediction
        loss = float(ray_losses.mean())
        losses.append(loss)
        if initial is None:
            initial = max(loss, 1e-9)
        bad = bad + 1 if loss > 1e3 * initial else 0
        if bad >= 100:
            raise errors.TrainingError(f"stage-2 diverged at step {step}: loss {loss:.3g}")
        if np.any(hit):
            tr.adam()
        update_error_map(emap, batch.cells, ray_losses)
        if log is not None and step % 50 == 0:
            log(step, loss)
    tr.export()
    return losses
