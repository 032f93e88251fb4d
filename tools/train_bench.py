"""Stage-2 training throughput (diagnostic): train_light_field steps per
second on the GPU (train.py) and, where /root/reference exists, the
reference's own train_light_field on the host CPU with the same asset,
views, config and rng.

usage: python tools/train_bench.py [--steps N] [--batch B] [--size S] [--views V] [--ref-steps R]
"""
import argparse
import copy
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--batch", type=int, default=4096)
    p.add_argument("--size", type=int, default=128)
    p.add_argument("--views", type=int, default=8)
    p.add_argument("--ref-steps", type=int, default=0)
    a = p.parse_args()
    from golden_util import asset
    from paper_2303_04086_b200.model import orbit_camera
    cams = [orbit_camera(2 * np.pi * v / a.views, 0.3, radius=2.0, size=a.size) for v in range(a.views)]
    rng = np.random.default_rng(5)
    images = rng.uniform(0.0, 1.0, (a.views, a.size, a.size, 3)).astype(np.float32)
    alphas = rng.uniform(0.0, 1.0, (a.views, a.size, a.size)).astype(np.float32)

    class Cfg:
        steps, batch_rays, lr_features, lr_mlp = a.steps, a.batch, 1e-2, 1e-3
        error_cell, error_floor, error_rho = 8, 1e-3, 0.1
    out = {"steps": a.steps, "batch_rays": a.batch, "views": a.views, "size": a.size}
    if a.steps:
        import torch
        from paper_2303_04086_b200.train import train_light_field
        warm = copy.deepcopy(asset("toy_sphere"))
        Cfg.steps = 3
        train_light_field(warm, images, alphas, cams, Cfg, np.random.default_rng(11))
        Cfg.steps = a.steps
        ga = copy.deepcopy(asset("toy_sphere"))
        torch.cuda.synchronize()
        t = time.perf_counter()
        losses = train_light_field(ga, images, alphas, cams, Cfg, np.random.default_rng(11))
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        out.update(gpu_steps_per_s=a.steps / el, gpu_rays_per_s=a.steps * a.batch / el,
                   loss_first=float(losses[0]), loss_last=float(losses[-1]))
    if a.ref_steps:
        sys.path.insert(0, "/root/reference/pkg/src")
        from radfarm import assetio
        from radfarm.lightfield import LightFieldTrainConfig, train_light_field as ref_train
        import gzip
        import tempfile
        raw = gzip.decompress(open(os.path.join(ROOT, "tests", "golden", "assets", "toy_sphere.nolf.gz"), "rb").read())
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "a.nolf")
            open(path, "wb").write(raw)
            ra = assetio.read_asset(path)
        from radfarm.scenes import orbit_camera as ref_cam
        rcams = [ref_cam(2 * np.pi * v / a.views, 0.3, radius=2.0, size=a.size) for v in range(a.views)]
        cfg = LightFieldTrainConfig(steps=a.ref_steps, batch_rays=a.batch)
        t = time.perf_counter()
        ref_train(ra, images, alphas, rcams, cfg, np.random.default_rng(11))
        el = time.perf_counter() - t
        out.update(ref_steps=a.ref_steps, ref_steps_per_s=a.ref_steps / el, ref_rays_per_s=a.ref_steps * a.batch / el)
    print(out)


if __name__ == "__main__":
    main()
