"""Generate the committed golden fixtures by running the REFERENCE (radfarm).

This script is test infrastructure. It imports the reference package from
``/root/reference/pkg/src`` (read-only, present only in the build container),
builds small deterministic assets with the reference's own functions, and
dumps:

* ``assets/<name>.nolf.gz``  -- the reference ``write_asset`` bytes, gzipped;
* ``render_<case>.npz``       -- per-ray inputs and every intermediate of
  ``lightfield.render_rays`` (lightfield.py:400-456) re-run stage by stage
  with the reference's functions, checked against the reference's own
  ``render_range`` / ``render_rays`` output before saving;
* ``compose.npz``             -- ``farm.compose`` (farm.py:129-172) goldens;
* ``scene.npz``               -- ``renderer.render_frame`` + ``compose`` goldens.

Run:  python tests/golden/make_golden.py   (takes ~1 min)
Nothing under tests/, bench.py or the package reads /root/reference at run
time; only the fixtures this writes are consumed.
"""

from __future__ import annotations

import dataclasses
import gzip
import io
import math
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

from radfarm import assetio  # noqa: E402
from radfarm.atlas import AtlasSource, query_atlas  # noqa: E402
from radfarm.core import (  # noqa: E402
    aabb_intersect_batch,
    camera_dirs,
    sh_encode_batch,
    transform_points,
    uniform_scale_of,
)
from radfarm.encoding import _base_weights, psh_encode_with_cache, hashgrid_encode_with_cache  # noqa: E402
from radfarm.farm import compose  # noqa: E402
from radfarm.lightfield import (  # noqa: E402
    LightFieldTrainConfig,
    collect_hit_points,
    MarchParams,
    RenderCounters,
    ablation_variant,
    bake_density_cubes,
    bake_diffuse_cubes,
    init_light_field,
    march_rays,
    render_rays,
)
from radfarm.core import Frame  # noqa: E402
from radfarm.neural import mlp_forward  # noqa: E402
from radfarm.renderer import RayRange, render_frame, render_range  # noqa: E402
from radfarm.scenes import box_scene, orbit_camera, sphere_scene, two_spheres_scene  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SCENES = {"sphere": sphere_scene, "box": box_scene, "two": two_spheres_scene}


def make_asset(kind: str, seed: int, diffuse_atlas=True, wiring=None, b=16, r=4, n_psh=16):
    """Toy asset exactly as the reference's conftest ``toy_asset`` builds it
    (pkg/tests/conftest.py:14-28), parameterised by density scene and seed."""
    objs = SCENES[kind]().objects

    def density(p):
        return np.max(np.stack([o.density(p) for o in objs]), axis=0)

    atlas = bake_density_cubes(density, b=b, r=r)
    cfg = LightFieldTrainConfig(
        psh_resolution=n_psh, shell_cameras=12, shell_image_size=16,
        diffuse_levels=3, diffuse_table_size=2**10,
    )
    asset = init_light_field(atlas, MarchParams(step=1 / (b * r)), cfg,
                             np.random.default_rng(seed), wiring=wiring)
    if diffuse_atlas:
        asset.diffuse_atlas = bake_diffuse_cubes(asset, shell_cameras=8, shell_image_size=8)
    asset.name = f"{kind}{seed}"
    return asset


def save_asset(asset, name):
    os.makedirs(os.path.join(OUT, "assets"), exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.nolf")
        assetio.write_asset(asset, p)
        raw = open(p, "rb").read()
    with open(os.path.join(OUT, "assets", f"{name}.nolf.gz"), "wb") as f:
        f.write(gzip.compress(raw, mtime=0))
    # round-trip through the reference reader so the golden renders use the
    # exact arrays a .nolf consumer sees (assetio.py:174-255)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.nolf")
        open(p, "wb").write(raw)
        return assetio.read_asset(p)


def stage_trace(asset, origins, dirs):
    """Re-run render_rays (lightfield.py:400-456) stage by stage with the
    reference's own functions, keeping every intermediate."""
    out = {}
    w2o = np.linalg.inv(asset.object_to_world)
    scale = uniform_scale_of(w2o)
    o_obj = transform_points(np.asarray(origins, dtype=np.float64), w2o)
    d_raw = np.asarray(dirs, dtype=np.float64) @ w2o[:3, :3].T
    d_obj = d_raw / np.linalg.norm(d_raw, axis=1, keepdims=True)
    out.update(w2o=w2o, scale=np.float64(scale), o_obj=o_obj, d_obj=d_obj)
    t_near, t_far, boxhit = aabb_intersect_batch(o_obj, d_obj, asset.proxy, 0.0, np.inf)
    out.update(t_near=t_near, t_far=t_far, boxhit=boxhit)
    n = len(origins)
    hit_all = np.zeros(n, bool)
    t_hit_all = np.full(n, np.inf)
    alpha_c_all = np.zeros(n)
    samples_all = np.zeros(n, np.int64)
    trans_all = np.ones(n)
    istar_all = np.full(n, -1, np.int64)
    if np.any(boxhit):
        res = march_rays(asset.density_source(), o_obj[boxhit], d_obj[boxhit],
                         t_near[boxhit], t_far[boxhit], asset.march)
        hit_all[boxhit] = res.hit
        t_hit_all[boxhit] = res.t_hit
        alpha_c_all[boxhit] = res.alpha_c
        samples_all[boxhit] = res.samples
        trans_all[boxhit] = res.t_last_trans
        rows = np.flatnonzero(boxhit)
        hr = rows[res.hit]
        # hit sample index i*: t_hit = t_near + (i*+0.5)*step (lightfield.py:159)
        istar_all[hr] = np.rint((res.t_hit[res.hit] - t_near[hr]) / asset.march.step - 0.5).astype(np.int64)
        p_h_all = np.zeros((n, 3))
        p_h_all[boxhit] = res.p_h
    else:
        p_h_all = np.zeros((n, 3))
    out.update(hit=hit_all, t_hit=t_hit_all, alpha_c=alpha_c_all, samples=samples_all,
               t_last_trans=trans_all, istar=istar_all, p_h=p_h_all)
    hit_rows = np.flatnonzero(hit_all)
    out["hit_rows"] = hit_rows
    if len(hit_rows) and asset.psh is not None:
        p_h = p_h_all[hit_rows]
        if not asset.wiring.use_hit_point:
            p_h = np.clip(o_obj[hit_rows] + t_near[hit_rows][:, None] * d_obj[hit_rows], 0.0, 1.0)
        base, w = _base_weights(p_h, asset.psh.resolution)
        es, (slots, _) = psh_encode_with_cache(asset.psh, asset.psh_features, p_h)
        ev = sh_encode_batch(d_obj[hit_rows])
        ac = np.clip(alpha_c_all[hit_rows], 1e-4, 1 - 1e-4)
        if asset.wiring.refine_opacity:
            fs_in = np.concatenate([es, ev, ac[:, None]], axis=1)
        else:
            fs_in = np.concatenate([es, ev], axis=1)
        fs_out, _ = mlp_forward(asset.specular_mlp, fs_in)
        out.update(psh_base=base, psh_w=w, psh_slots=slots, es=es, sh=ev,
                   fs_in=fs_in.astype(np.float32), fs_out=fs_out, shade_p=p_h)
        if asset.diffuse_atlas is not None:
            out["diffuse"] = query_atlas(asset.diffuse_atlas, p_h)
        else:
            ed, _ = hashgrid_encode_with_cache(asset.diffuse_encoder, asset.diffuse_features, p_h)
            fd_out, _ = mlp_forward(asset.diffuse_mlp, ed)
            out["ed"] = ed
            out["diffuse"] = fd_out
    return out


def camera_arrays(cam):
    return dict(pose=cam.pose, intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
                size=np.array([cam.width, cam.height]))


def render_case(asset, cam, rect=None, tag=""):
    x0, y0, x1, y1 = rect if rect is not None else (0, 0, cam.width, cam.height)
    counters = RenderCounters()
    tile, instr = render_range(asset, RayRange(cam, x0, y0, x1, y1), counters)
    xs, ys = np.arange(x0, x1), np.arange(y0, y1)
    px, py = np.meshgrid(xs, ys)
    dirs = camera_dirs(cam, px.reshape(-1), py.reshape(-1))
    origins = np.broadcast_to(cam.position, dirs.shape)
    tr = stage_trace(asset, origins, dirs)
    rgba = tile.rgba.reshape(-1, 4)
    depth = tile.depth.reshape(-1)
    # the staged trace must reproduce the reference render bit for bit
    rgba2, depth2 = render_rays(asset, origins, dirs)
    assert np.array_equal(rgba, rgba2) and np.array_equal(depth, depth2), tag
    d = dict(rect=np.array([x0, y0, x1, y1]), dirs=dirs, origin=np.asarray(cam.position),
             rgba=rgba, depth=depth,
             counters=np.array([counters.fs_evals, counters.fd_evals,
                                counters.hit_pixels, counters.march_samples]),
             transform=np.asarray(asset.object_to_world, dtype=np.float64),
             wiring=np.array(dataclasses.astuple(asset.wiring), dtype=bool),
             **camera_arrays(cam), **tr)
    return d


def rays_case(asset, rng, n=512):
    """Arbitrary world rays incl. axis-parallel directions (core.py:216-220)."""
    o = rng.uniform(-1.0, 2.0, (n, 3))
    target = rng.uniform(0.2, 0.8, (n, 3))
    d = target - o
    d[: n // 8, 1:] = 0.0  # +-x parallel to y/z slabs
    d[n // 8 : n // 4, 0] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    counters = RenderCounters()
    rgba, depth = render_rays(asset, o, d, counters)
    tr = stage_trace(asset, o, d)
    return dict(origins=o, dirs=d, rgba=rgba, depth=depth,
                counters=np.array([counters.fs_evals, counters.fd_evals,
                                   counters.hit_pixels, counters.march_samples]),
                transform=np.asarray(asset.object_to_world, dtype=np.float64),
                wiring=np.array(dataclasses.astuple(asset.wiring), dtype=bool), **tr)


def savez(name, d):
    np.savez_compressed(os.path.join(OUT, name), **d)


def placed(asset, m):
    return dataclasses.replace(asset, object_to_world=np.asarray(m, dtype=np.float64))


def rot_z(theta):
    c, s = math.cos(theta), math.sin(theta)
    m = np.eye(4)
    m[:2, :2] = [[c, -s], [s, c]]
    return m


def main():
    rng = np.random.default_rng(1234)
    assets = {}
    for kind, seed in (("sphere", 3), ("box", 1), ("two", 2)):
        a = make_asset(kind, seed)
        assets[kind] = save_asset(a, f"toy_{kind}")
    live = make_asset("sphere", 5, diffuse_atlas=False)
    assets["live"] = save_asset(live, "toy_live")
    norefine = make_asset("sphere", 6, wiring=ablation_variant(["refine_opacity"]))
    assets["norefine"] = save_asset(norefine, "toy_norefine")
    print("assets:", {k: (v.density_atlas.cube_count, v.psh.table_size, v.psh.offset_size)
                      for k, v in assets.items()})

    sph = assets["sphere"]
    cases = {
        "sphere_far": (sph, orbit_camera(0.8, 0.3, radius=2.0, size=64), None),
        "sphere_close": (sph, orbit_camera(2.1, -0.4, radius=1.0, size=48), None),
        "sphere_inside": (sph, orbit_camera(0.3, 0.1, radius=0.35, size=32), None),
        "sphere_tile": (sph, orbit_camera(0.4, 0.3, radius=2.0, size=48), (7, 13, 31, 40)),
        "box_far": (assets["box"], orbit_camera(1.3, 0.5, radius=1.8, size=48), None),
        "two_far": (assets["two"], orbit_camera(0.7, 0.2, radius=2.0, size=48), None),
        "live_far": (assets["live"], orbit_camera(0.8, 0.3, radius=2.0, size=40), None),
        "norefine_far": (assets["norefine"], orbit_camera(0.5, 0.2, radius=2.0, size=40), None),
    }
    m = rot_z(0.6)
    m[:3, :3] *= 0.5
    m[:3, 3] = [0.9, -0.2, 0.3]
    cases["sphere_xform"] = (placed(sph, m), orbit_camera(0.8, 0.3, radius=2.0, size=48,
                                                         target=(1.0, 0.1, 0.55)), None)
    for flag in ("hit_point", "opacity", "tint", "diffuse_color"):
        a = dataclasses.replace(sph, wiring=ablation_variant([flag]))
        cases[f"abl_{flag}"] = (a, orbit_camera(0.8, 0.3, radius=2.0, size=32), None)
    for name, (a, cam, rect) in cases.items():
        d = render_case(a, cam, rect, tag=name)
        savez(f"render_{name}.npz", d)
        print(name, "rays", len(d["rgba"]), "hits", int(d["hit"].sum()),
              "samples", int(d["samples"].sum()))

    savez("rays_sphere.npz", rays_case(sph, rng))
    savez("rays_sphere_xform.npz", rays_case(placed(sph, m), rng))

    # ---- hit shells the toy assets were built from (synth restatement pins) ----
    sh = {}
    for kind in ("sphere", "box", "two"):
        a = assets[kind]
        src = AtlasSource(a.density_atlas)
        sh[f"{kind}_psh"] = collect_hit_points(src, a.march, n_cameras=12, image_size=16)
        sh[f"{kind}_dif"] = collect_hit_points(src, a.march, n_cameras=8, image_size=8)
    savez("shells.npz", sh)

    # ---- compose goldens (farm.py:129-172) ----
    comp = {}
    for ci, (k, h, w) in enumerate(((1, 5, 7), (3, 8, 8), (5, 9, 11), (12, 6, 10))):
        rgba = np.zeros((k, h, w, 4), np.float32)
        depth = np.full((k, h, w), np.inf, np.float32)
        for i in range(k):
            alpha = rng.uniform(0.0, 1.0, (h, w)).astype(np.float32)
            alpha[rng.uniform(size=(h, w)) < 0.3] = 0.0
            alpha[rng.uniform(size=(h, w)) < 0.1] = 1.0
            rgba[i, ..., :3] = (rng.uniform(0, 1, (h, w, 3)) * alpha[..., None]).astype(np.float32)
            rgba[i, ..., 3] = alpha
            dd = rng.choice([1.0, 1.5, 2.0, 2.5], size=(h, w)).astype(np.float32)  # many ties
            depth[i] = np.where(alpha > 0, dd, np.inf)
        frames = [Frame(width=w, height=h, rgba=rgba[i].copy(), depth=depth[i].copy())
                  for i in range(k)]
        out = compose(frames)
        comp[f"in_rgba_{ci}"] = rgba
        comp[f"in_depth_{ci}"] = depth
        comp[f"out_rgba_{ci}"] = out.rgba
        comp[f"out_depth_{ci}"] = out.depth
    savez("compose.npz", comp)

    # ---- multi-asset scene (renderer.render_frame + farm.compose) ----
    scene = []
    names = []
    for i, kind in enumerate(("sphere", "box", "two", "sphere")):
        th = 2 * math.pi * i / 4
        mm = rot_z(th)
        mm[:3, :3] *= 0.5
        mm[:3, 3] = [math.cos(th) * 0.6, math.sin(th) * 0.6, 0.0]
        scene.append((assets[kind], mm))
        names.append(kind)
    cam = orbit_camera(0.5, 0.6, radius=2.5, size=64, target=(0.2, 0.2, 0.25))
    frames = render_frame(scene, cam)
    out = compose(frames)
    savez("scene.npz", dict(
        names=np.array(names), transforms=np.stack([s[1] for s in scene]),
        frame_rgba=np.stack([f.rgba for f in frames]),
        frame_depth=np.stack([f.depth for f in frames]),
        rgba=out.rgba, depth=out.depth, **camera_arrays(cam)))
    print("done")


if __name__ == "__main__":
    main()
