"""Reference-scale golden for BASELINE config 1, made by running the REFERENCE.

Test infrastructure (like make_golden.py): imports radfarm from
``/root/reference/pkg/src`` (build container only) and writes
``tests/golden/fullsize_config1.npz``:

* the config-1 asset exactly as SURVEY.md 8(d) defines it -- ``sphere_scene()``
  baked ``bake_density_cubes(b=32, r=8)`` (lightfield.py:534-544),
  ``init_light_field(atlas, MarchParams(1/256), LightFieldTrainConfig(
  psh_resolution=64), default_rng(0))`` (lightfield.py:600-651) and
  ``bake_diffuse_cubes`` with its default shell (lightfield.py:547-576) --
  recorded as SHA-256 digests of every array that the GPU-box restatement
  (synth.make_asset("sphere", seed=0)) must reproduce bit for bit, plus
  per-cube f64 sums of the diffuse cubes (those come from an fp32 MLP whose
  summation order differs from OpenBLAS sgemm by ~1e-7);
* one 256x256 view, ``orbit_camera(0.8, 0.3, radius=2.0, size=256)``, through
  ``render_range`` (renderer.py:63-93): rgba, depth, counters, and the staged
  trace's hit rows, hit sample indices, active sample counts and PSH slots;
  plus the "close" variant of SURVEY 8(d) config 1 (radius 1.0);

and ``tests/golden/fullsize_zodiac.npz``: BASELINE config 4's 12-asset
zodiac scene (asset i: density sphere / box / two-spheres cycling, seed i,
the same reference pipeline; placements and camera from synth.zodiac_*, i.e.
the bench's own workload definition) rendered by the reference's
``render_frame`` + ``compose`` (renderer.py:96-107, farm.py:129-172) from the
bench's step-0 camera at 1/8 of 4K per axis (480x270): digests of all 12
assets, the composed frame, per-asset depths and counters.

The asset itself (~25 MB) is not committed: the GPU box rebuilds it with
synth and the digests prove it identical.  Run: python
tests/golden/make_golden_fullsize.py (a few minutes on 8 cores).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import make_golden as MG  # noqa: E402  (puts the reference on sys.path)
from golden_util import asset_digests, cube_sums  # noqa: E402

from radfarm.lightfield import (LightFieldTrainConfig, MarchParams, RenderCounters,  # noqa: E402
                                bake_density_cubes, bake_diffuse_cubes, init_light_field)
from radfarm.renderer import RayRange, render_range  # noqa: E402
from radfarm.farm import compose  # noqa: E402
from radfarm.renderer import render_frame  # noqa: E402
from radfarm.scenes import orbit_camera, sphere_scene  # noqa: E402

from tools import synth  # noqa: E402  (workload definition: zodiac placements + camera)


def ref_asset(kind, seed):
    """The reference pipeline at its defaults (b=32, r=8, PSH N=64)."""
    objs = MG.SCENES[kind]().objects

    def density(p):
        return np.max(np.stack([o.density(p) for o in objs]), axis=0)

    atlas = bake_density_cubes(density, b=32, r=8)
    asset = init_light_field(atlas, MarchParams(step=1.0 / 256), LightFieldTrainConfig(psh_resolution=64),
                             np.random.default_rng(seed))
    asset.diffuse_atlas = bake_diffuse_cubes(asset)
    return asset


def trace_case(asset, cam, tag):
    t1 = time.time()
    d = MG.render_case(asset, cam, tag=tag)
    print(f"{tag}: render + trace {time.time() - t1:.1f} s: hits {int(d['hit'].sum())}", flush=True)
    return dict(
        rect=d["rect"], rgba=d["rgba"], depth=d["depth"], counters=d["counters"],
        hit_rows=d["hit_rows"], istar=d["istar"][d["hit_rows"]], samples=d["samples"],
        t_hit=d["t_hit"][d["hit_rows"]], psh_slots=d["psh_slots"], es=d["es"], fs_out=d["fs_out"],
        diffuse=d["diffuse"], pose=d["pose"], intr=d["intr"], size=d["size"],
        transform=d["transform"], wiring=d["wiring"])


def digest_arrays(asset, prefix=""):
    dig = asset_digests(asset)
    return {f"{prefix}digest_names": np.array(sorted(dig)),
            f"{prefix}digests": np.array([dig[k] for k in sorted(dig)]),
            f"{prefix}diffuse_cube_sums": cube_sums(asset.diffuse_atlas.cubes),
            f"{prefix}diffuse_cubes_shape": np.array(asset.diffuse_atlas.cubes.shape),
            f"{prefix}psh_sizes": np.array([asset.psh.table_size, asset.psh.offset_size])}


def main():
    which = sys.argv[1:] or ["config1", "zodiac"]
    if "config1" in which:
        t0 = time.time()
        asset = ref_asset("sphere", 0)
        print(f"config-1 asset built in {time.time() - t0:.1f} s: cubes {asset.density_atlas.cube_count}, "
              f"psh m={asset.psh.table_size} mphi={asset.psh.offset_size}, "
              f"diffuse cubes {asset.diffuse_atlas.cube_count}", flush=True)
        keep = trace_case(asset, orbit_camera(0.8, 0.3, radius=2.0, size=256), "config1_far")
        close = trace_case(asset, orbit_camera(0.8, 0.3, radius=1.0, size=256), "config1_close")
        keep.update({f"close_{k}": v for k, v in close.items()})
        keep.update(digest_arrays(asset))
        MG.savez("fullsize_config1.npz", keep)
    if "zodiac" in which:
        W, H = 480, 270
        cam = synth.zodiac_camera(W, H, azimuth=0.3)
        tr = synth.zodiac_transforms(12)
        scene, keep = [], {}
        for i in range(12):
            t0 = time.time()
            a = ref_asset(synth.ZODIAC_KINDS[i % 3], i)
            print(f"zodiac asset {i} built in {time.time() - t0:.1f} s", flush=True)
            scene.append((a, tr[i]))
            keep.update(digest_arrays(a, prefix=f"a{i}_"))
        t1 = time.time()
        counters = RenderCounters()
        frames = render_frame(scene, cam, counters)
        out = compose(frames)
        print(f"zodiac render_frame + compose {time.time() - t1:.1f} s", flush=True)
        keep.update(kinds=np.array([synth.ZODIAC_KINDS[i % 3] for i in range(12)]),
                    transforms=np.stack(tr), rgba=out.rgba, depth=out.depth,
                    frame_depth=np.stack([f.depth for f in frames]),
                    counters=np.array([counters.fs_evals, counters.fd_evals, counters.hit_pixels,
                                       counters.march_samples]),
                    **MG.camera_arrays(cam))
        MG.savez("fullsize_zodiac.npz", keep)
    for f in ("fullsize_config1.npz", "fullsize_zodiac.npz"):
        p = os.path.join(MG.OUT, f)
        if os.path.exists(p):
            print("written", p, os.path.getsize(p), "bytes")


if __name__ == "__main__":
    main()
