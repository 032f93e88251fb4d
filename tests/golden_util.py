"""Loading of the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the reference)."""

import dataclasses
import glob
import hashlib
import os

import numpy as np

from paper_2303_04086_b200.model import Camera, ModelWiring
from paper_2303_04086_b200.nolf_io import read_asset

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASE_ASSET = {"sphere": "toy_sphere", "box": "toy_box", "two": "toy_two", "live": "toy_live",
              "norefine": "toy_norefine", "abl": "toy_sphere"}
WIRING_FIELDS = [f.name for f in dataclasses.fields(ModelWiring)]

_assets = {}


def asset(name):
    if name not in _assets:
        _assets[name] = read_asset(os.path.join(GOLDEN, "assets", f"{name}.nolf.gz"))
    return _assets[name]


def load(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def render_cases():
    return sorted(os.path.basename(p)[7:-4] for p in glob.glob(os.path.join(GOLDEN, "render_*.npz")))


def case_asset(case, g):
    """The asset a render case used: the golden .nolf with the case's wiring
    and transform applied (as the generator's dataclasses.replace did)."""
    a = asset(CASE_ASSET[case.split("_")[0]])
    wiring = ModelWiring(**dict(zip(WIRING_FIELDS, (bool(x) for x in g["wiring"]))))
    return dataclasses.replace(a, wiring=wiring, object_to_world=np.asarray(g["transform"]))


def camera(g):
    fx, fy, cx, cy = g["intr"]
    w, h = g["size"]
    return Camera(pose=g["pose"], fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))


def sha(a) -> str:
    """SHA-256 of an array's dtype, shape and bytes."""
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def asset_digests(asset) -> dict:
    """SHA-256 of every asset array the synth restatement must reproduce
    exactly (name -> hex); diffuse cubes are compared by cube_sums instead."""
    d = {
        "density_index": sha(asset.density_atlas.index),
        "density_cubes": sha(asset.density_atlas.cubes),
        "psh_offsets": sha(np.asarray(asset.psh.offsets, np.int64)),
        "psh_features": sha(asset.psh_features),
        "diffuse_index": sha(asset.diffuse_atlas.index),
    }
    for tag, m in (("fs", asset.specular_mlp), ("fd", asset.diffuse_mlp)):
        for i, (w, b) in enumerate(zip(m.weights, m.biases)):
            d[f"{tag}_w{i}"] = sha(w)
            d[f"{tag}_b{i}"] = sha(b)
    for i, f in enumerate(asset.diffuse_features):
        d[f"ed_feat_{i}"] = sha(f)
    return d


def cube_sums(cubes) -> np.ndarray:
    """Per-cube f64 sums (the diffuse cubes' fingerprint)."""
    return np.asarray(cubes, np.float64).reshape(len(cubes), -1).sum(axis=1)
