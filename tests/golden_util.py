"""Loading of the committed golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the reference)."""

import dataclasses
import glob
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
