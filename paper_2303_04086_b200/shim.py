"""Drop-in rebinding of the reference's render path.

``install()`` points every name through which the reference calls its hot
path at this package's CUDA-backed functions.  Modules import by value, so
each binding site is patched explicitly:

  radfarm.lightfield.render_rays / render_ray   (used by render_ray, lightfield.py:460)
  radfarm.renderer.render_rays                  (bound renderer.py:13, used :78)
  radfarm.renderer.render_range / render_frame  (renderer.py:63, 96)
  radfarm.farm.render_range                     (bound farm.py:32, used Worker.execute :124)
  radfarm.farm.compose                          (module global, used _finish_frames :545;
                                                 cli.py:137 imports it lazily)
  radfarm.pipeline.render_range                 (pipeline.py:25, used :139)
  radfarm.bench.render_range                    (bench.py:27, used :235)
  radfarm.protocol.encode_frame                 (protocol.py:256)
  radfarm.farm.encode_frame                     (bound farm.py:30, used tick :587)

Results are returned as the reference's own ``Tile`` / ``Frame`` classes and
errors are raised as the reference's own exception classes.
"""

from __future__ import annotations

import importlib

from . import errors, render

_SAVED: list = []

_BINDINGS = [
    ("radfarm.lightfield", "render_rays", render.render_rays),
    ("radfarm.lightfield", "render_ray", render.render_ray),
    ("radfarm.renderer", "render_rays", render.render_rays),
    ("radfarm.renderer", "render_range", render.render_range),
    ("radfarm.renderer", "render_frame", render.render_frame),
    ("radfarm.farm", "render_range", render.render_range),
    ("radfarm.farm", "compose", render.compose),
    ("radfarm.pipeline", "render_range", render.render_range),
    ("radfarm.bench", "render_range", render.render_range),
    ("radfarm.protocol", "encode_frame", render.encode_frame),
    ("radfarm.farm", "encode_frame", render.encode_frame),
]


def install() -> list:
    """Rebind the reference's hot path; returns the (module, name) pairs patched."""
    if _SAVED:
        return [(m, n) for m, n, _ in _SAVED]
    errs = importlib.import_module("radfarm.errors")
    errors.rebind(errs)
    core = importlib.import_module("radfarm.core")
    rend = importlib.import_module("radfarm.renderer")
    render.TYPES["Frame"] = core.Frame
    render.TYPES["Tile"] = rend.Tile
    render.TYPES["FrameData"] = importlib.import_module("radfarm.protocol").FrameData
    done = []
    for mod_name, attr, fn in _BINDINGS:
        mod = importlib.import_module(mod_name)
        if not hasattr(mod, attr):
            raise AttributeError(f"{mod_name}.{attr} not found: reference layout changed")
        _SAVED.append((mod_name, attr, getattr(mod, attr)))
        setattr(mod, attr, fn)
        done.append((mod_name, attr))
    return done


def uninstall() -> None:
    while _SAVED:
        mod_name, attr, orig = _SAVED.pop()
        setattr(importlib.import_module(mod_name), attr, orig)
    errors.restore()
    render.TYPES.update(render.OWN_TYPES)


def installed() -> bool:
    return bool(_SAVED)
