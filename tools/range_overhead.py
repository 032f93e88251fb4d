"""The drop-in path's per-call cost (what a farm worker calls per light
tile): render_range on 32x32 tiles, wall time per call, through this repo's
mirror (GPU) or the reference (host CPU, where /root/reference exists).

usage: python tools/range_overhead.py gpu|ref [size]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "gpu"
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    if which == "gpu":
        from golden_util import asset
        from paper_2303_04086_b200 import render as R
        from paper_2303_04086_b200.model import RayRange, orbit_camera
        a = asset("toy_sphere")
        cam = orbit_camera(0.8, 0.3, radius=2.0, size=size)
        call = lambda x0, y0: R.render_range(a, RayRange(cam, x0, y0, x0 + 32, y0 + 32))   # noqa: E731
    else:
        sys.path.insert(0, "/root/reference/pkg/src")
        import gzip
        import tempfile
        from radfarm import assetio
        from radfarm.renderer import RayRange, render_range
        from radfarm.scenes import orbit_camera
        raw = gzip.decompress(open(os.path.join(ROOT, "tests", "golden", "assets", "toy_sphere.nolf.gz"), "rb").read())
        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "a.nolf")
            open(p, "wb").write(raw)
            a = assetio.read_asset(p)
        cam = orbit_camera(0.8, 0.3, radius=2.0, size=size)
        call = lambda x0, y0: render_range(a, RayRange(cam, x0, y0, x0 + 32, y0 + 32))   # noqa: E731
    tiles = [(x, y) for y in range(0, size, 32) for x in range(0, size, 32)]
    for x, y in tiles[:4]:
        call(x, y)
    ts, hits = [], 0
    for x, y in tiles:
        t = time.perf_counter()
        tile, instr = call(x, y)
        ts.append(time.perf_counter() - t)
        hits += int(instr["hits"])
    ts = np.array(ts) * 1e6
    print({"impl": which, "tiles": len(tiles), "hits": hits, "us_per_call_median": round(float(np.median(ts)), 1),
           "us_per_call_p90": round(float(np.percentile(ts, 90)), 1),
           "frame_ms_by_tiles": round(float(ts.sum()) / 1e3, 2)})


if __name__ == "__main__":
    main()
