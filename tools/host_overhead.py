"""Host-side cost of one fused frame launch (config 4), measured on the GPU box:
the Python mirror's SceneRenderer.render vs the raw C-ABI call and its parts.

usage: python tools/host_overhead.py [n]
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2303_04086_b200 import _native as N  # noqa: E402
from paper_2303_04086_b200 import render as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
torch.cuda.set_device(0)
args = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
scene = bench.build_scene(12)
W, H = 3840, 2160
r = R.SceneRenderer(scene)
r.mlp_mode(N.MLP_BF16)
tiles = R.frame_tiles(W, H, 32)
td = torch.from_numpy(tiles).cuda()
P = len(tiles) * 1024
cams = [r.camera_array([bench.camera_for_step(k, W, H)]) for k in range(n)]
r.reserve(cams, P)
out = {"rgba8": torch.zeros((W * H, 4), dtype=torch.uint8, device="cuda"),
       "depth16": torch.full((W * H,), -1, dtype=torch.int16, device="cuda"),
       "counters": torch.zeros(4, dtype=torch.int64, device="cuda")}
st = torch.cuda.current_stream().cuda_stream


def timed(label, f):
    """host time of one call with the device idle (no ring back-pressure)"""
    for k in range(5):
        f(k)
    ts = []
    for k in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f(k)
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    ts = np.array(ts) * 1e6
    print(f"{label:40s} host {np.median(ts):8.1f} us/call (p10 {np.percentile(ts, 10):.1f}, p90 {np.percentile(ts, 90):.1f})")


timed("SceneRenderer.render (prefilled)", lambda k: r.render(cams[k], td, len(tiles), 1024, out, frame_layout=True,
                                                            prefilled=True))
timed("nolf_scene_workspace_bytes", lambda k: N.lib().nolf_scene_workspace_bytes(r._inst_arr, len(r.insts), cams[k], 1, P))
so = N.SceneOut()
so.rgba8, so.depth16, so.tile_stride, so.depth_far, so.layout, so.prefilled = (out["rgba8"].data_ptr(),
                                                                             out["depth16"].data_ptr(), 1024, 10.0, 1, 1)
ws = r._ws
timed("nolf_render_scene (raw ctypes)", lambda k: N.lib().nolf_render_scene(
    r._inst_arr, len(r.insts), cams[k], 1, td.data_ptr(), len(tiles), C.byref(so), 0.5, out["counters"].data_ptr(),
    ws.data_ptr(), ws.numel(), st))
