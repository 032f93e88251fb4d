"""Record the reference farm's ray->worker assignment (tests/golden/dispatch.json).

Runs the REFERENCE MasterNode (farm.py:229-602) tick by tick for one session
and records, per tick, every task it dispatches: (task id, asset, rect,
class, rays, worker id).  Worker.execute is replaced by a recorder that
returns an empty tile, so nothing is rendered (the policy under test is
_build_frame_tasks -> schedule_tick -> _dispatch, farm.py:330-462).
"""

import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from radfarm import farm as F  # noqa: E402
from radfarm.protocol import ClientHello, PoseUpdate, SceneEdit  # noqa: E402
from radfarm.renderer import Tile  # noqa: E402
from radfarm.scenes import orbit_camera  # noqa: E402
from radfarm.scheduler import Thresholds  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dispatch.json")


class _Stub:
    """Just enough of LightFieldAsset for the master (proxy only)."""

    def __init__(self, name):
        from radfarm.core import Aabb
        self.name = name
        self.proxy = Aabb(min=(0.0, 0.0, 0.0), max=(1.0, 1.0, 1.0))


def run(case):
    log = []

    def execute(self, assets, task):
        log.append([task.base.task_id, task.asset_id, list(task.rect), task.base.task_class.value,
                    int(task.base.rays), self.worker_id, bool(task.base.skip)])
        x0, y0, x1, y1 = task.rect
        tile = Tile(x0=x0, y0=y0, rgba=np.zeros((y1 - y0, x1 - x0, 4), np.float32),
                    depth=np.full((y1 - y0, x1 - x0), np.inf, np.float32))
        return F.TaskResult(task.base.task_id, ok=True, tile=tile, instr={}, worker_id=self.worker_id)

    orig = F.Worker.execute
    F.Worker.execute = execute
    try:
        assets = {n: _Stub(n) for n in case["assets"]}
        cfg = F.FarmConfig(heavy_workers=case["heavy"], light_workers=case["light"],
                           light_rays_per_tick=case["rays_per_tick"], tick_s=0.005,
                           tile_size=case["tile"], thresholds=Thresholds(**case["thresholds"]),
                           stats_every_ticks=0)
        m = F.MasterNode(assets, cfg)
        size = case["size"]
        cam = orbit_camera(case["azimuth"], case["elevation"], radius=case["radius"], size=size)
        hello = ClientHello(width=size, height=size, fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy,
                            target_fps=case["fps"])
        m.open_session(hello, None)
        sid = 1
        for name, tr in case["edits"]:
            m.ingest(sid, SceneEdit(op="add", asset=name, transform=np.asarray(tr)), 0.0)
        m.ingest(sid, PoseUpdate(seq=1, pose=cam.pose), 0.0)
        ticks = []
        for t in range(case["ticks"]):
            log.clear()
            m.tick(t * cfg.tick_s)
            ticks.append(list(log))
        return {"case": case, "pose": cam.pose.tolist(), "ticks": ticks}
    finally:
        F.Worker.execute = orig


def placed(scale, tx, ty, tz):
    m = np.eye(4)
    m[:3, :3] *= scale
    m[:3, 3] = [tx, ty, tz]
    return m.tolist()


CASES = [
    # far view: every asset light -> 32x32 tiles round-robin over light workers
    dict(assets=["a", "b"], heavy=1, light=7, rays_per_tick=16384, tile=32, size=128,
         azimuth=0.8, elevation=0.3, radius=6.0, fps=30.0, ticks=6, edits=[],
         thresholds=dict(pix_fraction=0.10, depth=2.0)),
    # near view: heavy whole-frame tasks on the heavy worker, one per tick
    dict(assets=["a", "b"], heavy=1, light=7, rays_per_tick=16384, tile=32, size=128,
         azimuth=0.8, elevation=0.3, radius=1.2, fps=30.0, ticks=6, edits=[],
         thresholds=dict(pix_fraction=0.10, depth=2.0)),
    # mixed scene: a near (heavy) asset, far light assets, one off-screen (skip)
    dict(assets=["a", "b", "c", "d"], heavy=2, light=3, rays_per_tick=8192, tile=24, size=96,
         azimuth=0.5, elevation=0.25, radius=2.5, fps=60.0, ticks=10,
         edits=[["b", placed(0.5, 1.5, 0.2, 0.1)], ["c", placed(0.3, -1.0, 1.8, 0.4)],
                ["d", placed(1.0, 40.0, 40.0, 40.0)]],
         thresholds=dict(pix_fraction=0.10, depth=2.0)),
    # capacity-starved: few light rays per tick -> tasks spill over ticks
    dict(assets=["a", "b", "c"], heavy=1, light=2, rays_per_tick=2048, tile=16, size=64,
         azimuth=1.9, elevation=-0.2, radius=4.0, fps=20.0, ticks=12,
         edits=[["a", placed(0.7, 0.2, -0.3, 0.0)], ["c", placed(1.3, -0.4, 0.4, -0.2)]],
         thresholds=dict(pix_fraction=0.05, depth=2.5)),
]


def main():
    out = [run(c) for c in CASES]
    for r in out:
        print(len(r["ticks"]), [len(t) for t in r["ticks"]])
    json.dump(out, open(OUT, "w"))


if __name__ == "__main__":
    main()
