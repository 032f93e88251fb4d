"""GPU farm workers: the reference master's ray -> worker assignment executed
on B200 ranks.

The reference farm (radfarm/farm.py) runs one master loop per tick: build a
frame's tasks (``_build_frame_tasks`` farm.py:330-389 -- one whole-frame
HEAVY task per near asset, 32x32 LIGHT tiles otherwise, SKIP for assets off
screen), serve repeats from the tile cache (``_dedup_and_cache``
farm.py:393-435), schedule (``schedule_tick`` scheduler.py:283-367),
dispatch (``_dispatch`` farm.py:439-462: heavy -> ``heavy_pool.pop(0)``,
light -> least-loaded light worker), render synchronously in
``Worker.execute`` (farm.py:96-126: ``render_range`` of the placed asset),
blit tiles into per-asset frames (``_deliver_tile`` farm.py:475-490) and
compose finished frames (``_finish_frames`` farm.py:509-550, missing tiles
transparent after a timeout).

``GpuFarm`` keeps that policy bit for bit (``schedule.FarmAssigner``, pinned
to the reference's recorded dispatches) and makes every farm worker a GPU:
worker k of the master's list (heavy workers first, then light) runs on
rank k mod N.  All ranks run the deterministic assigner in lockstep (no
broadcast), each rank renders its own tasks with the CUDA path
(``nolf_render_rect`` into device buffers: exactly ``render_range``'s
pixels), the tiles go to rank 0 in one exchange per tick (NCCL send/recv of
device buffers; gloo/CPU in tests), and rank 0 assembles per-asset frames
and composes them on the GPU (``nolf_compose`` == farm.compose).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .model import Frame
from .schedule import FarmAssigner, Thresholds


@dataclass
class FarmFrame:
    """A composed frame delivered by a tick (rank 0)."""
    index: int
    frame: Frame                 # host copy (farm.compose output)
    timed_out_tiles: int


def _torch():
    import torch
    return torch


class GpuFarm:
    """Reference-policy farm whose workers are GPU ranks.

    ``assets``: name -> LightFieldAsset (replicated on every rank).  Every
    rank constructs the farm with the same arguments and calls ``tick`` in
    lockstep; rank 0 returns the frames finished in the tick.  ``execute``
    (tests) replaces the GPU renderer: execute(task, camera, transform) ->
    (rgba (h,w,4) f32, depth (h,w) f32) tensors on ``device``; ``compose``
    (tests) replaces nolf_compose."""

    def __init__(self, assets: dict, heavy_workers: int = 1, light_workers: int = 2,
                 light_rays_per_tick: int = 16384, tick_s: float = 0.005, tile_size: int = 32,
                 thresholds: Thresholds | None = None, frame_timeout_ticks: int = 2,
                 cache_ttl_s: float = 2.0, world: int = 1, rank: int = 0, device=None, execute=None,
                 compose=None):
        torch = _torch()
        self.assets = assets
        self.assigner = FarmAssigner({n: a.proxy for n, a in assets.items()}, heavy_workers=heavy_workers,
                                     light_workers=light_workers, light_rays_per_tick=light_rays_per_tick,
                                     tick_s=tick_s, tile_size=tile_size, thresholds=thresholds,
                                     frame_timeout_ticks=frame_timeout_ticks, cache_ttl_s=cache_ttl_s)
        self.world, self.rank = world, rank
        workers = self.assigner.heavy + self.assigner.light
        self.worker_rank = {w: i % world for i, w in enumerate(workers)}
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._execute = execute or self._render_task
        self._compose = compose          # (K,P,4), (K,P) tensors -> (P,4), (P,); default nolf_compose
        self.tile_cache = {}     # shared_key -> (expiry, rgba, depth)   (rank 0)
        self.buffers = {}        # asset -> (rgba (H,W,4), depth (H,W)) of the frame being assembled (rank 0)
        self.log = []            # every dispatch: (task id, asset, rect, class, rays, worker, skip, rank)

    # ---------------------------------------------------------------- session
    def open(self, width, height, fx, fy, cx, cy, target_fps, scene=None):
        self.assigner.open(width, height, fx, fy, cx, cy, target_fps, scene)

    def edit_add(self, name, transform):
        self.assigner.edit_add(name, transform)

    def set_pose(self, pose):
        self.assigner.set_pose(pose)

    # ---------------------------------------------------------------- worker
    def _render_task(self, task, camera, transform):
        """Worker.execute (farm.py:96-126) on this rank's GPU: render_range of
        the placed asset over the task's rect, left on the device."""
        torch = _torch()
        from . import render as R
        x0, y0, x1, y1 = task.rect
        h, w = y1 - y0, x1 - x0
        rgba = torch.zeros((h, w, 4), dtype=torch.float32, device=self.device)
        depth = torch.full((h, w), float("inf"), dtype=torch.float32, device=self.device)
        if task.skip:
            return rgba, depth
        inst = R._instance(self.assets[task.asset_id], transform)
        cnt = torch.zeros(4, dtype=torch.int64, device=self.device)
        ws = R.workspace(int(N.lib().nolf_workspace_bytes(1, h * w)))
        cs = N.camera_struct(camera)
        N.check(N.lib().nolf_render_rect(C.byref(inst), C.byref(cs), x0, y0, x1, y1, rgba.data_ptr(),
                                         depth.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws.numel(),
                                         R._stream_ptr()))
        return rgba, depth

    # ---------------------------------------------------------------- exchange
    def _gather(self, dispatched, mine):
        """Rank 0 receives every other rank's tiles (sizes known from the
        common dispatch list): one flat f32 buffer per rank, NCCL send/recv
        of device buffers (gloo: host)."""
        torch = _torch()
        if self.world == 1:
            return mine
        import torch.distributed as dist
        on_cpu = dist.get_backend() == "gloo"
        sizes = {r: 0 for r in range(self.world)}
        order = {r: [] for r in range(self.world)}
        for t, w in dispatched:
            r = self.worker_rank[w]
            x0, y0, x1, y1 = t.rect
            sizes[r] += (x1 - x0) * (y1 - y0) * 5
            order[r].append(t)
        if self.rank != 0:
            if sizes[self.rank]:
                flat = torch.cat([torch.cat([mine[t.task_id][0].reshape(-1), mine[t.task_id][1].reshape(-1)])
                                  for t in order[self.rank]])
                dist.send(flat.cpu() if on_cpu else flat, dst=0)
            return {}
        out = dict(mine)
        dev = torch.device("cpu") if on_cpu else self.device
        for r in range(1, self.world):
            if not sizes[r]:
                continue
            flat = torch.empty(sizes[r], dtype=torch.float32, device=dev)
            dist.recv(flat, src=r)
            flat = flat.to(self.device)
            off = 0
            for t in order[r]:
                x0, y0, x1, y1 = t.rect
                n = (x1 - x0) * (y1 - y0)
                out[t.task_id] = (flat[off:off + 4 * n].reshape(y1 - y0, x1 - x0, 4),
                                  flat[off + 4 * n:off + 5 * n].reshape(y1 - y0, x1 - x0))
                off += 5 * n
        return out

    # ---------------------------------------------------------------- assembly (rank 0)
    def _deliver(self, frame, task, rgba, depth):
        """_deliver_tile (farm.py:475-490): blit into the asset's frame buffer."""
        torch = _torch()
        cam = frame["camera"]
        buf = self.buffers.get(task.asset_id)
        if buf is None:
            buf = (torch.zeros((cam.height, cam.width, 4), dtype=torch.float32, device=self.device),
                   torch.full((cam.height, cam.width), float("inf"), dtype=torch.float32, device=self.device))
            self.buffers[task.asset_id] = buf
        x0, y0, x1, y1 = task.rect
        buf[0][y0:y1, x0:x1] = rgba
        buf[1][y0:y1, x0:x1] = depth

    def _finish(self, fin) -> FarmFrame:
        """_finish_frames (farm.py:509-550): compose the asset frames in scene
        order (absent ones / missing tiles transparent)."""
        torch = _torch()
        from . import render as R
        frame = fin["frame"]
        cam = frame["camera"]
        H, W = cam.height, cam.width
        rg, dp = [], []
        for name in frame["order"]:
            buf = self.buffers.get(name)
            if buf is None:
                buf = (torch.zeros((H, W, 4), dtype=torch.float32, device=self.device),
                       torch.full((H, W), float("inf"), dtype=torch.float32, device=self.device))
            rg.append(buf[0].reshape(H * W, 4))
            dp.append(buf[1].reshape(H * W))
        if rg:
            o_rgba, o_depth = (self._compose or R.compose_device)(torch.stack(rg), torch.stack(dp))
            out = Frame(width=W, height=H, rgba=o_rgba.reshape(H, W, 4).cpu().numpy(),
                        depth=o_depth.reshape(H, W).cpu().numpy())
        else:
            out = Frame(width=W, height=H, rgba=np.zeros((H, W, 4), np.float32),
                        depth=np.full((H, W), np.inf, np.float32))
        self.buffers = {}
        return FarmFrame(frame["index"], out, len(fin["timed_out"]))

    # ---------------------------------------------------------------- tick
    def tick(self, now: float):
        """One master tick on every rank (collective).  Returns (dispatches
        of this tick, frames finished) -- frames on rank 0 only."""
        fa = self.assigner
        log = fa.tick(now)
        frame = fa.frame
        tasks = frame["tasks"] if frame is not None else {}
        dispatched = [(tasks[e[0]], e[5]) for e in log]
        mine = {}
        for t, w in dispatched:
            if self.worker_rank[w] == self.rank:
                mine[t.task_id] = self._execute(t, frame["camera"], frame["transforms"][t.asset_id])
        tiles = self._gather(dispatched, mine)
        self.log.extend(tuple(e) + (self.worker_rank[e[5]],) for e in log)
        finished = []
        if self.rank == 0:
            # tile-cache hits first (served in _dedup_and_cache), then this tick's renders
            for t in fa.last_cache_hits:
                ent = self.tile_cache.get(t.shared_key)
                if ent is not None:
                    self._deliver(frame, t, ent[1], ent[2])
            for t, w in dispatched:
                rgba, depth = tiles[t.task_id]
                if not t.skip:
                    self.tile_cache[t.shared_key] = (now + fa.ttl, rgba, depth)
                self._deliver(frame, t, rgba, depth)
            self.tile_cache = {k: v for k, v in self.tile_cache.items() if v[0] > now}
            if fa.last_finished is not None:
                finished.append(self._finish(fa.last_finished))
        elif fa.last_finished is not None:
            self.buffers = {}
        return log, finished
