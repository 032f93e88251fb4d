"""Ray -> GPU assignment, restated from the reference farm (bit-exact policy).

The reference assigns rays to workers in its master loop; with GPUs as the
workers this is the ray -> GPU assignment the north star requires to match
bit for bit.  ``FarmAssigner`` restates the single-session master tick
without rendering:

  _build_frame_tasks     farm.py:330-389  (estimate_nhit -> classify -> rects)
  estimate_nhit          renderer.py:119-173
  classify_task          scheduler.py:135-144
  quantize_pose          scheduler.py:191-200 (shared-ray cache key)
  _dedup_and_cache       farm.py:393-435  (single session: tile-cache hits)
  schedule_tick          scheduler.py:283-367 (Algorithm 1)
  _dispatch              farm.py:439-462  (heavy: pop(0); light: least loaded,
                                           ties to the first worker)
  _collect/_finish_frames farm.py:492-550 (cache insert, frame completion,
                                           timeouts, update_wait_time)

``tests/test_schedule.py`` replays the reference MasterNode's recorded
dispatches (tests/golden/dispatch.json) tick by tick.  ``tile_partition``
is the throughput-mode map (tile t -> GPU t mod N) used by bench.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .model import Camera

_EXACT_PIXEL_BUDGET = 16384


@dataclass
class NhitEstimate:
    n_pixel: int
    avg_depth: float
    frame_fraction: float


def _camera_dirs(cam, px, py):
    u = (np.asarray(px, np.float64) + 0.5 - cam.cx) / cam.fx
    v = -(np.asarray(py, np.float64) + 0.5 - cam.cy) / cam.fy
    d = np.stack([u, v, -np.ones_like(u)], axis=-1) @ cam.rotation.T
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def _slab(o, d, lo, hi):
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        t0 = (lo[None, :] - o) * inv
        t1 = (hi[None, :] - o) * inv
    a, b = np.minimum(t0, t1), np.maximum(t0, t1)
    par = d == 0.0
    ins = (o >= lo[None, :]) & (o <= hi[None, :])
    a = np.where(par, np.where(ins, -np.inf, np.inf), a)
    b = np.where(par, np.where(ins, np.inf, -np.inf), b)
    tn = np.maximum(a.max(axis=-1), 0.0)
    tf = np.minimum(b.min(axis=-1), np.inf)
    return tn, tf, tn <= tf


def estimate_nhit(proxy, object_to_world, camera) -> NhitEstimate:
    """Screen coverage + mean entry depth of a proxy box (renderer.py:119-173)."""
    o2w = np.asarray(object_to_world, np.float64)
    w2o = np.linalg.inv(o2w)
    lo, hi = np.asarray(proxy.min, np.float64), np.asarray(proxy.max, np.float64)
    bits = (np.arange(8)[:, None] >> np.arange(3)[None, :]) & 1
    corners = np.where(bits.astype(bool), hi, lo)
    cw = corners @ o2w[:3, :3].T + o2w[:3, 3]
    cs = (cw - camera.position) @ camera.rotation
    z = -cs[:, 2]
    none = NhitEstimate(0, float("inf"), 0.0)
    if np.all(z <= 1e-9):
        return none
    if np.any(z <= 1e-9):
        bx0, by0, bx1, by1 = 0, 0, camera.width, camera.height
    else:
        px = cs[:, 0] / z * camera.fx + camera.cx - 0.5
        py = -cs[:, 1] / z * camera.fy + camera.cy - 0.5
        bx0 = max(0, int(np.floor(px.min())))
        by0 = max(0, int(np.floor(py.min())))
        bx1 = min(camera.width, int(np.ceil(px.max())) + 1)
        by1 = min(camera.height, int(np.ceil(py.max())) + 1)
        if bx0 >= bx1 or by0 >= by1:
            return none
    stride = 1
    while ((bx1 - bx0) // stride + 1) * ((by1 - by0) // stride + 1) > _EXACT_PIXEL_BUDGET:
        stride *= 2
    gx, gy = np.meshgrid(np.arange(bx0, bx1, stride), np.arange(by0, by1, stride))
    dirs = _camera_dirs(camera, gx.reshape(-1), gy.reshape(-1))
    origins = np.broadcast_to(camera.position, dirs.shape)
    o_obj = origins @ w2o[:3, :3].T + w2o[:3, 3]
    d_raw = dirs @ w2o[:3, :3].T
    lin = w2o[:3, :3]
    scale = float(np.linalg.norm(lin, axis=0).mean())
    d_obj = d_raw / np.linalg.norm(d_raw, axis=1, keepdims=True)
    t_near, _, hit = _slab(o_obj, d_obj, lo, hi)
    n_hit = int(hit.sum())
    if n_hit == 0:
        return none
    n_pixel = min(n_hit * stride * stride, camera.width * camera.height)
    return NhitEstimate(n_pixel, float(np.mean(t_near[hit]) / scale),
                        n_pixel / (camera.width * camera.height))


@dataclass
class Thresholds:
    pix_fraction: float = 0.10
    depth: float = 2.0


def classify_task(est: NhitEstimate, thr: Thresholds):
    """(class, skip): heavy iff coverage >= pix OR depth <= depth; zero coverage -> light skip."""
    if est.n_pixel == 0:
        return "light", True
    heavy = est.frame_fraction >= thr.pix_fraction or est.avg_depth <= thr.depth
    return ("heavy" if heavy else "light"), False


def quantize_pose(pose, trans_cell: float, rot_cell_deg: float = 5.0) -> tuple:
    pose = np.asarray(pose, np.float64)
    t = tuple(np.floor(pose[:3, 3] / trans_cell).astype(int).tolist())
    r = pose[:3, :3]
    yaw = math.degrees(math.atan2(r[1, 0], r[0, 0]))
    pitch = math.degrees(math.asin(max(-1.0, min(1.0, -r[2, 0]))))
    roll = math.degrees(math.atan2(r[2, 1], r[2, 2]))
    return t + tuple(int(math.floor(v / rot_cell_deg)) for v in (yaw, pitch, roll))


@dataclass
class Task:
    task_id: str
    asset_id: str
    rect: tuple
    task_class: str
    rays: int
    skip: bool
    shared_key: tuple


@dataclass
class _Session:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    target_fps: float
    scene: list
    pose: np.ndarray | None = None
    t_avg: float = 0.0
    wait_time: float = 0.0
    target_time: float = 0.0
    pending: list = field(default_factory=list)
    rho: float = 0.3

    def camera(self) -> Camera:
        return Camera(pose=self.pose, fx=self.fx, fy=self.fy, cx=self.cx, cy=self.cy,
                      width=self.width, height=self.height)


class FarmAssigner:
    """Single-session restatement of the reference master tick's task
    construction, scheduling and worker choice (see module docstring)."""

    def __init__(self, proxies: dict, heavy_workers=1, light_workers=2, light_rays_per_tick=16384,
                 tick_s=0.005, tile_size=32, thresholds=None, frame_timeout_ticks=2,
                 cache_ttl_s=2.0, rot_cell_deg=5.0):
        self.proxies = proxies
        self.heavy = [f"heavy{i}" for i in range(heavy_workers)]
        self.light = [f"light{i}" for i in range(light_workers)]
        self.rays_per_tick = light_rays_per_tick
        self.tick_s = tick_s
        self.tile = tile_size
        self.thr = thresholds or Thresholds()
        self.timeout = frame_timeout_ticks
        self.ttl = cache_ttl_s
        self.rot_cell = rot_cell_deg
        self.tick_index = 0
        self.seq = 0
        self.cache = {}            # shared_key -> expiry
        self.assembly = None       # (born_tick, expected set)
        self.session = None
        # what the last tick did, for an executor (farm.GpuFarm): the frame
        # being assembled, tasks served from the tile cache, a finished frame
        self.frame = None          # {"index", "camera", "order", "transforms", "tasks": {id: Task}}
        self.frame_index = -1
        self.last_cache_hits = []  # [Task]
        self.last_finished = None  # {"frame": <self.frame>, "timed_out": set of task ids}

    def open(self, width, height, fx, fy, cx, cy, target_fps, scene=None):
        scene = scene if scene is not None else [(n, np.eye(4)) for n in sorted(self.proxies)]
        s = _Session(width, height, fx, fy, cx, cy, target_fps, list(scene))
        s.wait_time = 1.0 / target_fps - s.t_avg
        self.session = s

    def edit_add(self, name, transform):
        s = self.session
        s.scene = [e for e in s.scene if e[0] != name] + [(name, np.asarray(transform))]

    def set_pose(self, pose):
        self.session.pose = np.asarray(pose, np.float64)

    # farm.py:330-389
    def _build(self):
        s = self.session
        cam = s.camera()
        expected = set()
        self.frame_index += 1
        self.frame = {"index": self.frame_index, "camera": cam, "order": [n for n, _ in s.scene],
                      "transforms": {n: np.asarray(tr, np.float64) for n, tr in s.scene}, "tasks": {}}
        for name, tr in s.scene:
            proxy = self.proxies[name]
            cls, skip = classify_task(estimate_nhit(proxy, tr, cam), self.thr)
            diag = float(np.linalg.norm(np.asarray(proxy.max, float) - np.asarray(proxy.min, float)))
            pose_key = quantize_pose(s.pose, max(diag, 1e-6) * (1.0 / 64.0), self.rot_cell)
            if skip or cls == "heavy":
                rects = [(0, 0, cam.width, cam.height)]
            else:
                rects = [(tx, ty, min(tx + self.tile, cam.width), min(ty + self.tile, cam.height))
                         for ty in range(0, cam.height, self.tile)
                         for tx in range(0, cam.width, self.tile)]
            for rect in rects:
                self.seq += 1
                rays = 0 if skip else (rect[2] - rect[0]) * (rect[3] - rect[1])
                t = Task(f"f{self.seq:08d}", name, rect, cls, rays, skip,
                         (name, pose_key, rect, cam.width, cam.height))
                expected.add(t.task_id)
                s.pending.append(t)
                self.frame["tasks"][t.task_id] = t
        self.assembly = [self.tick_index, expected]

    # scheduler.py:283-367 for one session
    def _schedule(self, now):
        s = self.session
        assignments, taken = [], set()
        if not (s.pending and s.target_time <= now):
            return assignments
        starved = s.target_time <= now - self.tick_s
        heavy_free = len(self.heavy)
        rays = self.rays_per_tick * len(self.light)

        def try_assign(t):
            nonlocal heavy_free, rays
            if id(t) in taken:
                return
            if not t.skip:
                if t.task_class == "heavy":
                    if heavy_free < 1:
                        return
                    heavy_free -= 1
                else:
                    if t.rays > rays:
                        return
                    rays -= t.rays
            assignments.append(t)
            taken.add(id(t))

        if starved:
            for t in sorted(s.pending, key=lambda t: (t.task_class != "heavy", t.task_id)):
                try_assign(t)
        else:
            live = [t for t in s.pending if not t.skip]
            need_h = sum(1 for t in live if t.task_class == "heavy")
            need_r = sum(t.rays for t in live if t.task_class == "light")
            if need_h <= heavy_free and need_r <= rays:
                for t in sorted(s.pending, key=lambda t: t.task_id):
                    try_assign(t)
        s.pending = [t for t in s.pending if id(t) not in taken]
        return assignments

    # farm.py:439-462
    def _dispatch(self, assignments):
        heavy_pool = list(self.heavy)
        light_load = {w: 0 for w in self.light}
        out = []
        for t in assignments:
            if t.task_class == "heavy" and heavy_pool:
                w = heavy_pool.pop(0)
            elif self.light:
                w = min(self.light, key=lambda w: light_load[w])
                light_load[w] += t.rays
            else:
                self.session.pending.append(t)          # _requeue
                continue
            out.append((t, w))
        return out

    def tick(self, now: float):
        """One master tick; returns [(task_id, asset, rect, class, rays, worker, skip)]."""
        s = self.session
        self.last_cache_hits = []
        self.last_finished = None
        if s.pose is not None and self.assembly is None and not s.pending and s.target_time <= now:
            self._build()
        # _dedup_and_cache (single session: only cache hits can occur)
        self.cache = {k: e for k, e in self.cache.items() if e > now}
        if s.target_time <= now:
            for t in list(s.pending):
                if not t.skip and t.shared_key in self.cache:
                    s.pending.remove(t)
                    self.last_cache_hits.append(t)
                    if self.assembly is not None:
                        self.assembly[1].discard(t.task_id)
        dispatched = self._dispatch(self._schedule(now))
        log = []
        for t, w in dispatched:
            log.append((t.task_id, t.asset_id, list(t.rect), t.task_class, t.rays, w, t.skip))
            if not t.skip:
                self.cache[t.shared_key] = now + self.ttl
            if self.assembly is not None:
                self.assembly[1].discard(t.task_id)
        # _finish_frames
        if self.assembly is not None:
            born, expected = self.assembly
            timed_out = self.tick_index - born >= self.timeout and expected
            if not expected or timed_out:
                self.last_finished = {"frame": self.frame, "timed_out": set(expected) if timed_out else set()}
                if timed_out:
                    s.pending = [t for t in s.pending if t.task_id not in expected]
                completion = max(0.0, now - born * self.tick_s)
                s.t_avg = (1.0 - s.rho) * s.t_avg + s.rho * completion
                s.wait_time = 1.0 / s.target_fps - s.t_avg
                s.target_time = now + max(s.wait_time, 0.0)
                self.assembly = None
        self.tick_index += 1
        return log


def tile_partition(n_tiles: int, world: int, rank: int) -> np.ndarray:
    """Tile-interleaved ray-tile -> GPU map: tile t renders on GPU t mod N."""
    return np.arange(rank, n_tiles, world, dtype=np.int64)


def row_owners(n_rows: int, world: int, weights=None) -> np.ndarray:
    """Owner rank of every tile row: round robin (row r -> r mod N), or a
    smooth weighted round robin when per-rank ``weights`` are given (a rank
    with weight w gets ~w / sum(w) of the rows, still interleaved)."""
    if weights is None or all(w == weights[0] for w in weights):
        return np.arange(n_rows, dtype=np.int64) % world
    w = np.asarray(weights, np.float64)
    credit = np.zeros(world)
    out = np.empty(n_rows, np.int64)
    for r in range(n_rows):
        credit += w
        k = int(np.argmax(credit))
        out[r] = k
        credit[k] -= w.sum()
    return out


def tile_rows(tiles: np.ndarray, tile: int) -> np.ndarray:
    """Global tile-row index of every tile (rows counted across cameras)."""
    tiles = np.asarray(tiles)
    heights = np.zeros(int(tiles[:, 0].max()) + 1 if len(tiles) else 1, np.int64)
    for c in range(len(heights)):
        sel = tiles[:, 0] == c
        heights[c] = tiles[sel, 4].max() if sel.any() else 0
    rows_per_cam = -(-heights // tile)
    base = np.concatenate([[0], np.cumsum(rows_per_cam)[:-1]])
    return base[tiles[:, 0]] + tiles[:, 2] // tile


def row_partition(tiles: np.ndarray, world: int, rank: int, tile: int, weights=None) -> np.ndarray:
    """Throughput-mode map: tile ROWS interleaved over GPUs (row index
    counted across cameras), so a GPU's pixels form strided bands of the
    frame -- one strided DMA per band moves them to host memory.  ``weights``
    skews the share per rank (row_owners)."""
    row = tile_rows(tiles, tile)
    owners = row_owners(int(row.max()) + 1 if len(row) else 0, world, weights)
    return np.flatnonzero(owners[row] == rank).astype(np.int64)


def gather_slots(n_tiles: int, world: int, parts=None) -> np.ndarray:
    """Rank-major slot of every tile after an equal-size gather of each
    rank's n_max tile slots (parts: per-rank tile index lists; default the
    tile-interleaved partition)."""
    if parts is None:
        n_max = -(-n_tiles // world)
        t = np.arange(n_tiles)
        return (t % world) * n_max + t // world
    n_max = max(len(p) for p in parts)
    slots = np.full(n_tiles, -1, np.int64)
    for r, p in enumerate(parts):
        slots[p] = r * n_max + np.arange(len(p))
    return slots
