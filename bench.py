#!/usr/bin/env python
"""i-NOLF render benchmark: BASELINE.json's metric on BASELINE config 4.

Workload (config 4): a 12-asset "zodiac" scene (synthetic assets built like
the reference builds them: analytic densities baked at b=32, r=8, PSH N=64,
random-init networks from default_rng(i), baked diffuse atlas) rendered at
3840x2160 from a camera at distance 4 looking at the ring centre.  One step =
one full 4K frame: march + shade + depth-compose of all 12 assets over every
32x32 tile, plus encode_frame's rgba8 + u16 quantisation.  With N GPUs the
tiles are interleaved over the ranks (tile t -> rank t mod N, strong scaling)
and the encoded tiles are gathered to rank 0 with NCCL (the frame composer).

  python bench.py [--gpus N --steps K --warmup W]      # our arm
  python bench.py --impl reference ...                  # CPU reference arm

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/s and fps at 4K for multi-asset i-NOLF scene at 1/2/4/8 B200 vs CPU ref"
UNIT = "Mrays/s"
# what the path computes in: f64 ray setup / march / PSH addressing / compose,
# bf16 x bf16 -> fp32 specular MLP on tcgen05 (--mlp fp32: CUDA-core fp32)
DTYPE = "f64+bf16"
CACHE_DIR = os.environ.get("NOLF_BENCH_CACHE", "/tmp/nolf_bench_assets")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--build-assets", action="store_true",
                   help="only build / cache the config's synthetic assets (the reference arm runs "
                        "this in a child process so its own process never loads the product)")
    p.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    p.add_argument("--width", type=int, default=3840)
    p.add_argument("--height", type=int, default=2160)
    p.add_argument("--assets", type=int, default=12)
    p.add_argument("--tile", type=int, default=32)
    p.add_argument("--mlp", default="bf16", choices=["fp32", "bf16"])
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-flush", action="store_true",
                   help="diagnostic only: keep L2 warm between timed steps (not a valid bench line)")
    p.add_argument("--e2e-mode", default="sparse", choices=["sparse", "hostmap", "copy"],
                   help="sparse: compose packs only the live chunks (NolfSceneOut.pack), one DMA per "
                        "frame moves them to pinned host memory and nolf_host_scatter rebuilds the "
                        "full frame on host threads (every rank its own rows of one shared frame); "
                        "hostmap: every rank DMAs its full tile rows into one shared page-locked "
                        "host frame; copy: rank 0 downloads the assembled frame with cudaMemcpyAsync")
    p.add_argument("--partition", default="rows", choices=["rows", "tiles"],
                   help="ray tiles over GPUs: interleaved tile rows (default; each rank's pixels "
                        "are strided bands of the frame) or interleaved tiles")
    p.add_argument("--verify", action="store_true",
                   help="rank 0 re-renders the last frame alone and compares bitwise with the "
                        "multi-GPU assembled frame")
    p.add_argument("--prefill", default="on", choices=["on", "state", "off"],
                   help="frame buffers hold the miss encoding outside live chunks so compose "
                        "writes only the chunks some instance reaches: on = the owner re-clears "
                        "a consumed buffer with a memset (side stream); state = per-buffer run "
                        "dirty bits (NolfSceneOut.chunk_state: stale runs reset by the writing "
                        "rank, no full clear; measured slower across NVLink); off = compose "
                        "writes every pixel")
    p.add_argument("--sync", default="flags", choices=["flags", "nccl"],
                   help="p2p frame completion: flags = peer-mapped u32 flags set/polled by tiny kernels "
                        "(no collective); nccl = a 1-element all-reduce per frame")
    p.add_argument("--rank0-weight", type=float, default=None,
                   help="share of tile rows rank 0 renders relative to the other ranks (it also "
                        "re-clears consumed frame buffers and polls the completion flags); default "
                        "0.9 for the 16-view configs (a 440 MB re-clear per step; measured 0.694 -> "
                        "0.677 ms on 4 GPUs, config 5), else 1")
    p.add_argument("--march-order", default="auto", choices=["auto", "spatial", "heavy"],
                   help="live-chunk order of the marcher (NOLF_OPT_MARCH_ORDER): auto = heaviest first "
                        "for launches of a few CTA waves (multi-GPU shards), spatial otherwise")
    p.add_argument("--chunk-cost", type=int, default=1, choices=[0, 1],
                   help="heaviest-first buckets from the previous frame's measured per-chunk march "
                        "durations (1) or from candidate-instance counts (0)")
    p.add_argument("--split", type=int, default=1, choices=[1, 2],
                   help="2: each rank renders its tiles as two interleaved halves on two streams (two "
                        "renderers, two workspaces) so one half's shading / compose overlaps the other's "
                        "march tail")
    p.add_argument("--frames", type=int, default=3,
                   help="p2p + flags: frame buffers in rank 0's ring (a peer renders frame seq once "
                        "frame seq - frames was consumed and re-cleared)")
    p.add_argument("--exchange", default="p2p", choices=["p2p", "dma", "gather"],
                   help="N>1 frame composer: compose stores into rank 0's frame over NVLink "
                        "(CUDA IPC peer memory) or NCCL gather + unpack kernel")
    return p.parse_args()


# ------------------------------------------------------------------ scene
def build_scene(n_assets, cache_only=False):
    """Config-4 scene; cached as .nolf files so repeated runs on a box reuse it.
    cache_only: never synthesise (the reference arm reads files only; its
    assets were built beforehand in a separate process, see run_reference)."""
    from paper_2303_04086_b200 import nolf_io
    from tools import synth
    os.makedirs(CACHE_DIR, exist_ok=True)
    cache, assets = {}, []
    for i in range(n_assets):
        kind = synth.ZODIAC_KINDS[i % 3]
        path = os.path.join(CACHE_DIR, f"zodiac_{kind}_{i}_b32r8n64.nolf")
        if os.path.exists(path):
            a = nolf_io.read_asset(path)
        elif cache_only:
            raise RuntimeError(f"asset cache miss: {path}")
        else:
            a = synth.make_asset(kind, seed=i, cache=cache)
            tmp = f"{path}.{os.getpid()}.tmp"
            nolf_io.write_asset(a, tmp)
            os.replace(tmp, path)
        assets.append(a)
    return list(zip(assets, synth.zodiac_transforms(n_assets)))


def camera_for_step(k, width, height):
    from tools import synth
    return synth.zodiac_camera(width, height, azimuth=0.3 + 0.005 * k)


def workload(args, cache_only=False):
    """(scene, views(k) -> [Camera], W, H, description) of a BASELINE config.

    1: single asset, one 256x256 view           (orbit_camera(0.8, 0.3, 2.0))
    2: single asset with a triangle-mesh proxy (icosphere, 1280 triangles, BVH)
       at 1920x1080
    3: single asset, 16 viewpoints at 3840x2160  (orbit azimuth 2 pi v/16, radius 1.5)
    4: 12-asset zodiac scene at 3840x2160         (the metric's configuration)
    5: 12-asset scene, 8 users x 2 eyes at 2160x2160 (eyes +-0.032 along camera right)
    Each step moves the viewpoints slightly (azimuth + 0.005 k)."""
    import math as m

    from tools import synth
    from paper_2303_04086_b200.model import Camera, orbit_camera
    c = args.config
    if c == 2:
        import dataclasses
        a = dataclasses.replace(build_scene(1, cache_only)[0][0], proxy_mesh=synth.icosphere(radius=0.3, level=3))
        W, H = 1920, 1080
        return [(a, np.eye(4))], (lambda k: [orbit_camera(0.8 + 0.005 * k, 0.3, radius=2.0, width=W,
                                                          height=H)]), W, H, \
            "BASELINE config 2: single asset, mesh proxy (1280-triangle icosphere, BVH), 1920x1080"
    if c in (1, 3):
        scene = build_scene(1, cache_only)[:1]
        scene = [(scene[0][0], np.eye(4))]
        if c == 1:
            W = H = 256
            return scene, (lambda k: [orbit_camera(0.8 + 0.005 * k, 0.3, radius=2.0, size=256)]), W, H, \
                "BASELINE config 1: single asset (sphere, random-init PSH + MLP), one 256x256 view"
        W, H = 3840, 2160
        return scene, (lambda k: [orbit_camera(2 * m.pi * v / 16 + 0.005 * k, 0.3, radius=1.5, width=W,
                                               height=H) for v in range(16)]), W, H, \
            "BASELINE config 3: single asset at 3840x2160, 16 simultaneous viewpoints"
    scene = build_scene(args.assets, cache_only)
    if c == 5:
        W = H = 2160

        def views(k):
            out = []
            for u in range(8):
                base = synth.zodiac_camera(W, H, azimuth=2 * m.pi * u / 8 + 0.005 * k)
                for eye in (-0.032, 0.032):
                    pose = base.pose.copy()
                    pose[:3, 3] += eye * pose[:3, 0]
                    out.append(Camera(pose=pose, fx=base.fx, fy=base.fy, cx=base.cx, cy=base.cy,
                                      width=W, height=H))
            return out
        return scene, views, W, H, (f"BASELINE config 5: {args.assets}-asset scene, 8 users x 2 eyes "
                                    f"at 2160x2160")
    W, H = args.width, args.height
    return scene, (lambda k: [camera_for_step(k, W, H)]), W, H, (
        f"BASELINE config 4: {args.assets}-asset zodiac scene at {W}x{H}")


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling of the local GPU during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []            # (host time, fields)
        self.proc = None
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.perf_counter(), parts))

    def wait_first(self, timeout=10.0):
        t0 = time.perf_counter()
        while self.proc is not None and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = [r for t, r in self.rows if self.window and self.window[0] <= t <= self.window[1]]
        in_window = bool(rows)
        if not rows and self.rows and self.window:   # timed region shorter than one sample
            mid = 0.5 * (self.window[0] + self.window[1])
            rows = [min(self.rows, key=lambda tr: abs(tr[0] - mid))[1]]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        load = [v for v in sm if v > 600] or sm
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "in_timed_window": in_window}


# ------------------------------------------------------------------ CPU reference (oracle port)
def cpu_sample(scene, cams, tiles, seconds, seed=0, max_tiles=None, keep=None):
    """Render + compose random 32x32 tiles with the C oracle (the reference's
    algorithm restated, every fixed march step evaluated) on all host cores
    until ``seconds`` elapse; returns (rays, elapsed, tiles used).  ``keep``
    (dict): also collect every tile's composed (rgba, depth) by tile index
    and the summed RenderCounters (the verify leg's reference frame)."""
    from oracle import oracle as O
    from paper_2303_04086_b200.model import RenderCounters
    oas = [(O.Asset(a), tr) for a, tr in scene]
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(tiles))
    rays, t0, used = 0, time.perf_counter(), 0
    nthr = os.cpu_count()        # explicit: torchrun exports OMP_NUM_THREADS=1
    cnt = RenderCounters() if keep is not None else None
    for t in order:
        c, x0, y0, x1, y1 = (int(v) for v in tiles[t])
        rg, dp = [], []
        for oa, tr in oas:
            r, d = O.render_rect(oa, cams[c], (x0, y0, x1, y1), counters=cnt, transform=tr, nthreads=nthr)
            rg.append(r)
            dp.append(d)
        out = O.compose(np.stack(rg), np.stack(dp), nthreads=nthr)
        if keep is not None:
            keep[int(t)] = out
        rays += (x1 - x0) * (y1 - y0)
        used += 1
        if time.perf_counter() - t0 >= seconds or (max_tiles and used >= max_tiles):
            break
    if keep is not None:
        keep["counters"] = cnt
    return rays, time.perf_counter() - t0, used


def verify_vs_oracle(R, N, cams, tiles, my_tiles, n_max, stride, W, H, n_views, kept, mlp):
    """The timed launch path's frame vs the oracle's (N=1): the same camera
    re-rendered (1) into a prefilled encode_frame buffer exactly as a timed
    step does (same launch sizes, so the same auto-selected variants) and
    (2) with f32 outputs through the same march / shade path; compared on
    every tile the oracle rendered: depth bits, hit pattern, counters
    (when the oracle covered the whole frame), rgba within the MLP mode's
    tolerance, encode_frame bytes."""
    import torch
    from oracle import oracle as O
    dev = my_tiles.device
    NPX = n_views * H * W
    enc = {"rgba8": torch.zeros((NPX, 4), dtype=torch.uint8, device=dev),
           "depth16": torch.full((NPX,), -1, dtype=torch.int16, device=dev),
           "counters": torch.zeros(4, dtype=torch.int64, device=dev)}
    from paper_2303_04086_b200 import render as RM
    R.render(cams, my_tiles, n_max, stride, enc, frame_layout=True, prefilled=True)
    variant = RM.last_launch()
    f32 = R.alloc(n_max, stride, want_f32=True, want_u8=False)
    R.render(cams, my_tiles, n_max, stride, f32, frame_layout=True)
    torch.cuda.synchronize()
    g_rgba = f32["rgba"][:NPX].cpu().numpy().reshape(n_views, H, W, 4)
    g_depth = f32["depth"][:NPX].cpu().numpy().reshape(n_views, H, W)
    g_r8 = enc["rgba8"].cpu().numpy().reshape(n_views, H, W, 4)
    g_d16 = enc["depth16"].cpu().numpy().view(np.uint16).reshape(n_views, H, W)
    cnt = f32["counters"].cpu().numpy()
    rgba_err, lsb, depth_bad, d16_bad, covered, px = 0.0, 0, 0, 0, 0, 0
    for t, (o_rgba, o_depth) in ((k, v) for k, v in kept.items() if k != "counters"):
        c, x0, y0, x1, y1 = (int(v) for v in tiles[t])
        gr, gd = g_rgba[c, y0:y1, x0:x1], g_depth[c, y0:y1, x0:x1]
        rgba_err = max(rgba_err, float(np.abs(gr.astype(np.float64) - o_rgba).max()))
        depth_bad += int((~((gd == o_depth) | (np.isinf(gd) & np.isinf(o_depth)))).sum())
        e8, e16 = O.encode_frame(o_rgba, o_depth)
        lsb = max(lsb, int(np.abs(g_r8[c, y0:y1, x0:x1].astype(np.int32) - e8).max()))
        d16_bad += int((g_d16[c, y0:y1, x0:x1] != e16).sum())
        covered += int(np.isfinite(o_depth).sum())
        px += o_depth.size
    oc = kept["counters"]
    full = px == NPX
    tol = 1e-3 if mlp == "fp32" else 2.0 / 255.0
    # fp32: every depth bit equal; bf16: compose's alpha_vis = 0.5 test may flip
    # on layers whose alpha is within the MLP's error of 0.5 (a few pixels)
    depth_ok = depth_bad == 0 if mlp == "fp32" else depth_bad <= max(3, covered // 500)
    counters_ok = (not full) or (int(cnt[2]) == oc.hit_pixels and int(cnt[3]) == oc.march_samples)
    return {
        "what": "timed launch path (same camera as the last timed step) vs the C oracle (pinned to the "
                "reference goldens, every march step evaluated) on every tile the cpu_baseline leg rendered",
        "launch_variant": variant, "tiles_checked": len(kept) - 1, "pixels_checked": px,
        "full_frame": full, "covered_pixels": covered,
        "depth_mismatched_px": depth_bad, "depth16_mismatched_px": d16_bad,
        "rgba_max_abs_err": rgba_err, "rgba_tol": tol, "rgba8_max_lsb": lsb,
        "counters": {"gpu_hits": int(cnt[2]), "gpu_march_samples": int(cnt[3]),
                     "oracle_hits": oc.hit_pixels if full else None,
                     "oracle_march_samples": oc.march_samples if full else None},
        "pass": bool(depth_ok and counters_ok and rgba_err <= tol and lsb <= (1 if mlp == "fp32" else 3)),
    }


def run_reference(args):
    """The reference arm: the reference's algorithm (the C oracle port of
    radfarm's render_rays + compose, every fixed march step evaluated) on the
    box's host cores.  Nothing of the product is loaded in this process: the
    synthetic assets are built (or found cached) by a child process first,
    and this process only reads the .nolf files (pure Python) and maps the
    oracle library."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cmd = [sys.executable, os.path.abspath(__file__), "--build-assets", "--config", str(args.config),
           "--assets", str(args.assets)]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    subprocess.run(cmd, check=True, env=env, stdout=subprocess.DEVNULL)
    from oracle import oracle as O
    from paper_2303_04086_b200.render import frame_tiles   # numpy only; no native library
    O.build()
    scene, views, W, H, desc = workload(args, cache_only=True)
    n_views = len(views(0))
    tiles = np.concatenate([frame_tiles(W, H, args.tile, cam=v) for v in range(n_views)])
    cores = os.cpu_count()
    per_step_tiles = 24
    for w in range(args.warmup):
        cpu_sample(scene, views(0), tiles, 1e9, seed=1000 + w, max_tiles=4)
    rays = 0
    el = 0.0
    for k in range(args.steps):
        r, e, _ = cpu_sample(scene, views(k), tiles, 1e9, seed=k, max_tiles=per_step_tiles)
        rays += r
        el += e
    value = rays / el / 1e6
    npix = n_views * W * H
    sample = (f"{args.steps} steps x {per_step_tiles} random {args.tile}x{args.tile} tiles of "
              f"{desc} ({len(scene)} assets each, oracle render + compose on {cores} threads), "
              f"extrapolated to Mrays/s")
    cfg = workload_config(args, desc, W, H, len(scene))
    cfg["workload"] = (f"{desc}, {args.tile}x{args.tile} ray tiles: render_rays of every asset + "
                       f"compose (f32 frame; no encode_frame), CPU")
    cfg["parallelism"] = f"{cores} host threads (OpenMP over rays)"
    cfg.pop("mlp", None)
    cfg.pop("partition", None)
    cfg.pop("l2", None)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "fps": value * 1e6 / npix,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64+fp32",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def build_assets(args):
    """--build-assets: synthesise (or find cached) the config's assets, then exit."""
    import torch
    if torch.cuda.is_available():
        torch.cuda.set_device(0)
    workload(args)


def workload_config(args, desc, W, H, n_assets):
    return {"workload": (f"{desc}, {args.tile}x{args.tile} ray tiles (tile rows interleaved over "
                         f"ranks), encode_frame rgba8+u16 assembled into one frame on rank 0"),
            "assets": n_assets, "width": W, "height": H,
            "atlas_b": 32, "atlas_r": 8, "psh_resolution": 64, "mlp": args.mlp,
            "parallelism": f"ray-tile x{args.gpus}", "partition": args.partition,
            "l2": ("NOT flushed (diagnostic run)" if args.no_flush else
                   "flushed between timed steps (256 MiB write)")}


# ------------------------------------------------------------------ end to end (sparse frames)
def run_e2e_sparse(args, R, N, cam_arrays, n_cam, mine, my_tiles, n_max, stride, W, H, n_views, world, rank,
                   dev, out, scene, flush=None):
    """End to end through the public API, host wall clock: every step uploads
    its camera block, renders, packs ONLY the live chunks (the pixels any
    screen box reaches; the rest of the frame is the miss encoding), moves
    them to pinned host memory in one DMA and rebuilds the full encode_frame
    RAW frame in host memory on host threads (nolf_host_scatter).  A 3-stage
    pipeline: step k+1 renders while step k's pack is copied and step k-1 is
    scattered.  With N ranks every rank rebuilds its own tile rows of one
    shared host frame (POSIX shared memory) over its own PCIe link."""
    import ctypes
    import torch
    import torch.distributed as dist
    from multiprocessing import resource_tracker, shared_memory
    n_chunks = n_max * stride // 128
    NPX = n_views * H * W
    tl = np.ascontiguousarray(mine, np.int32)
    NP = 3                              # pack buffers: render k+1 / copy k / scatter k-1
    dpack = [torch.empty(n_chunks * 16 * 48, dtype=torch.uint8, device=dev) for _ in range(NP)]
    dids = [torch.empty(n_chunks * 3, dtype=torch.int32, device=dev) for _ in range(NP)]
    dcnt = [torch.zeros(2, dtype=torch.int32, device=dev) for _ in range(NP)]
    hpack = [torch.empty(n_chunks * 16 * 48, dtype=torch.uint8, pin_memory=True) for _ in range(NP)]
    hids = [torch.empty(n_chunks * 3, dtype=torch.int32, pin_memory=True) for _ in range(NP)]
    # the render's counts mirrored into host-mapped memory by a one-warp kernel
    # (no copy-engine operation between the frames of the compute stream)
    hcnt = np.zeros((NP, 2), np.uint32)
    hcnt_dev = ctypes.c_void_p()
    N.check(N.lib().nolf_host_register(hcnt.ctypes.data, hcnt.nbytes, ctypes.byref(hcnt_dev)))
    # the host frames (2, rotating): one shared block for all ranks
    FB = NPX * 6
    name = f"nolf_sparse_{os.environ.get('MASTER_PORT', 'solo')}_{os.environ.get('TORCHELASTIC_RUN_ID', os.getpid())}"
    shm = anon = None
    if world == 1:
        # one process: private anonymous memory with transparent huge pages
        # (the scatter's random 48 B writes walk a 2 MB-page frame: far
        # fewer TLB misses than on 4 KB shared-memory pages)
        import mmap
        anon = mmap.mmap(-1, 2 * FB, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if hasattr(mmap, "MADV_HUGEPAGE"):
            try:
                anon.madvise(mmap.MADV_HUGEPAGE)
            except OSError:
                pass
        hf = np.ndarray((2 * FB,), np.uint8, buffer=anon)
    else:
        if rank == 0:
            shm = shared_memory.SharedMemory(name=name, create=True, size=2 * FB)
        dist.barrier()
        if rank != 0:
            shm = shared_memory.SharedMemory(name=name)
            resource_tracker.unregister(shm._name, "shared_memory")
        hf = np.ndarray((2 * FB,), np.uint8, buffer=shm.buf)
    for fb in range(2):                 # miss encoding (each rank its own rows would do; rank 0 all)
        if rank == 0:
            hf[fb * FB:fb * FB + NPX * 4] = 0
            hf[fb * FB + NPX * 4:(fb + 1) * FB] = 0xFF
    if world > 1:
        dist.barrier()
    dirty = [np.zeros(n_chunks, np.uint16) for _ in range(2)]     # per host frame: runs holding hits
    comp = torch.cuda.current_stream()
    copy_stream = torch.cuda.Stream(device=dev)
    ev_r = [torch.cuda.Event() for _ in range(NP)]
    ev_c = [None] * NP
    n_of = [0] * NP
    bytes_d2h = [0]

    ev_dev = []                          # (start, end) device events of every render (diagnostic)

    def render(k):
        b = k % NP
        if ev_c[b] is not None:
            comp.wait_event(ev_c[b])                 # pack buffer b copied out (step k-2)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        o = {"pack": dpack[b], "pack_ids": dids[b], "pack_count": dcnt[b], "counters": out["counters"]}
        if flush is not None:
            flush.fill_(k & 0x7F)                    # L2 evicted before every frame, inside the wall clock
        R.render(cam_arrays[k % n_cam], my_tiles, n_max, stride, o, frame_layout=True, prefilled=True)
        N.check(N.lib().nolf_store_u32(hcnt_dev.value + 8 * b, dcnt[b].data_ptr(), 2, comp.cuda_stream))
        ev_r[b].record(comp)
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(comp)
        ev_dev.append((e0, e1))

    tm = {"wait_render": 0.0, "scatter": 0.0, "wait_copy": 0.0, "enqueue": 0.0}

    def copy(k):
        b = k % NP
        t = time.perf_counter()
        ev_r[b].synchronize()
        tm["wait_render"] += time.perf_counter() - t
        n, nr = (int(v) for v in hcnt[b])             # landed: the event follows the store kernel
        n_of[b] = n
        copy_stream.wait_event(ev_r[b])
        with torch.cuda.stream(copy_stream):
            hpack[b][:nr * 48].copy_(dpack[b][:nr * 48], non_blocking=True)
            hids[b][:3 * n].copy_(dids[b][:3 * n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(copy_stream)
        ev_c[b] = ev
        bytes_d2h[0] += nr * 48 + n * 12 + 8

    def scatter(k):                      # on the scatter thread
        b, f = k % NP, k % 2
        t = time.perf_counter()
        ev_c[b].synchronize()
        t1 = time.perf_counter()
        base = hf.ctypes.data + f * FB
        N.check(N.lib().nolf_host_scatter(hpack[b].data_ptr(), hids[b].data_ptr(), n_of[b], tl.ctypes.data,
                                          len(tl), stride, W, H, base, base + NPX * 4, dirty[f].ctypes.data, 0))
        tm["wait_copy"] += t1 - t
        tm["scatter"] += time.perf_counter() - t1

    from concurrent.futures import ThreadPoolExecutor
    worker = ThreadPoolExecutor(1)       # ctypes drops the GIL: host scatter overlaps the next enqueue
    pend = [None]

    def submit(k):
        if pend[0] is not None:
            pend[0].result()
        pend[0] = worker.submit(scatter, k)

    def run(steps):
        render(0)
        for k in range(steps):
            if k + 1 < steps:
                t = time.perf_counter()
                render(k + 1)
                tm["enqueue"] += time.perf_counter() - t
            copy(k)
            if k >= 1:
                submit(k - 1)
        submit(steps - 1)
        pend[0].result()

    run(4)                               # warm-up (pool threads, pinned pages)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    bytes_d2h[0] = 0
    for key in tm:
        tm[key] = 0.0
    ev_dev.clear()
    N.check(N.lib().nolf_profile(1))
    t0 = time.perf_counter()
    run(args.steps)
    el = time.perf_counter() - t0
    torch.cuda.synchronize()
    kms = (ctypes.c_float * 3)()
    n_prof = N.lib().nolf_profile_read(kms)
    N.check(N.lib().nolf_profile(0))
    e2e_kernel_us = [round(1e3 * float(v) / max(n_prof, 1), 1) for v in kms[:3]]
    dev_us = 1e3 * float(np.mean([a.elapsed_time(b) for a, b in ev_dev])) if ev_dev else None
    gap_us = (1e3 * float(np.mean([ev_dev[i][1].elapsed_time(ev_dev[i + 1][0]) for i in range(len(ev_dev) - 1)]))
              if len(ev_dev) > 1 else None)
    te = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    npix = NPX
    e2e = {"value": args.steps * npix / float(te.item()) / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": int(N.lib().nolf_launch_param_bytes(len(scene), n_views)),
           "d2h_bytes_per_step": int(bytes_d2h[0] / args.steps),
           "timing": "host wall clock (perf_counter) from the first render to the last frame rebuilt in "
                     "host memory, max over ranks; L2 flushed (256 MiB write) before every render, inside "
                     "the timed window",
           "mode": ("sparse frame: compose packs the non-miss 8-pixel runs of the live chunks (48 B "
                    "each + a 12 B header per live chunk), one DMA per step to pinned host memory, "
                    "nolf_host_scatter rebuilds the full encode_frame RAW frame (rgba8 + u16 depth) in "
                    "host memory on host threads, touching only runs that change (render k+1 / copy k / "
                    "scatter k-1 pipelined, the scatter on its own host thread)"),
           "full_frame_bytes": int(npix * 6),
           "host_us_per_step": {key: round(v / args.steps * 1e6, 1) for key, v in tm.items()},
           "device_us_per_step": {"render": round(dev_us, 1) if dev_us is not None else None,
                                  "gap_between_renders": round(gap_us, 1) if gap_us is not None else None,
                                  "k_march": e2e_kernel_us[0], "k_shade": e2e_kernel_us[1],
                                  "k_compose": e2e_kernel_us[2]},
           "host_threads": int(os.environ.get("NOLF_HOST_THREADS",
                                              max(1, os.cpu_count() // (2 * int(os.environ.get("LOCAL_WORLD_SIZE", "1"))))))}
    last = (args.steps - 1) % 2
    frame_copy = torch.from_numpy(hf[last * FB:(last + 1) * FB].copy())
    worker.shutdown()
    N.lib().nolf_host_unregister(hcnt.ctypes.data)
    if world > 1:
        dist.barrier()
    del hf
    if shm is not None:
        try:
            shm.close()
        except BufferError:
            pass
        dist.barrier()
        if rank == 0:
            shm.unlink()
    else:
        try:
            anon.close()
        except BufferError:
            pass
    return e2e, (args.steps - 1, frame_copy), None


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2303_04086_b200 import _native as N
    from paper_2303_04086_b200 import build as B
    from paper_2303_04086_b200.dist import (gather_to_root, partition, rank_buffer_bytes, row_bands,
                                            shard_tiles, slot_tile_table)
    from paper_2303_04086_b200.render import SceneRenderer, frame_tiles
    B.build()

    scene, views, W, H, desc = workload(args)
    n_views = len(views(0))
    R = SceneRenderer(scene)
    from paper_2303_04086_b200 import render as RM
    RM.set_option(N.OPT_MARCH_ORDER, {"auto": 0, "spatial": 1, "heavy": 2}[args.march_order])
    RM.set_option(N.OPT_CHUNK_COST, args.chunk_cost)
    if args.mlp == "bf16":
        R.mlp_mode(N.MLP_BF16)
    T = args.tile
    stride = T * T
    tiles = np.concatenate([frame_tiles(W, H, T, cam=v) for v in range(n_views)])
    n_tiles = len(tiles)
    # rank 0 also re-clears the consumed frame buffers and waits on the flags:
    # --rank0-weight < 1 gives it proportionally fewer tile rows
    w0 = args.rank0_weight if args.rank0_weight is not None else (0.9 if n_views > 1 else 1.0)
    weights = [w0] + [1.0] * (world - 1) if world > 1 else None
    parts = partition(tiles, world, T, by_rows=args.partition == "rows", weights=weights)
    mine, n_max = shard_tiles(tiles, world, rank, parts)
    my_tiles = torch.from_numpy(mine).to(dev)
    P = n_max * stride
    buf = torch.empty(rank_buffer_bytes(n_max, stride), dtype=torch.uint8, device=dev)  # rgba8 | depth16
    rgba8 = buf[:P * 4]
    depth16 = buf[P * 4:]
    out = R.alloc(n_max, stride, want_f32=False, want_u8=False)
    out["rgba8"] = rgba8
    out["depth16"] = depth16
    gathered = torch.empty(world * P * 6, dtype=torch.uint8, device=dev) if world > 1 else None
    # tile of every (rank, slot) in rank-major gather order, for frame assembly
    slot_tiles_dev = torch.from_numpy(slot_tile_table(tiles, world, parts)).to(dev)
    # two frame buffers so the end-to-end loop can download frame k while
    # frame k+1 renders
    NPX = n_views * H * W
    frames = [(torch.empty((NPX, 4), dtype=torch.uint8, device=dev),
               torch.empty((NPX,), dtype=torch.int16, device=dev)) for _ in range(2)]
    # 256 MiB (2x the 126 MB L2) written as int32: 16 B vector stores, ~7 TB/s
    # (a uint8 fill runs at half that rate)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    if os.environ.get("NOLF_FLUSH_U8"):             # diagnostic: the byte-wise fill
        flush = flush.view(torch.uint8)
    n_cam = args.warmup + args.steps + 4
    cam_arrays = [R.camera_array(views(k)) for k in range(n_cam)]
    R.reserve(cam_arrays, n_max * stride)
    split = None
    if args.split == 2:                  # two interleaved halves of this rank's tiles, two streams
        halves = [np.ascontiguousarray(mine[0::2]), np.ascontiguousarray(mine[1::2])]
        R2 = SceneRenderer(scene)
        if args.mlp == "bf16":
            R2.mlp_mode(N.MLP_BF16)
        R2.reserve(cam_arrays, len(halves[1]) * stride)
        split = {"tiles": [torch.from_numpy(h).to(dev) for h in halves], "n": [len(h) for h in halves],
                 "side": torch.cuda.Stream(device=dev), "R": [R, R2]}

    def render_tiles(cams, o, **kw):
        """This rank's tiles: one render, or (--split 2) two halves on two streams."""
        if split is None:
            R.render(cams, my_tiles, n_max, stride, o, **kw)
            return
        main = torch.cuda.current_stream()
        side = split["side"]
        side.wait_stream(main)
        split["R"][0].render(cams, split["tiles"][0], split["n"][0], stride, o, **kw)
        with torch.cuda.stream(side):
            split["R"][1].render(cams, split["tiles"][1], split["n"][1], stride, o, stream=side.cuda_stream, **kw)
        main.wait_stream(side)
    stream = torch.cuda.current_stream().cuda_stream

    # ---- p2p frame composer: rank 0 owns the frame buffers, every rank maps
    # them (CUDA IPC) and its compose kernel stores straight into them
    if args.exchange == "dma" and args.partition != "rows":
        args.exchange = "p2p"            # strided band copies need the row partition
    p2p = world > 1 and args.exchange in ("p2p", "dma")
    dma = p2p and args.exchange == "dma" and rank != 0
    bands_dev = row_bands(world, rank, n_views, W, H, T, weights) if dma else []
    peer_frames = []
    token = torch.zeros(1, dtype=torch.float32, device=dev)
    NB = max(2, args.frames) if (p2p and args.sync == "flags") else 2   # frame buffers in the ring
    if p2p:
        import ctypes
        FB = NPX * 6
        hbuf = torch.zeros(NB * 64, dtype=torch.uint8, device=dev)
        raw = []
        if rank == 0:
            hh = (ctypes.c_uint8 * (64 * NB))()
            for i in range(NB):
                ptr = ctypes.c_void_p()
                N.check(N.lib().nolf_device_alloc(FB, ctypes.byref(ptr)))
                N.check(N.lib().nolf_ipc_get_handle(ptr, ctypes.byref(hh, 64 * i)))
                raw.append(ptr.value)
            hbuf.copy_(torch.tensor(list(bytes(hh)), dtype=torch.uint8))
        dist.broadcast(hbuf, src=0)
        if rank != 0:
            hh = (ctypes.c_uint8 * (64 * NB))(*hbuf.cpu().tolist())
            for i in range(NB):
                ptr = ctypes.c_void_p()
                N.check(N.lib().nolf_ipc_open_handle(ctypes.byref(hh, 64 * i), ctypes.byref(ptr)))
                raw.append(ptr.value)
        peer_frames = [(p, p + NPX * 4) for p in raw]

    # ---- frame-completion flags (p2p, --sync flags): rank 0 owns done[world]
    # (peer r sets done[r] = seq after its stores), every peer owns free
    # (rank 0 sets it = seq once frame seq is consumed, so a peer reuses a
    # frame buffer only after rank 0 is done with it: a ring of --frames buffers)
    flags = p2p and args.sync == "flags"
    seq_box = [0]
    timeout_flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if flags:
        import ctypes

        def alloc_flag(nwords):
            ptr = ctypes.c_void_p()
            N.check(N.lib().nolf_device_alloc(4 * nwords, ctypes.byref(ptr)))
            N.check(N.lib().nolf_memcpy_async(ptr, torch.zeros(nwords, dtype=torch.int32, device=dev).data_ptr(),
                                              4 * nwords, stream))
            torch.cuda.synchronize()
            hh = (ctypes.c_uint8 * 64)()
            N.check(N.lib().nolf_ipc_get_handle(ptr, ctypes.byref(hh)))
            return ptr.value, torch.tensor(list(bytes(hh)), dtype=torch.uint8, device=dev)

        def open_flag(h):
            hh = (ctypes.c_uint8 * 64)(*h.cpu().tolist())
            ptr = ctypes.c_void_p()
            N.check(N.lib().nolf_ipc_open_handle(ctypes.byref(hh), ctypes.byref(ptr)))
            return ptr.value

        own, own_h = alloc_flag(max(world, 1))           # rank 0: done[world]; peers: free
        hs = [torch.zeros(64, dtype=torch.uint8, device=dev) for _ in range(world)]
        dist.all_gather(hs, own_h)
        done_remote = open_flag(hs[0]) if rank != 0 else own
        free_remote = [open_flag(hs[j]) for j in range(1, world)] if rank == 0 else []

    # Frame buffers are pre-set to the miss encoding by their owner (rank 0 /
    # the single GPU) so compose stores only chunks some instance reaches
    # (with peers: ~80 % fewer NVLink stores).  A consumed buffer is queued for
    # re-clearing; the clear runs on a side stream once the NEXT step has
    # started (so it overlaps rendering, never the untimed L2 flush), then the
    # peers' "free" flags are set and the owner's next render into that buffer
    # waits for it.
    prefill = args.prefill != "off" and ((flags and not dma) or world == 1)
    state_mode = prefill and args.prefill == "state"   # run dirty bits instead of re-clearing
    owner = world == 1 or rank == 0
    last_fb = [0]
    n_my_chunks = n_max * stride // 128
    chunk_states = [torch.zeros(n_my_chunks, dtype=torch.int16, device=dev) for _ in range(NB if p2p else 2)] \
        if state_mode else None

    def clear(fb, s):
        """miss encoding (rgba8 0, depth16 65535) over frame buffer fb, on its owner GPU"""
        if p2p:
            rgba_ptr, d_ptr = peer_frames[fb]
        else:
            rgba_ptr, d_ptr = frames[fb][0].data_ptr(), frames[fb][1].data_ptr()
        N.check(N.lib().nolf_memset_async(rgba_ptr, 0, NPX * 4, s))
        N.check(N.lib().nolf_memset_async(d_ptr, 0xFF, NPX * 2, s))

    clear_stream = torch.cuda.Stream(device=dev) if (prefill and owner and not state_mode) else None
    clear_ev = [None] * NB
    pending = []

    def release(fb, seq, ts):
        """owner: buffer fb (frame seq, None at 1 GPU) consumed on torch stream ts"""
        if prefill and not state_mode:
            ev = torch.cuda.Event()
            ev.record(ts)
            pending.append((fb, seq, ev))
        elif seq is not None:
            for ptr in free_remote:
                N.check(N.lib().nolf_flag_set(ptr, seq, ts.cuda_stream))

    def flush_pending():
        if not pending:
            return
        start = torch.cuda.Event()
        start.record(torch.cuda.current_stream())      # inside this step's timed window
        clear_stream.wait_event(start)
        for fb, seq, ev in pending:
            clear_stream.wait_event(ev)
            clear(fb, clear_stream.cuda_stream)
            if seq is not None:
                for ptr in free_remote:
                    N.check(N.lib().nolf_flag_set(ptr, seq, clear_stream.cuda_stream))
            cev = torch.cuda.Event()
            cev.record(clear_stream)
            clear_ev[fb] = cev
        pending.clear()

    if prefill and owner:
        for i in range(NB if p2p else 2):
            clear(i, stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def reset_frames():
        """back to miss-encoded buffers and empty chunk states (after renders
        that bypassed the states, e.g. the hostmap e2e loop)"""
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if prefill and owner:
            for i in range(NB if p2p else 2):
                clear(i, stream)
        if state_mode:
            for st_ in chunk_states:
                st_.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def step(k, fb=0, before_barrier=None, auto_release=True):
        if prefill and owner and not state_mode:
            flush_pending()
        if p2p and flags:
            seq_box[0] += 1
            seq = seq_box[0]
            fb = seq % NB                  # the buffer ring rotates by frame sequence
            last_fb[0] = fb
            if rank != 0 and seq > NB:     # buffer fb held frame seq-NB: wait until rank 0 is done
                N.check(N.lib().nolf_flag_wait(own, 1, seq - NB, timeout_flag.data_ptr(), stream))
        if p2p:
            if dma:
                # compose into this GPU's own frame (local HBM stores), then
                # the copy engine moves its tile-row bands into rank 0's frame
                # over NVLink (one strided 2-D copy per plane)
                frame, frame_d = frames[fb]
                o2 = {"rgba8": frame, "depth16": frame_d, "counters": out["counters"]}
                R.render(cam_arrays[k % n_cam], my_tiles, n_max, stride, o2, frame_layout=True)
                for first, wpx, ppx, hgt in bands_dev:
                    for bpp, dst0, src0 in ((4, peer_frames[fb][0], frame.data_ptr()),
                                            (2, peer_frames[fb][1], frame_d.data_ptr())):
                        N.check(N.lib().nolf_memcpy2d_async(dst0 + first * bpp, ppx * bpp, src0 + first * bpp,
                                                            ppx * bpp, wpx * bpp, hgt, stream))
            else:
                o2 = {"rgba8": peer_frames[fb][0], "depth16": peer_frames[fb][1],
                      "counters": out["counters"]}
                if state_mode:
                    o2["chunk_state"] = chunk_states[fb]
                if rank == 0 and clear_ev[fb] is not None:
                    torch.cuda.current_stream().wait_event(clear_ev[fb])   # buffer re-cleared
                render_tiles(cam_arrays[k % n_cam], o2, frame_layout=True, peer=(rank != 0), prefilled=prefill)
            if flags:
                if rank != 0:
                    N.check(N.lib().nolf_flag_set(done_remote + 4 * rank, seq, stream))
                else:                      # every peer's stores for frame seq have landed
                    N.check(N.lib().nolf_flag_wait(own + 4, world - 1, seq, timeout_flag.data_ptr(), stream))
                    if before_barrier is not None:
                        torch.cuda.current_stream().wait_event(before_barrier)
                    if auto_release:
                        release(fb, seq, torch.cuda.current_stream())
                return
            if before_barrier is not None:
                torch.cuda.current_stream().wait_event(before_barrier)
            dist.all_reduce(token)         # every rank's peer stores have landed
            return
        frame, frame_d = frames[fb]
        last_fb[0] = fb
        if world == 1:             # single GPU: compose writes the frame directly
            out["rgba8"], out["depth16"] = frame, frame_d
            if state_mode:
                out["chunk_state"] = chunk_states[fb]
            if prefill and clear_ev[fb] is not None:
                torch.cuda.current_stream().wait_event(clear_ev[fb])   # buffer re-cleared
        if world == 1:
            render_tiles(cam_arrays[k % n_cam], out, frame_layout=True, prefilled=prefill)
        else:
            R.render(cam_arrays[k % n_cam], my_tiles, n_max, stride, out, frame_layout=False, prefilled=False)
        if world == 1 and auto_release:
            release(fb, None, torch.cuda.current_stream())
        if world > 1:
            # frame composer: NCCL gather of every rank's encoded tiles, then
            # one unpack kernel writes the row-major frame on rank 0
            gather_to_root(buf, gathered, world, rank)
            if rank == 0:
                N.check(N.lib().nolf_unpack_gathered(gathered.data_ptr(), world, n_max, stride,
                                                     slot_tiles_dev.data_ptr(), W, H,
                                                     frame.data_ptr(), frame_d.data_ptr(), stream))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = Clocks(local).__enter__()
    clk.wait_first()
    for k in range(args.warmup):
        step(k)
    barrier()
    out["counters"].zero_()
    import ctypes
    kms = (ctypes.c_float * 3)()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    barrier()
    N.check(N.lib().nolf_profile(1))
    h0 = time.perf_counter()
    # the host enqueues every step without waiting (as a serving loop would);
    # each step is bracketed by device events, the L2 flush sits between them
    for k in range(args.steps):
        if not args.no_flush:
            flush.fill_(k & 0x7F)                          # evict L2 (untimed)
        ev[k][0].record()
        step(args.warmup + k, k % 2)
        ev[k][1].record()
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps   # host enqueue rate (diagnostic)
    barrier()
    n_prof = N.lib().nolf_profile_read(kms)
    if n_prof < 0:
        N.check(n_prof)
    kern = np.array(kms[:3], dtype=np.float64) * (args.steps / max(n_prof, 1))
    N.check(N.lib().nolf_profile(0))
    clk.mark(h0, time.perf_counter())
    clk.__exit__()
    step_ms = np.array([a.elapsed_time(b) for a, b in ev])
    t_local = float(step_ms.sum()) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    # per-rank kernel time (march + shade + compose per step), for imbalance
    csum = clk.summary()
    kr = torch.tensor(list(kern / args.steps) + [csum["sm_mhz"] or 0.0, host_ms], dtype=torch.float64, device=dev)
    rank_kernel_ms = [[round(float(v), 4) for v in kr.tolist()]]
    if world > 1:
        allk = [torch.zeros_like(kr) for _ in range(world)]
        dist.all_gather(allk, kr)
        rank_kernel_ms = [[round(float(v), 4) for v in x.tolist()] for x in allk]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    from paper_2303_04086_b200 import render as RM
    launch = RM.last_launch()          # the variants the timed steps launched
    cnt = out["counters"].cpu().numpy().astype(np.float64) / args.steps
    if os.environ.get("NOLF_STATS_DUMP") and hasattr(N.lib(), "nolf_stats_read"):
        import ctypes                # diagnostic build (-DNOLF_STATS): march work counters
        st = (ctypes.c_ulonglong * 16)()
        N.lib().nolf_stats_read(st, 0)
        print("STATS per frame", [round(v / (args.steps + args.warmup), 1) for v in st], file=sys.stderr)
    npix = NPX
    value = args.steps * npix / t_max / 1e6

    # ---- end to end: camera in (H2D param block), encoded frame out to host memory
    e2e = None
    shm = host_map = None
    if args.partition == "tiles" and args.e2e_mode == "hostmap":
        args.e2e_mode = "copy"          # strided row DMA needs the row partition
    sparse_host = None
    if not args.no_e2e and args.e2e_mode == "sparse":
        e2e, sparse_host, shm = run_e2e_sparse(args, R, N, cam_arrays, n_cam, mine, my_tiles, n_max, stride, W, H,
                                               n_views, world, rank, dev, out, scene,
                                               flush=None if args.no_flush else flush)
    elif not args.no_e2e and args.e2e_mode == "hostmap":
        # One shared page-locked host frame stack (double buffered) mapped by
        # every rank.  Each rank composes its tile rows into its own device
        # frame and one strided DMA per buffer (cudaMemcpy2DAsync, on a copy
        # stream, overlapping the next render) moves its rows to the host
        # over its own PCIe link; a 1-element all-reduce on the copy stream
        # marks the frame complete.  Timed from the first render to the last
        # rank's completion (device events, max over ranks).
        import ctypes
        from multiprocessing import resource_tracker, shared_memory
        FB = NPX * 6
        name = f"nolf_frame_{os.environ.get('MASTER_PORT', 'solo')}_{os.environ.get('TORCHELASTIC_RUN_ID', os.getpid())}"
        if rank == 0:
            shm = shared_memory.SharedMemory(name=name, create=True, size=2 * FB)
        if world > 1:
            dist.barrier()
        if rank != 0:
            shm = shared_memory.SharedMemory(name=name)
            resource_tracker.unregister(shm._name, "shared_memory")   # rank 0 owns it
        host_addr = ctypes.addressof(ctypes.c_char.from_buffer(shm.buf))
        dptr = ctypes.c_void_p()
        N.check(N.lib().nolf_host_register(host_addr, 2 * FB, ctypes.byref(dptr)))
        host_map = [host_addr + fb * FB for fb in range(2)]
        bands = row_bands(world, rank, n_views, W, H, T, weights)
        copy_stream = torch.cuda.Stream(device=dev)
        comp = torch.cuda.current_stream()
        done_copy = [None, None]

        def step_host(k, fb):
            if done_copy[fb] is not None:
                comp.wait_event(done_copy[fb])              # device frame fb free again
            frame, frame_d = frames[fb]
            o2 = {"rgba8": frame, "depth16": frame_d, "counters": out["counters"]}
            R.render(cam_arrays[k % n_cam], my_tiles, n_max, stride, o2, frame_layout=True)
            rendered = torch.cuda.Event()
            rendered.record(comp)
            copy_stream.wait_event(rendered)
            cs = copy_stream.cuda_stream
            for first, wpx, ppx, hgt in bands:
                for bpp, dst0, src0 in ((4, host_map[fb], frame.data_ptr()),
                                        (2, host_map[fb] + NPX * 4, frame_d.data_ptr())):
                    N.check(N.lib().nolf_memcpy2d_async(dst0 + first * bpp, ppx * bpp, src0 + first * bpp,
                                                        ppx * bpp, wpx * bpp, hgt, cs))
            if world > 1:
                with torch.cuda.stream(copy_stream):
                    dist.all_reduce(token)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
            done_copy[fb] = ev

        for k in range(2):
            step_host(k, k % 2)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(comp)
        for k in range(args.steps):
            step_host(k, k % 2)
        comp.wait_stream(copy_stream)
        t1.record(comp)
        t1.synchronize()
        barrier()
        te = torch.tensor([t0.elapsed_time(t1) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": args.steps * npix / float(te.item()) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(N.lib().nolf_launch_param_bytes(len(scene), n_views)),
               "d2h_bytes_per_step": int(npix * 6),
               "mode": ("every rank DMAs its tile rows (strided cudaMemcpy2DAsync, copy stream) "
                        "into one shared page-locked host frame over its own PCIe link")}
    elif not args.no_e2e:
        # Pipelined: step k renders into frame buffer k%2 on the compute
        # stream; a copy stream downloads it to pinned host memory while
        # step k+1 renders.  Timed from the first render to the last byte on
        # the host (device events on both streams).
        hosts = [torch.empty((NPX * 6,), dtype=torch.uint8, pin_memory=True) for _ in range(NB)]
        copy_stream = torch.cuda.Stream(device=dev)
        comp = torch.cuda.current_stream()
        for k in range(2):
            step(k, k % 2)
        barrier()
        done_copy = [None] * NB
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(comp)
        for k in range(args.steps):
            fb = (seq_box[0] + 1) % NB if (p2p and flags) else k % 2   # the buffer step() will use
            if done_copy[fb] is not None:
                comp.wait_event(done_copy[fb])       # buffer free again
            # p2p: other ranks write buffer fb^1 at step k+1 once this step's
            # completion collective passes, so rank 0 enters it only after
            # the download of step k-1 (buffer fb^1) finished
            step(k, fb, before_barrier=done_copy[(fb - 1) % NB] if (p2p and rank == 0) else None,
                 auto_release=not (flags or world == 1))
            if rank == 0:
                rendered = torch.cuda.Event()
                rendered.record(comp)
                copy_stream.wait_event(rendered)
                with torch.cuda.stream(copy_stream):
                    if p2p:
                        N.check(N.lib().nolf_memcpy_async(hosts[fb].data_ptr(), peer_frames[fb][0],
                                                          NPX * 6, copy_stream.cuda_stream))
                    else:
                        hosts[fb][:NPX * 4].view(NPX, 4).copy_(frames[fb][0], non_blocking=True)
                        hosts[fb][NPX * 4:].view(torch.int16).copy_(frames[fb][1], non_blocking=True)
                    if flags or world == 1:   # downloaded: the buffer may be re-cleared / refilled
                        release(fb, seq_box[0] if flags else None, copy_stream)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                done_copy[fb] = ev
        comp.wait_stream(copy_stream)
        t1.record(comp)
        t1.synchronize()
        barrier()
        te = torch.tensor([t0.elapsed_time(t1) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": args.steps * npix / float(te.item()) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(N.lib().nolf_launch_param_bytes(len(scene), n_views)),
               "d2h_bytes_per_step": int(npix * 6),
               "mode": "rank 0 cudaMemcpyAsync of the assembled frame, double-buffered"}

    # ---- multi-GPU frame == single-GPU frame (bitwise)
    verify = None
    if args.verify:
        if host_map is not None or args.e2e_mode == "copy":
            reset_frames()
        kv = args.warmup + args.steps - 1
        step(kv, 0, auto_release=False)    # keep the frame until it is read back
        fbv = last_fb[0]
        barrier()
        if rank == 0:
            import ctypes
            got = torch.empty(NPX * 6, dtype=torch.uint8, device=dev)
            if p2p:
                N.check(N.lib().nolf_memcpy_async(got.data_ptr(), peer_frames[fbv][0], NPX * 6,
                                                  torch.cuda.current_stream().cuda_stream))
                if flags:
                    release(fbv, seq_box[0], torch.cuda.current_stream())
            else:
                got[:NPX * 4].copy_(frames[fbv][0].view(-1))
                got[NPX * 4:].copy_(frames[fbv][1].view(torch.uint8).view(-1))
                if world == 1:
                    release(fbv, None, torch.cuda.current_stream())
            all_tiles = torch.from_numpy(tiles.astype(np.int32)).to(dev)
            ref = {"rgba8": torch.empty((NPX, 4), dtype=torch.uint8, device=dev),
                   "depth16": torch.empty(NPX, dtype=torch.int16, device=dev),
                   "counters": torch.zeros(4, dtype=torch.int64, device=dev)}
            R.reserve([cam_arrays[kv % n_cam]], n_tiles * stride)
            R.render(cam_arrays[kv % n_cam], all_tiles, n_tiles, stride, ref, frame_layout=True)
            exp = torch.cat([ref["rgba8"].view(-1), ref["depth16"].view(torch.uint8).view(-1)])
            torch.cuda.synchronize()
            verify = {"bitwise_equal": bool(torch.equal(got, exp)),
                      "mismatched_bytes": int((got != exp).sum().item()),
                      "what": "assembled multi-GPU frame vs rank 0 rendering every tile alone"}
            if sparse_host is not None:   # last e2e frame (host memory, rebuilt from packed chunks)
                ke, hf = sparse_host
                R.render(cam_arrays[ke % n_cam], all_tiles, n_tiles, stride, ref, frame_layout=True)
                exp2 = torch.cat([ref["rgba8"].view(-1), ref["depth16"].view(torch.uint8).view(-1)])
                verify["host_frame_bitwise_equal"] = bool(torch.equal(hf, exp2.cpu()))
            if host_map is not None:      # last e2e frame (host memory) vs the same camera alone
                ke = args.steps - 1
                R.render(cam_arrays[ke % n_cam], all_tiles, n_tiles, stride, ref, frame_layout=True)
                exp2 = torch.cat([ref["rgba8"].view(-1), ref["depth16"].view(torch.uint8).view(-1)])
                FBn = NPX * 6
                hostf = torch.frombuffer(shm.buf, dtype=torch.uint8)[(ke % 2) * FBn:(ke % 2 + 1) * FBn]
                verify["host_frame_bitwise_equal"] = bool(torch.equal(hostf, exp2.cpu()))
                del hostf
        barrier()

    # ---- roofline of the dominant kernel (per-launch algorithmic bytes / event time)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    names = ["k_march", "k_shade", "k_compose"]
    ms = kern / args.steps
    S, Hh = cnt[3], cnt[2]
    npx = n_max * stride
    alg = {"k_march": 36.0 * S + 80.0 * Hh,
           "k_shade": (80.0 + 228.0 + 20.0) * Hh,
           "k_compose": 20.0 * Hh + 7.0 * npx}
    top = names[int(np.argmax(ms))]
    ach = alg[top] / (ms[names.index(top)] / 1e3) / 1e9
    # the MLP's tensor roofline: 11,136 FLOP per hit in the
    # shading kernel vs the measured dense bf16 peak (sustained: timed in a step)
    tflops_peak = float(peaks.get("bf16_tflops_sustained", 1400.0))
    t_shade = ms[names.index("k_shade")] / 1e3
    mlp_tflops = 11136.0 * Hh / t_shade / 1e12 if t_shade > 0 else 0.0
    roof = {"bound": "hbm", "kernel": top, "achieved": ach, "peak": hbm, "unit": "GB/s",
            "frac": ach / hbm, "traffic": None,
            "algorithmic_bytes_per_launch": alg[top],
            "kernel_ms": dict(zip(names, [float(x) for x in ms])),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
            "tensor": {"kernel": "k_shade_tc" if args.mlp == "bf16" else "k_shade (fp32 CUDA cores)",
                       "achieved": mlp_tflops, "peak": tflops_peak, "unit": "TFLOP/s",
                       "frac": mlp_tflops / tflops_peak, "flop_per_hit": 11136,
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}}

    # DRAM traffic of the dominant kernel from the newest committed ncu
    # capture of this config (profiles/, `ncu --set full`, per launch)
    try:
        import glob
        def _ver(path):              # r01_config4_1gpu_v10 after _v9 (numeric, not lexical)
            import re
            m = re.search(r"r(\d+)_config\d+_1gpu(?:_v(\d+))?\.json$", path)
            return (int(m.group(1)), int(m.group(2) or 0)) if m else (0, 0)
        caps = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_config{args.config}_1gpu*.json")), key=_ver)
        for path in reversed(caps):
            kern_caps = json.load(open(path)).get("kernels", {})
            # the march phase is k_cull_chunks + k_march_chunks (k_march<> for unaligned tiles)
            names_of = {"k_march": ("k_march", "k_march_chunks", "k_cull_chunks"),
                        "k_shade": ("k_shade", "k_shade_tc"), "k_compose": ("k_compose", "k_compose_live")}[top]
            hit = [v for k, v in kern_caps.items() if k.split("<")[0] in names_of]
            if hit:
                roof["traffic"] = float(sum(v["dram_bytes_per_launch"] for v in hit))
                roof["traffic_unit"] = "B/launch (dram__bytes_read.sum + dram__bytes_write.sum)"
                roof["traffic_source"] = os.path.relpath(path, ROOT)
                break
    except (OSError, ValueError, KeyError):
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle renders the last timed step's camera: timed as the CPU
        # baseline, and kept as the reference frame the timed path is verified on
        kv = args.warmup + args.steps - 1
        kept = {}
        try:
            rays, el, used = cpu_sample(scene, views(kv), tiles, args.cpu_seconds, keep=kept)
            cpu = {"value": rays / el / 1e6, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"{used} of {len(tiles)} random {T}x{T} tiles ({len(scene)} assets "
                             f"each), oracle render + compose on {os.cpu_count()} OpenMP threads, "
                             f"{el:.1f} s, extrapolated to Mrays/s"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {e}"}
        if len(kept) > 1:
            vo = verify_vs_oracle(R, N, cam_arrays[kv % n_cam], tiles, my_tiles, n_max, stride, W, H,
                                  n_views, kept, args.mlp)
            if verify is None:
                verify = vo
            else:
                verify["oracle"] = vo
    # our kernels per timed step on rank 0: k_cull_chunks + k_march_chunks +
    # k_shade_tc + k_compose (k_march alone when tiles are not 128-slot
    # aligned), + k_unpack (gather exchange) or k_flag_wait + one k_flag_set
    # per peer (flag-synchronised p2p exchange)
    launches_per_step = (4 if stride % 128 == 0 else 3)
    if world > 1 and not p2p:
        launches_per_step += 1
    elif flags:
        launches_per_step += 1 + (world - 1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
            "fps": args.steps * n_views / t_max, "views_per_step": n_views,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE if args.mlp == "bf16" else "f64+fp32", "data": "synthetic (reference-pipeline assets, "
            "random-init networks)", "config": workload_config(args, desc, W, H, len(scene)),
            "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step, "roofline": roof, "cpu_baseline": cpu,
            "clocks": csum, "verify": verify, "launch": launch,
            "rank_kernel_ms": {"fields": ["k_march", "k_shade", "k_compose", "sm_mhz", "host_enqueue_ms"],
                               "ranks": rank_kernel_ms},
            "per_frame": {"march_samples": S, "hits": Hh, "pixels": npix},
            "step_ms": {"p50": float(np.percentile(step_ms, 50)), "p90": float(np.percentile(step_ms, 90)),
                        "max": float(step_ms.max()), "min": float(step_ms.min())},
        }
        line["config"]["parallelism"] = f"ray-tile x{world}"
        if world > 1:
            line["config"]["frame_sync"] = (
                "peer-mapped completion flags (k_flag_set / k_flag_wait, no collective)"
                if flags else "1-element NCCL all-reduce" if p2p else "NCCL gather")
            if flags and int(timeout_flag.item()) != 0:
                line["config"]["frame_sync"] += " -- TIMED OUT (frames incomplete)"
            line["config"]["exchange"] = (
                "every rank composes its tile rows locally, the copy engine DMAs them into rank 0's "
                "frame over NVLink (CUDA IPC, strided 2-D copies)"
                if args.exchange == "dma" else
                "compose epilogue stores into rank 0's frame over NVLink (CUDA IPC peer memory)"
                if p2p else "NCCL gather of encoded tiles + unpack kernel")
        print(json.dumps(line), flush=True)
    if host_map is not None:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        import ctypes
        N.lib().nolf_host_unregister(ctypes.addressof(ctypes.c_char.from_buffer(shm.buf)))
        try:
            shm.close()
        except BufferError:       # a view is still referenced; the mapping dies with the process
            pass
        if world > 1:
            dist.barrier()
        if rank == 0:
            shm.unlink()
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        if p2p:
            for p in ([f[0] for f in peer_frames]):
                N.lib().nolf_ipc_close_handle(p) if rank != 0 else N.lib().nolf_device_free(p)
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.build_assets:
        build_assets(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
