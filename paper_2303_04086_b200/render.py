"""Reference-signature render entry points backed by libnolf_b200.so.

  render_rays(asset, origins, dirs, counters=None)   lightfield.py:400-456
  render_ray(asset, ray, counters=None)              lightfield.py:459-463
  march_rays(asset, origins, dirs)                   lightfield.py:129-186, 418-425
  render_range(asset, ray_range, counters=None)      renderer.py:63-93
  render_frame(scene, camera, counters=None)         renderer.py:96-107
  compose(frames, asset_order=None, alpha_vis=0.5)   farm.py:129-172
  SceneRenderer / render_scene                       fused march+shade+compose
                                                     over screen tiles (fast path)

Host arrays in, host arrays out for the reference signatures (the copies are
part of the call, as a drop-in must); ``SceneRenderer`` keeps everything on
the device.  Per-asset device state is uploaded once and cached by the
identity of the asset's arrays (plus a checksum of its MLP parameters, which
the reference's own tests mutate in place); ``invalidate()`` drops it.
"""

from __future__ import annotations

import ctypes as C
import threading
import time
import zlib
from collections import OrderedDict
from typing import NamedTuple

import numpy as np

from . import _native as N
from . import errors
from .model import ENC_DEFLATE, ENC_RAW, Frame, FrameData, RayRange, RenderCounters, Tile, uniform_scale_of

_torch = None

# Result types; shim.install() swaps in the reference's own Tile / Frame.
OWN_TYPES = {"Frame": Frame, "Tile": Tile, "FrameData": FrameData}
TYPES = dict(OWN_TYPES)


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def _device():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("CUDA device required: the i-NOLF path has no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def _stream_ptr():
    return torch().cuda.current_stream().cuda_stream


# ------------------------------------------------------------------ assets
MLP_MODES = {"fp32": N.MLP_FP32, "bf16": N.MLP_BF16}
_MLP_MODE = N.MLP_FP32


def set_mlp_mode(mode: str) -> None:
    """Specular-MLP arithmetic for subsequent renders: "fp32" (CUDA cores,
    tolerance 1e-3) or "bf16" (tcgen05 tensor cores, tolerance 2/255).
    Assets that need the live diffuse network always shade in fp32."""
    global _MLP_MODE
    if mode not in MLP_MODES:
        raise errors.ConfigError(f"unknown MLP mode {mode!r}; have {sorted(MLP_MODES)}")
    _MLP_MODE = MLP_MODES[mode]


def bf16_capable(asset) -> bool:
    m = asset.specular_mlp
    return (m is not None and len(m.weights) == 3 and m.weights[0].shape[1] <= 32
            and (asset.diffuse_atlas is not None or not asset.wiring.use_diffuse_color))


class DeviceAsset:
    """Owns one nolf_asset_t (device copy of every table of an asset)."""

    object_to_world = None        # set for natively loaded assets (load_device_asset)

    def __init__(self, asset, device_index: int, handle=None):
        if handle is None:
            desc, keep = N.asset_desc(asset)
            h = C.c_void_p()
            N.check(N.lib().nolf_asset_create(C.byref(desc), int(device_index), C.byref(h)))
            del keep
        else:
            h = handle
        self.handle = h
        self.device_index = device_index
        self.nbytes = int(N.lib().nolf_asset_device_bytes(h))
        self.mode = N.MLP_FP32
        if asset is not None:
            self.bf16_ok = bf16_capable(asset)
        else:                     # ask the library (it validates the tensor-core layout)
            self.bf16_ok = N.lib().nolf_asset_set_mlp_mode(h, N.MLP_BF16) == 0
            N.check(N.lib().nolf_asset_set_mlp_mode(h, N.MLP_FP32))

    def set_mlp_mode(self, mode: int) -> None:
        if mode != self.mode:
            N.check(N.lib().nolf_asset_set_mlp_mode(self.handle, int(mode)))
            self.mode = mode

    def __del__(self):
        h = getattr(self, "handle", None)
        lib = getattr(N, "_lib", None) if N is not None else None   # None at interpreter exit
        if h and lib is not None:
            lib.nolf_asset_destroy(h)
            self.handle = None


_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_MAX = 64


def _fingerprint(asset, device_index):
    if getattr(asset, "analytic_color", None) is not None or (
            asset.density_atlas is None and getattr(asset, "analytic_density", None) is not None):
        raise errors.DomainError(
            "analytic (closed-form) assets are a CPU test bypass and are not supported by the "
            "B200 render path; bake them into cube atlases first")
    if asset.density_atlas is None:
        raise errors.StateError("asset is not baked; no density cache to march")
    arrays = [asset.density_atlas.index, asset.density_atlas.cubes, asset.psh.offsets,
              asset.psh_features]
    if asset.diffuse_atlas is not None:
        arrays += [asset.diffuse_atlas.index, asset.diffuse_atlas.cubes]
    if asset.diffuse_features is not None:
        arrays += list(asset.diffuse_features)
    mesh = getattr(asset, "proxy_mesh", None)
    if mesh is not None:
        arrays += [mesh[0], mesh[1]]
    crc = 0
    for m in (asset.specular_mlp, asset.diffuse_mlp):
        if m is not None:
            for a in list(m.weights) + list(m.biases):
                crc = zlib.crc32(np.ascontiguousarray(a).view(np.uint8), crc)
    w = asset.wiring
    key = (device_index, tuple(id(a) for a in arrays), crc,
           (asset.march.step, asset.march.t_stop, asset.march.alpha_floor),
           tuple(np.asarray(asset.proxy.min, float)), tuple(np.asarray(asset.proxy.max, float)),
           (w.use_hit_point, w.use_opacity, w.use_tint, w.refine_opacity, w.use_diffuse_color),
           tuple(m.heads) if (m := asset.specular_mlp) is not None else None)
    return key, arrays


def load_device_asset(path_or_bytes, device_index: int | None = None) -> DeviceAsset:
    """assetio.read_asset + upload in one native call (nolf_asset_load): the
    ``.nolf`` file (gzip accepted) is parsed, CRC-checked and uploaded by the
    library.  The result can be placed in scenes like any asset; its stored
    transform is ``.object_to_world``."""
    if device_index is None:
        _device()
        device_index = torch().cuda.current_device()
    h = C.c_void_p()
    o2w = (C.c_double * 16)()
    if isinstance(path_or_bytes, (bytes, bytearray, memoryview)):
        buf = bytes(path_or_bytes)
        N.check(N.lib().nolf_asset_load_mem(buf, len(buf), int(device_index), C.byref(h), o2w))
    else:
        N.check(N.lib().nolf_asset_load(str(path_or_bytes).encode(), int(device_index), C.byref(h), o2w))
    dev = DeviceAsset(None, device_index, handle=h)
    dev.object_to_world = np.array(o2w[:], np.float64).reshape(4, 4)
    return dev


def device_asset(asset, device_index: int | None = None) -> DeviceAsset:
    """Upload (or fetch the cached upload of) an asset on a CUDA device."""
    if isinstance(asset, DeviceAsset):
        return asset
    if device_index is None:
        _device()
        device_index = torch().cuda.current_device()
    key, arrays = _fingerprint(asset, device_index)
    hit = _CACHE.get(key)
    if hit is not None:
        _CACHE.move_to_end(key)
        return hit[0]
    dev = DeviceAsset(asset, device_index)
    _CACHE[key] = (dev, arrays)       # arrays pinned so their ids stay unique
    while len(_CACHE) > _CACHE_MAX:
        _CACHE.popitem(last=False)
    return dev


def invalidate() -> None:
    """Forget every cached device asset (call after in-place array edits)."""
    _CACHE.clear()


# ------------------------------------------------------------------ workspace
_WS = {}


def workspace(nbytes: int):
    t = torch()
    dev = _device()
    cur = _WS.get(dev.index)
    if cur is None or cur.numel() < nbytes:
        _WS[dev.index] = None
        cur = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=dev)
        _WS[dev.index] = cur
    return cur


_XFORM = {}          # o2w bytes -> (w2o, scale): the per-call inverse / scale check, memoised


def _instance(asset, transform=None) -> N.Instance:
    o2w = np.asarray(asset.object_to_world if transform is None else transform, np.float64)
    key = o2w.tobytes()
    hit = _XFORM.get(key)
    if hit is None:
        w2o = np.linalg.inv(o2w)                  # lightfield.py:408
        scale = uniform_scale_of(w2o)             # lightfield.py:409 (raises for non-uniform scales)
        if len(_XFORM) > 4096:
            _XFORM.clear()
        hit = _XFORM[key] = (w2o, scale)
    w2o, scale = hit
    dev = device_asset(asset)
    dev.set_mlp_mode(_MLP_MODE if dev.bf16_ok else N.MLP_FP32)
    inst = N.Instance()
    inst.asset = dev.handle
    flat = w2o.reshape(16)
    for i in range(16):
        inst.w2o[i] = float(flat[i])
    inst.scale = float(scale)
    inst._dev = dev                               # keep the handle alive
    return inst


def check_device_errors(stream=None) -> None:
    """Synchronise and raise CapacityError if any launch on this thread had
    to drop work on the device (nolf_check_errors)."""
    N.check(N.lib().nolf_check_errors(stream if stream is not None else _stream_ptr()))


def _merge(counters, cnt_dev):
    if counters is None:
        return
    c = cnt_dev.cpu().numpy()
    counters.fs_evals += int(c[0])
    counters.fd_evals += int(c[1])
    counters.hit_pixels += int(c[2])
    counters.march_samples += int(c[3])


# ------------------------------------------------------------------ test / debug hooks
def set_option(key: int, value: int) -> None:
    """Force a launch variant (nolf_set_option; _native.OPT_*) on this thread."""
    N.check(N.lib().nolf_set_option(int(key), int(value)))


def last_launch() -> dict:
    """Variants of this thread's last render launch (nolf_last_launch)."""
    info = (C.c_int32 * 4)()
    N.check(N.lib().nolf_last_launch(info))
    return {"chunked": bool(info[0]), "march_order": "heavy-first" if info[1] else "spatial",
            "compose_slots": int(info[2]), "shade": "k_shade_tc (bf16)" if info[3] else "k_shade (fp32)",
            "shade_ctas_per_sm": int(info[3])}


class debug_psh_slots:
    """While active, the shading kernels of this thread's render calls store
    the 8 PSH corner slots each hit gathered (nolf_debug_psh_slots):
    ``.slots()`` -> (rows, 8) int64 host array, -1 where no hit was shaded.
    Row = output row (render_rays / render_range) or layer * P + slot
    (render_scene)."""

    def __init__(self, rows: int):
        t = torch()
        self.buf = t.full((max(int(rows), 1), 8), -1, dtype=t.int32, device=_device())

    def __enter__(self):
        N.check(N.lib().nolf_debug_psh_slots(self.buf.data_ptr(), len(self.buf)))
        return self

    def __exit__(self, *exc):
        N.check(N.lib().nolf_debug_psh_slots(None, 0))

    def slots(self):
        torch().cuda.synchronize()
        return self.buf.cpu().numpy().astype(np.int64)


# ------------------------------------------------------------------ reference API
def mlp_eval(asset, x, mode: str = "fp32"):
    """The specular network alone on rows x (n, in) -> (n, 4) post-head
    (nolf_mlp_eval; used by the numerics tests)."""
    t = torch()
    dev = _device()
    xa = t.as_tensor(np.ascontiguousarray(x, np.float32)).to(dev)
    out = t.empty((len(xa), 4), dtype=t.float32, device=dev)
    N.check(N.lib().nolf_mlp_eval(device_asset(asset).handle, MLP_MODES[mode], xa.data_ptr(), len(xa),
                                  out.data_ptr(), _stream_ptr()))
    return out.cpu().numpy()


def render_rays(asset, origins, dirs, counters=None):
    """World-space rays -> (rgba (B,4) f32, depth (B,) f32); lightfield.py:400-456."""
    t = torch()
    origins = np.asarray(origins, dtype=np.float64)
    dirs = np.asarray(dirs, dtype=np.float64)
    if origins.ndim != 2 or origins.shape[1] != 3 or dirs.shape != origins.shape:
        raise errors.DomainError("origins and dirs must both be (B,3)")
    n = len(origins)
    inst = _instance(asset)
    dev = _device()
    shared = n > 0 and origins.strides[0] == 0
    o_host = np.ascontiguousarray(origins[:1] if shared else origins)
    o = t.from_numpy(o_host).to(dev)
    d = t.from_numpy(np.ascontiguousarray(dirs)).to(dev)
    rgba = t.empty((n, 4), dtype=t.float32, device=dev)
    depth = t.empty((n,), dtype=t.float32, device=dev)
    cnt = t.zeros(4, dtype=t.int64, device=dev)
    need = int(N.lib().nolf_workspace_bytes(1, n))
    ws = workspace(need)
    N.check(N.lib().nolf_render_rays(C.byref(inst), o.data_ptr(), 0 if shared else 1, d.data_ptr(), n,
                                     rgba.data_ptr(), depth.data_ptr(), cnt.data_ptr(), ws.data_ptr(),
                                     ws.numel(), _stream_ptr()))
    # one pinned staging block [counters | rgba | depth]: async copies, one sync
    host = _staging(32 + n * 20)
    h_cnt = host[:32].view(t.int64)
    h_rgba = host[32:32 + n * 16].view(t.float32).view(n, 4)
    h_depth = host[32 + n * 16:32 + n * 20].view(t.float32)
    h_cnt.copy_(cnt, non_blocking=True)
    h_rgba.copy_(rgba, non_blocking=True)
    h_depth.copy_(depth, non_blocking=True)
    check_device_errors()                 # synchronises the stream: the copies have landed
    out = h_rgba.numpy().copy(), h_depth.numpy().copy()
    if counters is not None:
        c = h_cnt.numpy()
        counters.fs_evals += int(c[0])
        counters.fd_evals += int(c[1])
        counters.hit_pixels += int(c[2])
        counters.march_samples += int(c[3])
    return out


class MarchResult(NamedTuple):
    """lightfield.MarchResult (lightfield.py:101-110) minus the transmittance."""
    hit: np.ndarray          # (B,) bool
    t_hit: np.ndarray        # (B,) f64, inf on a miss
    alpha_c: np.ndarray      # (B,) f64
    samples: np.ndarray      # (B,) i64 active samples
    p_h: np.ndarray          # (B,3) f64 clip(o + t_hit d, 0, 1), 0 on a miss


def march_rays(asset, origins, dirs) -> MarchResult:
    """The march alone, as render_rays runs it (lightfield.py:418-425): OBJECT-
    space rays, t_near / t_far from the asset's proxy box, then march_rays
    (lightfield.py:129-186) on the CUDA marcher (nolf_march_rays)."""
    t = torch()
    origins = np.asarray(origins, dtype=np.float64)
    dirs = np.asarray(dirs, dtype=np.float64)
    if origins.ndim != 2 or origins.shape[1] != 3 or dirs.shape != origins.shape:
        raise errors.DomainError("origins and dirs must both be (B,3)")
    n = len(origins)
    dev = _device()
    o = t.from_numpy(np.ascontiguousarray(origins)).to(dev)
    d = t.from_numpy(np.ascontiguousarray(dirs)).to(dev)
    hit = t.zeros(n, dtype=t.uint8, device=dev)
    t_hit = t.empty(n, dtype=t.float64, device=dev)
    alpha = t.empty(n, dtype=t.float64, device=dev)
    samples = t.empty(n, dtype=t.int64, device=dev)
    p_h = t.empty((n, 3), dtype=t.float64, device=dev)
    if n:
        N.check(N.lib().nolf_march_rays(device_asset(asset).handle, o.data_ptr(), 1, d.data_ptr(), n,
                                        hit.data_ptr(), t_hit.data_ptr(), alpha.data_ptr(), samples.data_ptr(),
                                        p_h.data_ptr(), None, 0, _stream_ptr()))
    # one pinned staging block [t_hit | alpha | samples | p_h | hit]: async copies, one sync
    host = _staging(n * (8 + 8 + 8 + 24 + 1) + 64)
    views = []
    off = 0
    for src, dt, shape in ((t_hit, t.float64, (n,)), (alpha, t.float64, (n,)), (samples, t.int64, (n,)),
                           (p_h, t.float64, (n, 3)), (hit, t.uint8, (n,))):
        nb = src.numel() * src.element_size()
        v = host[off:off + nb].view(dt).view(*shape)
        v.copy_(src, non_blocking=True)
        views.append(v)
        off += nb
    check_device_errors()                 # synchronises the stream: the copies have landed
    h_t, h_a, h_s, h_p, h_h = (v.numpy().copy() for v in views)
    return MarchResult(h_h.astype(bool), h_t, h_a, h_s, h_p)


def render_ray(asset, ray, counters=None):
    rgba, depth = render_rays(asset, np.asarray(ray.origin)[None, :],
                              np.asarray(ray.direction)[None, :], counters)
    return rgba[0], float(depth[0])


_RANGE_BUFS = {}
_STAGING = {}


def _staging(nbytes: int):
    """A pinned host block of at least nbytes for this thread (grown, reused)."""
    t = torch()
    key = threading.get_ident()
    cur = _STAGING.get(key)
    if cur is None or cur.numel() < nbytes:
        cur = t.empty(max(int(nbytes), 1 << 16) * 2, dtype=t.uint8, pin_memory=True)
        _STAGING[key] = cur
    return cur


def render_range(asset, ray_range, counters=None):
    """Render a RayRange rectangle -> (Tile, instr); renderer.py:63-93."""
    t = torch()
    counters = counters if counters is not None else RenderCounters()
    start = time.perf_counter()
    inst = _instance(asset)
    cam = ray_range.camera
    x0, y0, x1, y1 = ray_range.x0, ray_range.y0, ray_range.x1, ray_range.y1
    h, w = y1 - y0, x1 - x0
    dev = _device()
    # per-shape device outputs and one pinned host staging block, reused by
    # every call of this shape (a farm worker's light tiles are all 32x32):
    # one launch, three async copies and one synchronisation per call
    key = (threading.get_ident(), dev.index, h, w)
    bufs = _RANGE_BUFS.get(key)
    if bufs is None:
        host = t.empty(32 + h * w * 5 * 4, dtype=t.uint8, pin_memory=True)   # [counters | rgba | depth]
        bufs = (t.empty((h, w, 4), dtype=t.float32, device=dev), t.empty((h, w), dtype=t.float32, device=dev),
                t.zeros(4, dtype=t.int64, device=dev), host,
                host[32:32 + h * w * 16].view(t.float32).view(h, w, 4),
                host[32 + h * w * 16:].view(t.float32).view(h, w), host[:32].view(t.int64))
        _RANGE_BUFS[key] = bufs
    rgba, depth, cnt, _, h_rgba, h_depth, h_cnt = bufs
    cnt.zero_()
    ws = workspace(int(N.lib().nolf_workspace_bytes(1, h * w)))
    cs = N.camera_struct(cam)
    N.check(N.lib().nolf_render_rect(C.byref(inst), C.byref(cs), x0, y0, x1, y1, rgba.data_ptr(),
                                     depth.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws.numel(),
                                     _stream_ptr()))
    h_rgba.copy_(rgba, non_blocking=True)
    h_depth.copy_(depth, non_blocking=True)
    h_cnt.copy_(cnt, non_blocking=True)
    check_device_errors()                 # synchronises the stream: the copies have landed
    tile = TYPES["Tile"](x0=x0, y0=y0, rgba=h_rgba.numpy().copy(), depth=h_depth.numpy().copy())
    c = h_cnt.numpy()
    before_fs, before_hits = counters.fs_evals, counters.hit_pixels
    counters.fs_evals += int(c[0])
    counters.fd_evals += int(c[1])
    counters.hit_pixels += int(c[2])
    counters.march_samples += int(c[3])
    instr = {"wall_time_s": time.perf_counter() - start, "rays": int(h * w),
             "hits": counters.hit_pixels - before_hits, "fs_evals": counters.fs_evals - before_fs}
    del c
    return tile, instr


class _Rect:
    """Full-frame RayRange without re-validating (bounds are the frame's)."""

    def __init__(self, camera, x0, y0, x1, y1):
        self.camera, self.x0, self.y0, self.x1, self.y1 = camera, x0, y0, x1, y1


def render_frame(scene, camera, counters=None):
    """Per-asset full frames for depth composition; renderer.py:96-107."""
    frames = []
    for asset, transform in scene:
        placed = asset
        if transform is not None:
            import dataclasses
            placed = dataclasses.replace(asset, object_to_world=np.asarray(transform, np.float64))
        tile, _ = render_range(placed, _Rect(camera, 0, 0, camera.width, camera.height), counters)
        frames.append(TYPES["Frame"](width=camera.width, height=camera.height, rgba=tile.rgba,
                                     depth=tile.depth))
    return frames


def compose(frames, asset_order=None, alpha_vis: float = 0.5):
    """Depth-sorted front-to-back over of per-asset frames; farm.py:129-172."""
    if not frames:
        raise errors.ProtocolError("compose needs at least one frame")
    t = torch()
    h, w = frames[0].height, frames[0].width
    dev = _device()
    rgba = t.from_numpy(np.ascontiguousarray(np.stack([f.rgba for f in frames]), np.float32)).to(dev)
    depth = t.from_numpy(np.ascontiguousarray(np.stack([f.depth for f in frames]), np.float32)).to(dev)
    orgba, odepth = compose_device(rgba.reshape(len(frames), h * w, 4), depth.reshape(len(frames), h * w),
                                   alpha_vis)
    return TYPES["Frame"](width=w, height=h, rgba=orgba.reshape(h, w, 4).cpu().numpy(),
                          depth=odepth.reshape(h, w).cpu().numpy())


def compose_device(rgba, depth, alpha_vis: float = 0.5):
    """compose on device tensors: rgba (K,P,4) f32, depth (K,P) f32."""
    t = torch()
    K, P = depth.shape
    out_rgba = t.empty((P, 4), dtype=t.float32, device=rgba.device)
    out_depth = t.empty((P,), dtype=t.float32, device=rgba.device)
    N.check(N.lib().nolf_compose(K, P, rgba.contiguous().data_ptr(), depth.contiguous().data_ptr(),
                                 float(alpha_vis), out_rgba.data_ptr(), out_depth.data_ptr(),
                                 _stream_ptr()))
    return out_rgba, out_depth


def encode_frame(frame, encoding: int = ENC_RAW, depth_far: float = 10.0):
    """protocol.encode_frame (protocol.py:256-279): rgba8 + u16 depth
    quantised on the GPU (nolf_encode_frame, the compose epilogue's
    arithmetic), ENC_DEFLATE streams by zlib level 6 in the library
    (nolf_deflate) -> the reference's FrameData."""
    if encoding not in (ENC_RAW, ENC_DEFLATE):
        raise errors.ProtocolError(f"unknown frame encoding {encoding}")
    t = torch()
    dev = _device()
    h, w = frame.height, frame.width
    rgba = t.from_numpy(np.ascontiguousarray(frame.rgba, np.float32).reshape(-1, 4)).to(dev)
    depth = t.from_numpy(np.ascontiguousarray(frame.depth, np.float32).reshape(-1)).to(dev)
    r8 = t.empty((h * w, 4), dtype=t.uint8, device=dev)
    d16 = t.empty((h * w,), dtype=t.int16, device=dev)
    N.check(N.lib().nolf_encode_frame(rgba.data_ptr(), depth.data_ptr(), h * w, float(depth_far), r8.data_ptr(),
                                      d16.data_ptr(), _stream_ptr()))
    rgba_b = r8.cpu().numpy().tobytes()
    depth_b = d16.cpu().numpy().view("<u2").tobytes()
    if encoding == ENC_DEFLATE:
        rgba_b, depth_b = deflate(rgba_b), deflate(depth_b)
    return TYPES["FrameData"](pose_seq=0, frame_index=0, encoding=encoding, width=w, height=h,
                              depth_far=depth_far, rgba=rgba_b, depth=depth_b)


def deflate(data: bytes, level: int = 6) -> bytes:
    """zlib.compress(data, level) by the library's zlib (nolf_deflate)."""
    lib = N.lib()
    cap = C.c_size_t(0)
    N.check(lib.nolf_deflate(data, len(data), level, None, C.byref(cap)))
    buf = C.create_string_buffer(cap.value)
    N.check(lib.nolf_deflate(data, len(data), level, buf, C.byref(cap)))
    return buf.raw[:cap.value]


# ------------------------------------------------------------------ fast path
def frame_tiles(width: int, height: int, tile: int = 32, cam: int = 0) -> np.ndarray:
    """tile_ranges (renderer.py:176-187) as an (n,5) int32 [cam,x0,y0,x1,y1] table."""
    out = [(cam, tx, ty, min(tx + tile, width), min(ty + tile, height))
           for ty in range(0, height, tile) for tx in range(0, width, tile)]
    return np.asarray(out, dtype=np.int32).reshape(-1, 5)


class SceneRenderer:
    """Fused multi-asset renderer: march + shade + depth compose of every
    placed asset over a tile list, all resident on one device.

    ``scene`` is a list of (asset, transform) like render_frame's; each tile
    row is (camera index, x0, y0, x1, y1); pixels come back tile-packed with
    ``tile_stride`` slots per tile.
    """

    def __init__(self, scene, alpha_vis: float = 0.5, depth_far: float = 10.0):
        self.insts = [_instance(a, tr) for a, tr in scene]
        arr = (N.Instance * len(self.insts))()
        for i, inst in enumerate(self.insts):
            C.memmove(C.byref(arr[i]), C.byref(inst), C.sizeof(N.Instance))
        self._inst_arr = arr
        self.alpha_vis = float(alpha_vis)
        self.depth_far = float(depth_far)
        self.device = _device()
        self._ws = None

    def mlp_mode(self, mode: int) -> None:
        for inst in self.insts:
            inst._dev.set_mlp_mode(mode if inst._dev.bf16_ok else N.MLP_FP32)

    def alloc(self, n_tiles: int, tile_stride: int, want_f32=True, want_u8=True):
        t = torch()
        P = n_tiles * tile_stride
        out = {}
        if want_f32:
            out["rgba"] = t.empty((P, 4), dtype=t.float32, device=self.device)
            out["depth"] = t.empty((P,), dtype=t.float32, device=self.device)
        if want_u8:
            out["rgba8"] = t.empty((P, 4), dtype=t.uint8, device=self.device)
            out["depth16"] = t.empty((P,), dtype=t.int16, device=self.device)
        out["counters"] = t.zeros(4, dtype=t.int64, device=self.device)
        return out

    def _need(self, cams, P: int) -> int:
        cams = cams if isinstance(cams, C.Array) else self.camera_array(cams)
        need = int(N.lib().nolf_scene_workspace_bytes(self._inst_arr, len(self.insts), cams,
                                                      len(cams), int(P)))
        if need == 0:
            raise errors.DomainError("bad scene for workspace sizing")
        return need

    def reserve(self, camera_sets, P: int) -> int:
        """Size the workspace once for every camera set a run will render
        (growing it mid-run would put a cudaMalloc in the frame loop)."""
        need = max(self._need(c, P) for c in camera_sets)
        self._grow(need)
        return need

    def _grow(self, need: int):
        t = torch()
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            # 25 % headroom: screen boxes (hence queue sizes) move with the camera
            self._ws = t.empty(int(need * 1.25) + (1 << 20), dtype=t.uint8, device=self.device)

    def _workspace(self, cams, P: int):
        """Tight per-launch workspace (hit queues sized by the instances'
        screen boxes, compose layers by their maximum overlap)."""
        self._grow(self._need(cams, P))
        return self._ws

    @staticmethod
    def camera_array(cameras):
        cams = (N.Camera * len(cameras))()
        for i, c in enumerate(cameras):
            cams[i] = N.camera_struct(c)
        return cams

    def render(self, cameras, tiles_dev, n_tiles: int, tile_stride: int, out: dict, stream=None,
               frame_layout: bool = False, peer: bool = False, prefilled: bool = False):
        """One fused launch sequence.  ``out``: rgba / depth (f32), rgba8 /
        depth16 (encode_frame RAW), counters; optionally pack / pack_ids /
        pack_count (the sparse frame of live chunks, NolfSceneOut.pack;
        needs prefilled=True); chunk_state (a u16 of run dirty bits per 128-slot chunk per
        frame buffer: stale chunks are reset instead of re-clearing the
        frame, NolfSceneOut.chunk_state)."""
        cams = cameras if isinstance(cameras, C.Array) else self.camera_array(cameras)
        so = N.SceneOut()
        def ptr(key):              # tensors, or raw device addresses (peer mappings)
            v = out.get(key)
            return None if v is None else (v if isinstance(v, int) else v.data_ptr())

        so.rgba = ptr("rgba")
        so.depth = ptr("depth")
        so.rgba8 = ptr("rgba8")
        so.depth16 = ptr("depth16")
        so.tile_stride = int(tile_stride)
        so.depth_far = self.depth_far
        so.layout = 1 if frame_layout else 0
        so.peer = 1 if peer else 0
        so.prefilled = 1 if prefilled else 0
        so.pack = ptr("pack")
        so.pack_ids = ptr("pack_ids")
        so.pack_count = ptr("pack_count")
        so.chunk_state = ptr("chunk_state")
        st = stream if stream is not None else _stream_ptr()
        P = int(n_tiles) * int(tile_stride)
        # the library sizes the launch itself and refuses a short workspace:
        # only then is the plan computed here too (grow, retry)
        ws = self._ws if self._ws is not None else self._workspace(cams, P)
        lib = N.lib()

        def launch(ws):
            return lib.nolf_render_scene(self._inst_arr, len(self.insts), cams, len(cams), tiles_dev.data_ptr(),
                                         int(n_tiles), C.byref(so), self.alpha_vis, out["counters"].data_ptr(),
                                         ws.data_ptr(), ws.numel(), st)
        rc = launch(ws)
        if rc == N.NOLF_EINVAL and b"workspace too small" in lib.nolf_last_error():
            rc = launch(self._workspace(cams, P))
        N.check(rc)

    def check(self, stream=None) -> None:
        """Synchronise; CapacityError if a render dropped work on the device
        (invalid tiles, ...).  Renders also fail on the call after one that
        dropped work, once its asynchronous error read-back has landed."""
        check_device_errors(stream)


def slot_xy(local, w: int, h: int):
    """(x, y) inside a w x h tile of packed slot ``local`` (nolf_kernels.cuh:slot_xy)."""
    local = np.asarray(local, np.int64)
    if w % 8 == 0 and h % 4 == 0:
        blk, lane = local // 32, local % 32
        return (blk % (w // 8)) * 8 + lane % 8, (blk // (w // 8)) * 4 + lane // 8
    return local % w, local // w


def unpack_index(tiles: np.ndarray, tile_stride: int, width: int, height: int, cam: int = 0):
    """Packed-slot index of every pixel of camera ``cam`` (row-major H*W), -1 if absent.

    Inside a tile whose sides are multiples of 8 x 4 the slots run over 8x4
    pixel blocks (block-row-major, row-major inside a block: one warp per
    block); other tiles are row-major (nolf_kernels.cuh:slot_xy)."""
    idx = np.full(height * width, -1, dtype=np.int64)
    for t, (c, x0, y0, x1, y1) in enumerate(tiles):
        if c != cam:
            continue
        w, h = x1 - x0, y1 - y0
        ys, xs = np.mgrid[0:h, 0:w]
        if w % 8 == 0 and h % 4 == 0:
            local = ((ys // 4) * (w // 8) + xs // 8) * 32 + (ys % 4) * 8 + xs % 8
        else:
            local = ys * w + xs
        idx[((ys + y0) * width + xs + x0).reshape(-1)] = t * tile_stride + local.reshape(-1)
    return idx


def render_scene(scene, camera, counters=None, tile: int = 32):
    """Composed Frame of a scene in one fused launch sequence (== compose(render_frame(...)))."""
    t = torch()
    r = SceneRenderer(scene)
    tiles = frame_tiles(camera.width, camera.height, tile)
    tiles_dev = t.from_numpy(tiles).to(r.device)
    out = r.alloc(len(tiles), tile * tile, want_f32=True, want_u8=False)
    r.render([camera], tiles_dev, len(tiles), tile * tile, out, frame_layout=True)
    npx = camera.width * camera.height
    rgba = out["rgba"][:npx].reshape(camera.height, camera.width, 4)
    depth = out["depth"][:npx].reshape(camera.height, camera.width)
    check_device_errors()
    _merge(counters, out["counters"])
    return Frame(width=camera.width, height=camera.height, rgba=rgba.cpu().numpy(),
                 depth=depth.cpu().numpy())
