"""ctypes binding of the C ABI in include/nolf.h (libnolf_b200.so).

The library is built in-tree by ``paper_2303_04086_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or fails to load,
every render entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors

LIB_NAME = "libnolf_b200.so"
LIB_PATH = os.environ.get("NOLF_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     LIB_NAME)

NOLF_EINVAL, NOLF_ESTATE, NOLF_EDATA, NOLF_ECUDA, NOLF_ENOMEM, NOLF_ECAPACITY = -1, -2, -3, -4, -5, -6
HEAD_ACT = {"identity": 0, "sigmoid": 1, "exponential": 2}
ABI_VERSION = 4              # NOLF_ABI_VERSION of include/nolf.h
# nolf_set_option keys (include/nolf.h)
OPT_MARCH_ORDER, OPT_COMPOSE_SLOTS, OPT_HEAVY_WAVES, OPT_MARCH_SPLIT, OPT_CHUNK_COST = 1, 2, 3, 4, 5
MLP_FP32, MLP_BF16 = 0, 1


class AtlasDesc(C.Structure):
    _fields_ = [("b", C.c_int32), ("r", C.c_int32), ("channels", C.c_int32),
                ("n_cubes", C.c_int64), ("index", C.c_void_p), ("cubes", C.c_void_p)]


class MlpDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("widths", C.c_int32 * 5), ("w", C.c_void_p * 4),
                ("b", C.c_void_p * 4), ("n_heads", C.c_int32), ("head_act", C.c_int32 * 8),
                ("head_w", C.c_int32 * 8)]


class AssetDesc(C.Structure):
    _fields_ = [
        ("density", AtlasDesc), ("has_diffuse_atlas", C.c_int32), ("diffuse", AtlasDesc),
        ("psh_resolution", C.c_int32), ("psh_table_size", C.c_int64),
        ("psh_offset_size", C.c_int64), ("psh_offsets", C.c_void_p),
        ("primes_h0", C.c_uint64 * 3), ("primes_h1", C.c_uint64 * 3),
        ("psh_features", C.c_void_p), ("psh_features_dim", C.c_int32),
        ("hg_levels", C.c_int32), ("hg_features", C.c_int32), ("hg_table_size", C.c_int64),
        ("hg_resolution", C.c_int32 * 16), ("hg_dense", C.c_int32 * 16),
        ("hg_rows", C.c_int64 * 16), ("hg_feat", C.c_void_p * 16),
        ("specular", MlpDesc), ("diffuse_mlp", MlpDesc),
        ("step", C.c_double), ("t_stop", C.c_double), ("alpha_floor", C.c_double),
        ("proxy_min", C.c_double * 3), ("proxy_max", C.c_double * 3),
        ("use_hit_point", C.c_int32), ("use_opacity", C.c_int32), ("refine_opacity", C.c_int32),
        ("use_tint", C.c_int32), ("use_diffuse_color", C.c_int32),
        ("mesh_vertices", C.c_void_p), ("mesh_n_vertices", C.c_int64),
        ("mesh_triangles", C.c_void_p), ("mesh_n_triangles", C.c_int64),
    ]


class Instance(C.Structure):
    _fields_ = [("asset", C.c_void_p), ("w2o", C.c_double * 16), ("scale", C.c_double)]


class Camera(C.Structure):
    _fields_ = [("pose", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32)]


class SceneOut(C.Structure):
    _fields_ = [("rgba", C.c_void_p), ("depth", C.c_void_p), ("rgba8", C.c_void_p),
                ("depth16", C.c_void_p), ("tile_stride", C.c_int64), ("depth_far", C.c_double),
                ("layout", C.c_int32), ("peer", C.c_int32), ("prefilled", C.c_int32),
                ("pack", C.c_void_p), ("pack_ids", C.c_void_p), ("pack_count", C.c_void_p),
                ("chunk_state", C.c_void_p)]


_lib = None


def lib():
    """Load libnolf_b200.so (raises if absent: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_NAME} is not built ({LIB_PATH}); run "
                           "`python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "nolf_abi_version": ([], C.c_int),
        "nolf_last_error": ([], C.c_char_p),
        "nolf_asset_create": ([C.POINTER(AssetDesc), C.c_int, C.POINTER(vp)], C.c_int),
        "nolf_asset_load": ([C.c_char_p, C.c_int, C.POINTER(vp), C.POINTER(C.c_double)], C.c_int),
        "nolf_asset_load_mem": ([C.c_char_p, C.c_size_t, C.c_int, C.POINTER(vp), C.POINTER(C.c_double)], C.c_int),
        "nolf_asset_destroy": ([vp], C.c_int),
        "nolf_asset_set_mlp_mode": ([vp, C.c_int], C.c_int),
        "nolf_asset_device_bytes": ([vp], i64),
        "nolf_workspace_bytes": ([i32, i64], C.c_size_t),
        "nolf_scene_workspace_bytes": ([C.POINTER(Instance), i32, C.POINTER(Camera), i32, i64], C.c_size_t),
        "nolf_render_rays": ([C.POINTER(Instance), vp, i32, vp, i64, vp, vp, vp, vp, C.c_size_t, vp],
                             C.c_int),
        "nolf_render_rect": ([C.POINTER(Instance), C.POINTER(Camera), i32, i32, i32, i32, vp, vp, vp,
                              vp, C.c_size_t, vp], C.c_int),
        "nolf_render_scene": ([C.POINTER(Instance), i32, C.POINTER(Camera), i32, vp, i32,
                               C.POINTER(SceneOut), dbl, vp, vp, C.c_size_t, vp], C.c_int),
        "nolf_compose": ([i32, i64, vp, vp, dbl, vp, vp, vp], C.c_int),
        "nolf_march_rays": ([vp, vp, i32, vp, i64, vp, vp, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "nolf_eval_diffuse": ([vp, vp, i64, vp, vp], C.c_int),
        "nolf_profile": ([C.c_int], C.c_int),
        "nolf_debug_psh_slots": ([vp, i64], C.c_int),
        "nolf_set_option": ([i32, i64], C.c_int),
        "nolf_last_launch": ([vp], C.c_int),
        "nolf_check_errors": ([vp], C.c_int),
        "nolf_encode_frame": ([vp, vp, i64, dbl, vp, vp, vp], C.c_int),
        "nolf_deflate": ([vp, C.c_size_t, i32, vp, C.POINTER(C.c_size_t)], C.c_int),
        "nolf_zlib_version": ([], C.c_char_p),
        "nolf_train_shade": ([vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, dbl, vp, vp, vp, vp], C.c_int),
        "nolf_adam": ([vp, vp, vp, vp, i64, dbl, dbl, dbl, dbl, i64, vp, vp], C.c_int),
        "nolf_host_scatter": ([vp, vp, C.c_uint32, vp, i32, i64, i32, i32, vp, vp, vp, i32], C.c_int),
        "nolf_mlp_eval": ([vp, C.c_int, vp, i64, vp, vp], C.c_int),
        "nolf_device_alloc": ([C.c_size_t, C.POINTER(vp)], C.c_int),
        "nolf_device_free": ([vp], C.c_int),
        "nolf_ipc_get_handle": ([vp, vp], C.c_int),
        "nolf_ipc_open_handle": ([vp, C.POINTER(vp)], C.c_int),
        "nolf_ipc_close_handle": ([vp], C.c_int),
        "nolf_flag_set": ([vp, C.c_uint32, vp], C.c_int),
        "nolf_memset_async": ([vp, C.c_int32, C.c_size_t, vp], C.c_int),
        "nolf_flag_wait": ([vp, C.c_int32, C.c_uint32, vp, vp], C.c_int),
        "nolf_memcpy_async": ([vp, vp, C.c_size_t, vp], C.c_int),
        "nolf_store_u32": ([vp, vp, i32, vp], C.c_int),
        "nolf_memcpy2d_async": ([vp, C.c_size_t, vp, C.c_size_t, C.c_size_t, C.c_size_t, vp], C.c_int),
        "nolf_host_register": ([vp, C.c_size_t, C.POINTER(vp)], C.c_int),
        "nolf_host_unregister": ([vp], C.c_int),
        "nolf_profile_read": ([C.POINTER(C.c_float)], C.c_int),
        "nolf_launch_param_bytes": ([i32, i32], C.c_size_t),
        "nolf_unpack_gathered": ([vp, i32, i32, i64, vp, i32, i32, vp, vp, vp], C.c_int),
    }
    experiment = bool(os.environ.get("NOLF_LIB"))   # another build (A/B): may predate some entry points
    for name, (args, res) in sig.items():
        if experiment and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.nolf_abi_version() != ABI_VERSION:
        raise RuntimeError("libnolf_b200.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().nolf_last_error().decode(errors="replace")
    if rc == NOLF_EINVAL:
        raise errors.DomainError(msg)
    if rc == NOLF_ESTATE:
        raise errors.StateError(msg)
    if rc == NOLF_EDATA:
        raise errors.DataError(msg)
    if rc == NOLF_ECAPACITY:
        raise errors.CapacityError(msg)
    raise RuntimeError(f"nolf error {rc}: {msg}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def asset_desc(asset):
    """Fill an AssetDesc from any attribute-compatible asset.  Returns
    (desc, keepalive) -- the numpy arrays must outlive nolf_asset_create."""
    keep = []

    def arr(a, dtype):
        x = np.ascontiguousarray(np.asarray(a), dtype=dtype)
        keep.append(x)
        return x

    d = AssetDesc()

    def fill_atlas(dst, at, ch):
        idx = arr(at.index, np.int32)
        cubes = arr(at.cubes, np.float32)
        dst.b, dst.r, dst.channels = int(at.base_resolution), int(at.cube_resolution), ch
        dst.n_cubes = int(cubes.shape[0])
        dst.index = _ptr(idx)
        dst.cubes = _ptr(cubes) if cubes.size else None

    if asset.density_atlas is None:
        raise errors.StateError("asset is not baked; no density cache to march")
    fill_atlas(d.density, asset.density_atlas, 1)
    if asset.diffuse_atlas is not None:
        d.has_diffuse_atlas = 1
        fill_atlas(d.diffuse, asset.diffuse_atlas, 4)
    psh = asset.psh
    offs = arr(psh.offsets, np.int64)
    feats = arr(asset.psh_features, np.float32)
    d.psh_resolution = int(psh.resolution)
    d.psh_table_size = int(psh.table_size)
    d.psh_offset_size = int(psh.offset_size)
    d.psh_offsets = _ptr(offs)
    for k in range(3):
        d.primes_h0[k] = int(np.asarray(psh.primes_h0, np.uint64)[k])
        d.primes_h1[k] = int(np.asarray(psh.primes_h1, np.uint64)[k])
    d.psh_features = _ptr(feats)
    d.psh_features_dim = int(feats.shape[1])
    enc = asset.diffuse_encoder
    if enc is not None and asset.diffuse_features is not None:
        d.hg_levels = int(enc.levels)
        d.hg_features = int(enc.features_per_level)
        d.hg_table_size = int(enc.table_size)
        for l in range(enc.levels):
            f = arr(asset.diffuse_features[l], np.float32)
            d.hg_resolution[l] = int(enc.resolutions[l])
            d.hg_dense[l] = int(bool(enc.dense[l]))
            d.hg_rows[l] = int(f.shape[0])
            d.hg_feat[l] = _ptr(f)

    def fill_mlp(dst, m):
        if m is None:
            dst.n_layers = 0
            return
        dst.n_layers = len(m.weights)
        dst.widths[0] = int(m.weights[0].shape[1])
        for i, (w, b) in enumerate(zip(m.weights, m.biases)):
            w = arr(w, np.float32)
            b = arr(b, np.float32)
            dst.widths[i + 1] = int(w.shape[0])
            dst.w[i] = _ptr(w)
            dst.b[i] = _ptr(b)
        dst.n_heads = len(m.heads)
        for i, (act, width) in enumerate(m.heads):
            dst.head_act[i] = HEAD_ACT[act]
            dst.head_w[i] = int(width)

    fill_mlp(d.specular, asset.specular_mlp)
    fill_mlp(d.diffuse_mlp, asset.diffuse_mlp)
    d.step = float(asset.march.step)
    d.t_stop = float(asset.march.t_stop)
    d.alpha_floor = float(asset.march.alpha_floor)
    for k in range(3):
        d.proxy_min[k] = float(asset.proxy.min[k])
        d.proxy_max[k] = float(asset.proxy.max[k])
    mesh = getattr(asset, "proxy_mesh", None)
    if mesh is not None:
        mv = arr(mesh[0], np.float64).reshape(-1, 3)
        mt = arr(mesh[1], np.int32).reshape(-1, 3)
        d.mesh_vertices, d.mesh_n_vertices = _ptr(mv), len(mv)
        d.mesh_triangles, d.mesh_n_triangles = _ptr(mt), len(mt)
    w = asset.wiring
    d.use_hit_point = int(bool(w.use_hit_point))
    d.use_opacity = int(bool(w.use_opacity))
    d.refine_opacity = int(bool(w.refine_opacity))
    d.use_tint = int(bool(w.use_tint))
    d.use_diffuse_color = int(bool(w.use_diffuse_color))
    return d, keep


def camera_struct(cam) -> Camera:
    c = Camera()
    pose = np.asarray(cam.pose, np.float64).reshape(16)
    for i in range(16):
        c.pose[i] = float(pose[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c
