"""ctypes wrapper of the C oracle (oracle/nolf_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the package.

The oracle is a CPU restatement of the reference render path (see the file
header of nolf_oracle.c for the per-function reference lines).  It is pinned
against the reference's own outputs by tests/test_oracle.py, which compares it
with the golden vectors tests/golden/*.npz made by tests/golden/make_golden.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libnolf_oracle.so")
SRC = os.path.join(HERE, "nolf_oracle.c")

HEAD_ACT = {"identity": 0, "sigmoid": 1, "exponential": 2}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, OpenMP)."""
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(SRC):
        return SO
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           SRC, "-o", SO, "-lm"]
    subprocess.run(cmd, check=True)
    return SO


class OMlp(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("widths", C.c_int * 5), ("w", C.c_void_p * 4),
                ("b", C.c_void_p * 4), ("n_heads", C.c_int), ("head_act", C.c_int * 8),
                ("head_w", C.c_int * 8)]


class OAtlas(C.Structure):
    _fields_ = [("b", C.c_int), ("r", C.c_int), ("channels", C.c_int), ("index", C.c_void_p),
                ("cubes", C.c_void_p)]


class OAsset(C.Structure):
    _fields_ = [
        ("density", OAtlas), ("has_diffuse_atlas", C.c_int), ("diffuse", OAtlas),
        ("psh_n", C.c_int), ("psh_m", C.c_uint64), ("psh_mphi", C.c_uint64),
        ("psh_offsets", C.c_void_p), ("p0", C.c_uint64 * 3), ("p1", C.c_uint64 * 3),
        ("psh_features", C.c_void_p), ("psh_f", C.c_int),
        ("hg_levels", C.c_int), ("hg_f", C.c_int), ("hg_table", C.c_uint64),
        ("hg_res", C.c_int * 16), ("hg_dense", C.c_int * 16), ("hg_feat", C.c_void_p * 16),
        ("fs", OMlp), ("fd", OMlp),
        ("step", C.c_double), ("t_stop", C.c_double), ("alpha_floor", C.c_double),
        ("pmin", C.c_double * 3), ("pmax", C.c_double * 3),
        ("use_hit_point", C.c_int), ("use_opacity", C.c_int), ("refine_opacity", C.c_int),
        ("use_tint", C.c_int), ("use_diffuse_color", C.c_int),
        ("n_tri", C.c_int64), ("tri", C.c_void_p),
    ]


class ODebug(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "boxhit", "hit", "t_near", "t_far", "t_hit", "alpha_c", "p_h", "o_obj", "d_obj",
        "samples", "istar", "slots", "es", "fs_out", "diffuse")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            build()
        L = C.CDLL(SO)
        vp, i64, dbl = C.c_void_p, C.c_int64, C.c_double
        L.oracle_render_rays.argtypes = [C.POINTER(OAsset), vp, dbl, vp, C.c_int, vp, i64, vp, vp,
                                         vp, C.POINTER(ODebug), C.c_int]
        L.oracle_render_rect.argtypes = [C.POINTER(OAsset), vp, dbl, vp, dbl, dbl, dbl, dbl,
                                         C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, C.c_int]
        L.oracle_compose.argtypes = [C.c_int, i64, vp, vp, dbl, vp, vp, C.c_int]
        L.oracle_camera_dirs.argtypes = [vp, dbl, dbl, dbl, dbl, vp, vp, i64, vp]
        L.oracle_mesh_hit.argtypes = [vp, i64, vp, vp]
        L.oracle_mesh_hit.restype = dbl
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data


class Asset:
    """An OAsset plus the numpy arrays it points into."""

    def __init__(self, asset):
        self.keep = []
        A = OAsset()

        def arr(x, dt):
            y = np.ascontiguousarray(np.asarray(x), dtype=dt)
            self.keep.append(y)
            return y

        def atlas(dst, at):
            dst.b, dst.r, dst.channels = at.base_resolution, at.cube_resolution, at.channels
            dst.index = _p(arr(at.index, np.int32))
            dst.cubes = _p(arr(at.cubes, np.float32))

        atlas(A.density, asset.density_atlas)
        if asset.diffuse_atlas is not None:
            A.has_diffuse_atlas = 1
            atlas(A.diffuse, asset.diffuse_atlas)
        psh = asset.psh
        A.psh_n, A.psh_m, A.psh_mphi = psh.resolution, psh.table_size, psh.offset_size
        A.psh_offsets = _p(arr(psh.offsets, np.int64))
        for k in range(3):
            A.p0[k] = int(np.asarray(psh.primes_h0, np.uint64)[k])
            A.p1[k] = int(np.asarray(psh.primes_h1, np.uint64)[k])
        feats = arr(asset.psh_features, np.float32)
        A.psh_features = _p(feats)
        A.psh_f = feats.shape[1]
        enc = asset.diffuse_encoder
        if enc is not None:
            A.hg_levels, A.hg_f, A.hg_table = enc.levels, enc.features_per_level, enc.table_size
            for l in range(enc.levels):
                A.hg_res[l] = enc.resolutions[l]
                A.hg_dense[l] = int(bool(enc.dense[l]))
                A.hg_feat[l] = _p(arr(asset.diffuse_features[l], np.float32))

        def mlp(dst, m):
            dst.n_layers = len(m.weights)
            dst.widths[0] = m.weights[0].shape[1]
            for i, (w, b) in enumerate(zip(m.weights, m.biases)):
                dst.widths[i + 1] = w.shape[0]
                dst.w[i] = _p(arr(w, np.float32))
                dst.b[i] = _p(arr(b, np.float32))
            dst.n_heads = len(m.heads)
            for i, (a, wd) in enumerate(m.heads):
                dst.head_act[i] = HEAD_ACT[a]
                dst.head_w[i] = wd

        mlp(A.fs, asset.specular_mlp)
        if asset.diffuse_mlp is not None:
            mlp(A.fd, asset.diffuse_mlp)
        A.step, A.t_stop, A.alpha_floor = asset.march.step, asset.march.t_stop, asset.march.alpha_floor
        for k in range(3):
            A.pmin[k] = float(asset.proxy.min[k])
            A.pmax[k] = float(asset.proxy.max[k])
        w = asset.wiring
        A.use_hit_point, A.use_opacity = int(w.use_hit_point), int(w.use_opacity)
        A.refine_opacity, A.use_tint = int(w.refine_opacity), int(w.use_tint)
        A.use_diffuse_color = int(w.use_diffuse_color)
        mesh = getattr(asset, "proxy_mesh", None)
        if mesh is not None:
            v = np.asarray(mesh[0], np.float64).reshape(-1, 3)
            t = np.asarray(mesh[1], np.int64).reshape(-1, 3)
            tri = arr(v[t].reshape(-1, 9), np.float64)
            A.n_tri, A.tri = len(tri), _p(tri)
        self.A = A
        o2w = np.asarray(asset.object_to_world, np.float64)
        self.w2o = np.ascontiguousarray(np.linalg.inv(o2w))
        lin = self.w2o[:3, :3]
        self.scale = float(np.linalg.norm(lin, axis=0).mean())


def render_rays(asset, origins, dirs, counters=None, debug=False, nthreads=0):
    """Oracle of lightfield.render_rays; returns (rgba, depth[, debug dict])."""
    oa = asset if isinstance(asset, Asset) else Asset(asset)
    origins = np.asarray(origins, np.float64)
    dirs = np.ascontiguousarray(dirs, np.float64)
    n = len(dirs)
    shared = n > 0 and origins.strides[0] == 0
    o = np.ascontiguousarray(origins[:1] if shared else origins)
    rgba = np.zeros((n, 4), np.float32)
    depth = np.full(n, np.inf, np.float32)
    cnt = np.zeros(4, np.int64)
    dbg = None
    D = None
    if debug:
        D = dict(boxhit=np.zeros(n, np.uint8), hit=np.zeros(n, np.uint8),
                 t_near=np.zeros(n), t_far=np.zeros(n), t_hit=np.full(n, np.inf),
                 alpha_c=np.zeros(n), p_h=np.zeros((n, 3)), o_obj=np.zeros((n, 3)),
                 d_obj=np.zeros((n, 3)), samples=np.zeros(n, np.int64),
                 istar=np.full(n, -1, np.int64), slots=np.zeros((n, 8), np.int64),
                 es=np.zeros((n, 2), np.float32), fs_out=np.zeros((n, 4), np.float32),
                 diffuse=np.zeros((n, 4), np.float32))
        dbg = ODebug(**{k: _p(v) for k, v in D.items()})
    lib().oracle_render_rays(C.byref(oa.A), _p(oa.w2o), oa.scale, _p(o), 0 if shared else 1,
                             _p(dirs), n, _p(rgba), _p(depth), _p(cnt),
                             C.byref(dbg) if dbg is not None else None, int(nthreads))
    if counters is not None:
        counters.fs_evals += int(cnt[0])
        counters.fd_evals += int(cnt[1])
        counters.hit_pixels += int(cnt[2])
        counters.march_samples += int(cnt[3])
    if debug:
        D["boxhit"] = D["boxhit"].astype(bool)
        D["hit"] = D["hit"].astype(bool)
        return rgba, depth, D
    return rgba, depth


def render_rect(asset, cam, rect=None, counters=None, nthreads=0, transform=None):
    """Oracle of renderer.render_range's pixels: (rgba (h,w,4), depth (h,w))."""
    oa = asset if isinstance(asset, Asset) else Asset(asset)
    w2o, scale = oa.w2o, oa.scale
    if transform is not None:
        w2o = np.ascontiguousarray(np.linalg.inv(np.asarray(transform, np.float64)))
        scale = float(np.linalg.norm(w2o[:3, :3], axis=0).mean())
    x0, y0, x1, y1 = rect if rect is not None else (0, 0, cam.width, cam.height)
    h, w = y1 - y0, x1 - x0
    rgba = np.zeros((h, w, 4), np.float32)
    depth = np.full((h, w), np.inf, np.float32)
    cnt = np.zeros(4, np.int64)
    pose = np.ascontiguousarray(cam.pose, np.float64)
    lib().oracle_render_rect(C.byref(oa.A), _p(w2o), scale, _p(pose), cam.fx, cam.fy, cam.cx,
                             cam.cy, x0, y0, x1, y1, _p(rgba), _p(depth), _p(cnt), int(nthreads))
    if counters is not None:
        counters.fs_evals += int(cnt[0])
        counters.fd_evals += int(cnt[1])
        counters.hit_pixels += int(cnt[2])
        counters.march_samples += int(cnt[3])
    return rgba, depth


def compose(rgba, depth, alpha_vis=0.5, nthreads=0):
    """Oracle of farm.compose on stacked frames rgba (K,H,W,4), depth (K,H,W)."""
    rgba = np.ascontiguousarray(rgba, np.float32)
    depth = np.ascontiguousarray(depth, np.float32)
    K = rgba.shape[0]
    P = int(np.prod(depth.shape[1:]))
    out_rgba = np.zeros(depth.shape[1:] + (4,), np.float32)
    out_depth = np.zeros(depth.shape[1:], np.float32)
    lib().oracle_compose(K, P, _p(rgba), _p(depth), float(alpha_vis), _p(out_rgba),
                         _p(out_depth), int(nthreads))
    return out_rgba, out_depth


def camera_dirs(cam, px, py):
    px = np.ascontiguousarray(px, np.float64)
    py = np.ascontiguousarray(py, np.float64)
    out = np.zeros((len(px), 3))
    pose = np.ascontiguousarray(cam.pose, np.float64)
    lib().oracle_camera_dirs(_p(pose), cam.fx, cam.fy, cam.cx, cam.cy, _p(px), _p(py), len(px),
                             _p(out))
    return out


def encode_frame(rgba, depth, depth_far=10.0):
    """protocol.encode_frame RAW (protocol.py:256-266) restated in numpy:
    rgba8 = clip(round(rgba*255)) in float32 (half-to-even), depth16 =
    round(min(d, far)/far*65534) for finite d, else 65535."""
    rgba = np.asarray(rgba, np.float32)
    depth = np.asarray(depth, np.float32)
    r8 = np.clip(np.round(rgba * np.float32(255.0)), 0, 255).astype(np.uint8)
    q = np.full(depth.shape, 65535, np.uint16)
    fin = np.isfinite(depth)
    far = np.float32(depth_far)
    q[fin] = np.round(np.minimum(depth[fin], far) / far * np.float32(65534.0)).astype(np.uint16)
    return r8, q
