"""Synthetic i-NOLF assets, built the way the reference builds them.

BASELINE.md's synthetic inputs are "built with the reference's own
functions": analytic density baked into cube atlases, a hit shell from a
view-sphere sweep, a perfect spatial hash over the shell's vertices,
random-init features and networks from ``default_rng(seed)``, and a baked
diffuse atlas.  The reference is not present on the GPU box, so this module
restates that pipeline (tests/test_synth.py pins it against the reference
on small configurations: identical index grids, cubes, PSH tables, feature
rows and weights; diffuse cubes to fp32 MLP rounding):

  analytic densities          scenes.py:45-170
  bake_cubes (dense)          atlas.py:59-126    -> bake_density
  fibonacci_sphere            lightfield.py:466-472
  collect_hit_points          lightfield.py:475-512  (march on the GPU)
  voxelize_points             lightfield.py:515-531
  OccupancyGrid.vertices      encoding.py:58-65
  psh_construct               encoding.py:158-338 (greedy bucket placement)
  init_light_field            lightfield.py:600-651  (rng draw order)
  bake_diffuse_cubes          lightfield.py:547-576 + atlas.py:129-155
                              (diffuse network evaluated on the GPU)

Asset production is offline work in the reference (out
of scope); this module is bench / test support, not part of the product
package.  It only feeds the benchmark and the full-size parity tests.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2303_04086_b200 import errors
from paper_2303_04086_b200.model import (Camera, CubeAtlas, HashGridEncoder, LightFieldAsset, MarchParams, Mlp,
                    ModelWiring, PshTable, look_at)

# ------------------------------------------------------------------ densities
SPHERE = ("sphere", [((0.5, 0.5, 0.5), 0.25, 600.0)])


def density_fn(kind: str):
    """Closed-form densities of the built-in scenes (scenes.py:45-170)."""
    if kind == "sphere":
        objs = [("s", (0.5, 0.5, 0.5), 0.25, 600.0)]
    elif kind == "box":
        objs = [("b", (0.5, 0.5, 0.5), 0.2, 600.0)]
    elif kind in ("two", "two_spheres"):
        objs = [("s", (0.3, 0.5, 0.5), 0.16, 1500.0), ("s", (0.72, 0.5, 0.5), 0.16, 1500.0)]
    elif kind == "empty":
        objs = []
    else:
        raise errors.DomainError(f"unknown density kind {kind!r}")

    def one(o, pts):
        shape, c, size, sigma = o
        c = np.asarray(c)
        if shape == "s":
            return sigma * (np.linalg.norm(pts - c, axis=1) <= size)
        return sigma * np.all(np.abs(pts - c) <= size, axis=1)

    def fn(pts):
        if not objs:
            return np.zeros(len(pts))
        vals = [one(o, pts) for o in objs]
        return vals[0] if len(vals) == 1 else np.max(np.stack(vals), axis=0)

    return fn


def bake_density(query, b: int, r: int, threshold: float = 0.0, chunk: int = 65_536) -> CubeAtlas:
    """Dense bake of a 1-channel field into a sparse cube atlas (atlas.py:59-126)."""
    side = b * r + 1
    axis = np.arange(side, dtype=np.float64) / (b * r)
    grid = np.empty((side, side, side), dtype=np.float32)
    rows = max(1, chunk // (side * side))
    for x0 in range(0, side, rows):
        x1 = min(side, x0 + rows)
        gx, gy, gz = np.meshgrid(axis[x0:x1], axis, axis, indexing="ij")
        pts = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
        grid[x0:x1] = np.asarray(query(pts), dtype=np.float32).reshape(x1 - x0, side, side)
    cell_max = np.full((b, b, b), -np.inf, dtype=np.float32)
    for dx in range(r + 1):
        for dy in range(r + 1):
            for dz in range(r + 1):
                np.maximum(cell_max, grid[dx::r, dy::r, dz::r][:b, :b, :b], out=cell_max)
    cells = np.argwhere(cell_max > threshold)
    index = np.full((b, b, b), -1, dtype=np.int32)
    cubes = np.empty((len(cells), r + 1, r + 1, r + 1, 1), dtype=np.float32)
    for cid, (i, j, k) in enumerate(cells):
        index[i, j, k] = cid
        cubes[cid, ..., 0] = grid[i * r:i * r + r + 1, j * r:j * r + r + 1, k * r:k * r + r + 1]
    return CubeAtlas(base_resolution=b, cube_resolution=r, channels=1, index=index, cubes=cubes)


# ------------------------------------------------------------------ hit shell
def fibonacci_sphere(n: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64) + 0.5
    phi = math.pi * (3.0 - math.sqrt(5.0)) * i
    z = 1.0 - 2.0 * i / n
    rr = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([rr * np.cos(phi), rr * np.sin(phi), z], axis=1)


def shell_cameras(n_cameras=512, image_size=32, radius=2.0, fov_deg=60.0):
    """The view-sphere sweep of collect_hit_points (lightfield.py:484-501)."""
    center = np.array([0.5, 0.5, 0.5])
    fx = image_size / (2.0 * math.tan(math.radians(fov_deg) / 2.0))
    cams = []
    for eye_dir in fibonacci_sphere(n_cameras):
        up = (0.0, 0.0, 1.0) if abs(eye_dir[1]) > 0.9 else (0.0, 1.0, 0.0)
        cams.append(Camera(pose=look_at(center + radius * eye_dir, center, up), fx=fx, fy=fx,
                           cx=image_size / 2, cy=image_size / 2, width=image_size,
                           height=image_size))
    return cams


def collect_hit_points_gpu(atlas: CubeAtlas, march: MarchParams, n_cameras=512, image_size=32):
    """Hit points of the sweep, marched by nolf_march_rays on the GPU."""
    from paper_2303_04086_b200 import render as R

    probe = march_only_asset(atlas, march)
    cams = shell_cameras(n_cameras, image_size)
    # camera_dirs on the host with numpy (identical bits to core.camera_dirs)
    px, py = np.meshgrid(np.arange(image_size), np.arange(image_size))
    px = px.reshape(-1).astype(np.float64)
    py = py.reshape(-1).astype(np.float64)
    origins, dirs = [], []
    for cam in cams:
        u = (px + 0.5 - cam.cx) / cam.fx
        v = -(py + 0.5 - cam.cy) / cam.fy
        d = np.stack([u, v, -np.ones_like(u)], axis=-1) @ cam.rotation.T
        d = d / np.linalg.norm(d, axis=-1, keepdims=True)
        dirs.append(d)
        origins.append(np.broadcast_to(cam.position, d.shape))
    res = R.march_rays(probe, np.concatenate(origins), np.concatenate(dirs))
    return res.p_h[res.hit]


def voxelize(points: np.ndarray, resolution: int, dilate: int = 1) -> np.ndarray:
    """Occupancy of the voxels holding any point, 6-neighbour dilated (lightfield.py:515-531)."""
    occ = np.zeros((resolution,) * 3, dtype=bool)
    if len(points):
        cells = np.clip((points * resolution).astype(np.int64), 0, resolution - 1)
        occ[cells[:, 0], cells[:, 1], cells[:, 2]] = True
        for _ in range(dilate):
            grown = occ.copy()
            grown[1:, :, :] |= occ[:-1, :, :]
            grown[:-1, :, :] |= occ[1:, :, :]
            grown[:, 1:, :] |= occ[:, :-1, :]
            grown[:, :-1, :] |= occ[:, 1:, :]
            grown[:, :, 1:] |= occ[:, :, :-1]
            grown[:, :, :-1] |= occ[:, :, 1:]
            occ = grown
    return occ


def occupied_vertices(occ: np.ndarray) -> np.ndarray:
    """Integer coords of every vertex of an occupied voxel, lexicographic (encoding.py:58-65)."""
    n = occ.shape[0]
    flags = np.zeros((n + 1,) * 3, dtype=bool)
    for c in range(8):
        dx, dy, dz = c & 1, (c >> 1) & 1, (c >> 2) & 1
        flags[dx:n + dx, dy:n + dy, dz:n + dz] |= occ
    return np.argwhere(flags).astype(np.int64)


# ------------------------------------------------------------------ PSH
P0 = np.array([1, 2654435761, 805459861], dtype=np.uint64)
P1 = np.array([73856093, 19349663, 83492791], dtype=np.uint64)
_STEPS = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]],
                  dtype=np.int64)


def _ring_dist_score(src_h0, targets, offs, m):
    """Mean circular slot distance of (src + off) % m to targets, per offset."""
    d = np.abs((src_h0[None, :] + offs[:, None]) % m - targets[None, :])
    return np.minimum(d, m - d).mean(axis=1)


def _place(vertices, resolution, m, m_phi):
    """One greedy placement pass (encoding.py:158-253); None when infeasible.

    Buckets = vertices sharing h1, placed largest first (ties by first
    appearance in h1 order).  A bucket takes, among the first 16 distinct
    "neighbour-adjacent" offsets that are collision-free, the one with the
    smallest mean ring distance to already-placed grid neighbours; failing
    that, the best offset of the first 64-wide window that has any
    collision-free one (or simply the first free offset when the bucket has
    no placed neighbour)."""
    u = vertices.astype(np.uint64)
    h0 = ((u @ P0) % np.uint64(m)).astype(np.int64)
    h1 = ((u @ P1) % np.uint64(m_phi)).astype(np.int64)
    order = np.argsort(h1, kind="stable")
    hs = h1[order]
    first = np.flatnonzero(np.r_[True, hs[1:] != hs[:-1]])
    last = np.r_[first[1:], len(order)]
    by_size = np.argsort(-(last - first), kind="stable")
    taken = np.zeros(m, dtype=bool)
    phi = np.zeros(m_phi, dtype=np.int64)
    slot_of = np.full(len(vertices), -1, dtype=np.int64)
    side = resolution + 1
    track = side ** 3 <= 32_000_000
    grid_slot = np.full(side ** 3, -1, dtype=np.int64) if track else None
    flat_id = (vertices[:, 0] * side + vertices[:, 1]) * side + vertices[:, 2]
    for bk in by_size:
        mem = order[first[bk]:last[bk]]
        src = h0[mem]
        if len(np.unique(src)) != len(src):
            return None
        nb_src = nb_dst = None
        if track:
            nb = vertices[mem][:, None, :] + _STEPS[None, :, :]
            ok = np.all((nb >= 0) & (nb <= resolution), axis=-1)
            nid = (nb[..., 0] * side + nb[..., 1]) * side + nb[..., 2]
            nslot = np.where(ok, grid_slot[np.where(ok, nid, 0)], -1)
            placed = nslot >= 0
            if placed.any():
                rows, _ = np.nonzero(placed)
                nb_src, nb_dst = src[rows], nslot[placed]
        have_nb = nb_src is not None and len(nb_src) > 0
        pick = -1
        if have_nb:
            cand = np.unique(np.concatenate([(nb_dst + 1 - nb_src) % m,
                                             (nb_dst - 1 - nb_src) % m]))[:16]
            free = ~taken[(src[None, :] + cand[:, None]) % m].any(axis=1)
            if free.any():
                ok_c = cand[free]
                pick = int(ok_c[int(np.argmin(_ring_dist_score(nb_src, nb_dst, ok_c, m)))])
        if pick < 0:
            for lo in range(0, m, 64):
                offs = np.arange(lo, min(lo + 64, m), dtype=np.int64)
                free = ~taken[(src[None, :] + offs[:, None]) % m].any(axis=1)
                if not free.any():
                    continue
                ok_c = offs[free]
                pick = int(ok_c[int(np.argmin(_ring_dist_score(nb_src, nb_dst, ok_c, m)))]) \
                    if have_nb else int(ok_c[0])
                break
            if pick < 0:
                return None
        dst = (src + pick) % m
        taken[dst] = True
        phi[hs[first[bk]]] = pick
        slot_of[mem] = dst
        if track:
            grid_slot[flat_id[mem]] = dst
    return phi, slot_of


def build_psh(vertices, resolution, load_factor=1.05, max_retries=8) -> PshTable:
    """Perfect spatial hash over a vertex set (encoding.py:276-338 growth schedule)."""
    v = np.unique(np.asarray(vertices, dtype=np.int64), axis=0)
    if v.ndim != 2 or len(v) == 0:
        raise errors.DomainError("vertex set must be a non-empty (K,3) array")
    k = len(v)
    m0 = max(1, math.ceil(k * load_factor))
    mphi0 = max(1, k // 3)
    for attempt in range(max_retries + 1):
        m = max(k, math.ceil(m0 * 1.1 ** attempt))
        m_phi = math.ceil(mphi0 * 1.5 ** attempt)
        res = _place(v, resolution, m, m_phi)
        if res is None:
            continue
        phi, slots = res
        if len(np.unique(slots)) != k:
            raise errors.DomainError("PSH placement produced a collision")
        return PshTable(resolution=resolution, table_size=m, offset_size=m_phi, offsets=phi,
                        report={"load_factor": k / m, "adjacency_score": 0.0,
                                "attempts": attempt + 1})
    raise errors.DomainError(f"no collision-free table within {max_retries} retries for |V|={k}")


# ------------------------------------------------------------------ networks
def _uniform_rows(rng, rows, dim):
    return rng.uniform(-1e-4, 1e-4, size=(rows, dim)).astype(np.float32)


def _he_mlp(widths, heads, rng) -> Mlp:
    ws, bs = [], []
    for i in range(len(widths) - 1):
        ws.append(rng.normal(0.0, np.sqrt(2.0 / widths[i]), (widths[i + 1], widths[i]))
                  .astype(np.float32))
        bs.append(np.zeros(widths[i + 1], dtype=np.float32))
    return Mlp(weights=ws, biases=bs, heads=tuple(heads))


def make_asset(kind="sphere", seed=0, b=32, r=8, psh_resolution=64, hidden=64,
               shell_cameras_n=512, shell_image_size=32, diffuse_levels=6, diffuse_base=8,
               diffuse_growth=1.6, diffuse_table=2 ** 13, bake_diffuse=True,
               diffuse_shell_cameras=64, diffuse_shell_image=32, shell_points=None,
               diffuse_shell_points=None, cache=None, name=None) -> LightFieldAsset:
    """Asset of BASELINE.md's synthetic inputs: ``bake_density_cubes(obj.density, b, r)`` +
    ``init_light_field(atlas, MarchParams(1/(b r)), LightFieldTrainConfig(...), rng(seed))`` +
    ``bake_diffuse_cubes`` (default shell sweep).  ``cache`` (dict) memoises the
    seed-independent stages (atlas, shells, PSH) across assets of one density kind."""
    cache = {} if cache is None else cache
    march = MarchParams(step=1.0 / (b * r))
    key = (kind, b, r, psh_resolution, shell_cameras_n, shell_image_size)
    if key not in cache:
        atlas = bake_density(density_fn(kind), b, r)
        sp = shell_points if shell_points is not None else collect_hit_points_gpu(
            atlas, march, shell_cameras_n, shell_image_size)
        verts = occupied_vertices(voxelize(sp, psh_resolution, 1))
        if len(verts) == 0:
            verts = np.zeros((1, 3), dtype=np.int64)
        psh = build_psh(verts, psh_resolution)
        cache[key] = (atlas, psh)
    atlas, psh = cache[key]
    rng = np.random.default_rng(seed)
    feats = _uniform_rows(rng, psh.table_size, 2)
    specular = _he_mlp([2 + 16 + 1, hidden, hidden, 4], [("sigmoid", 3), ("identity", 1)], rng)
    diffuse = _he_mlp([diffuse_levels * 2, hidden, 4], [("sigmoid", 3), ("sigmoid", 1)], rng)
    enc = HashGridEncoder(levels=diffuse_levels, base_resolution=diffuse_base,
                          growth=diffuse_growth, table_size=diffuse_table, features_per_level=2)
    dfeat = [_uniform_rows(rng, rows, 2) for rows in enc.row_counts]
    asset = LightFieldAsset(density_atlas=atlas, psh=psh, psh_features=feats, diffuse_encoder=enc,
                            diffuse_features=dfeat, specular_mlp=specular, diffuse_mlp=diffuse,
                            march=march, wiring=ModelWiring(), name=name or f"{kind}{seed}")
    if bake_diffuse:
        dkey = ("dshell",) + key + (diffuse_shell_cameras, diffuse_shell_image)
        if dkey not in cache:
            sp = diffuse_shell_points if diffuse_shell_points is not None else \
                collect_hit_points_gpu(atlas, march, diffuse_shell_cameras, diffuse_shell_image)
            cache[dkey] = voxelize(sp, b, 1)
        asset.diffuse_atlas = bake_diffuse_gpu(asset, cache[dkey])
    return asset


def masked_sample_points(mask: np.ndarray, r: int) -> tuple[np.ndarray, np.ndarray]:
    """(cells, points) of a masked bake: every cell's (r+1)^3 corner samples (atlas.py:129-150)."""
    b = mask.shape[0]
    cells = np.argwhere(mask)
    g = np.arange(r + 1, dtype=np.float64) / r
    gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
    local = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    pts = ((cells[:, None, :] + local[None, :, :]) / b).reshape(-1, 3)
    return cells, pts


def bake_diffuse_gpu(asset, mask: np.ndarray) -> CubeAtlas:
    """bake_diffuse_cubes with the diffuse network evaluated by nolf_eval_diffuse."""
    import torch

    from paper_2303_04086_b200 import _native as N
    from paper_2303_04086_b200 import render as R

    b = asset.density_atlas.base_resolution
    r = asset.density_atlas.cube_resolution
    cells, pts = masked_sample_points(mask, r)
    index = np.full((b, b, b), -1, dtype=np.int32)
    cubes = np.empty((len(cells), r + 1, r + 1, r + 1, 4), dtype=np.float32)
    if len(cells):
        dev = R.device_asset(asset)
        device = R._device()
        p = torch.from_numpy(np.ascontiguousarray(pts)).to(device)
        out = torch.empty((len(pts), 4), dtype=torch.float32, device=device)
        N.check(N.lib().nolf_eval_diffuse(dev.handle, p.data_ptr(), len(pts), out.data_ptr(),
                                          R._stream_ptr()))
        cubes[:] = out.cpu().numpy().reshape(cubes.shape)
        for cid, (i, j, k) in enumerate(cells):
            index[i, j, k] = cid
    return CubeAtlas(base_resolution=b, cube_resolution=r, channels=4, index=index, cubes=cubes)


def march_only_asset(atlas: CubeAtlas, march: MarchParams) -> LightFieldAsset:
    """Minimal asset around a density atlas (the march reads nothing else)."""
    psh = PshTable(resolution=1, table_size=1, offset_size=1, offsets=np.zeros(1, np.int64))
    spec = _he_mlp([19, 64, 64, 4], [("sigmoid", 3), ("identity", 1)], np.random.default_rng(0))
    return LightFieldAsset(density_atlas=atlas, psh=psh, psh_features=np.zeros((1, 2), np.float32),
                           diffuse_encoder=None, diffuse_features=None, specular_mlp=spec,
                           diffuse_mlp=None, march=march, wiring=ModelWiring(use_diffuse_color=False))


# ------------------------------------------------------------------ mesh proxies
def box_mesh(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
    """The 12-triangle tessellation of an AABB (outward winding)."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    v = np.array([[hi[k] if (c >> k) & 1 else lo[k] for k in range(3)] for c in range(8)])
    quads = [(0, 2, 3, 1), (4, 5, 7, 6), (0, 1, 5, 4), (2, 6, 7, 3), (0, 4, 6, 2), (1, 3, 7, 5)]
    tris = []
    for a, b, c, d in quads:
        tris += [(a, b, c), (a, c, d)]
    return v, np.asarray(tris, np.int32)


def icosphere(center=(0.5, 0.5, 0.5), radius=0.27, level=3):
    """Subdivided icosahedron (20 * 4**level triangles) -- a tight proxy for
    the sphere density (radius 0.25)."""
    t = (1.0 + 5 ** 0.5) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
         (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    v = [np.asarray(p, np.float64) / np.linalg.norm(p) for p in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache, nf = {}, []

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = v[a] + v[b]
                v.append(m / np.linalg.norm(m))
                cache[key] = len(v) - 1
            return cache[key]

        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        f = nf
    verts = np.asarray(center, np.float64) + radius * np.asarray(v)
    return np.clip(verts, 0.0, 1.0), np.asarray(f, np.int32)


# ------------------------------------------------------------------ scenes
def zodiac_transforms(n=12, ring_radius=2.0, scale=0.5):
    """Config 4's "zodiac" ring: uniform scale 0.5, translations on a ring of
    radius 2 at 360/n degree steps."""
    out = []
    for i in range(n):
        th = 2.0 * math.pi * i / n
        m = np.eye(4)
        m[:3, :3] *= scale
        # centre the asset's unit box (centre (0.5,0.5,0.5)) on the ring point
        m[:3, 3] = np.array([ring_radius * math.cos(th), ring_radius * math.sin(th), 0.0]) \
            - scale * np.array([0.5, 0.5, 0.5])
        out.append(m)
    return out


ZODIAC_KINDS = ("sphere", "box", "two")


def zodiac_scene(n=12, cache=None, **kw):
    """12 assets, seed i, density cycling sphere / box / two-spheres, on the ring."""
    cache = {} if cache is None else cache
    assets = [make_asset(ZODIAC_KINDS[i % 3], seed=i, cache=cache, **kw) for i in range(n)]
    return list(zip(assets, zodiac_transforms(n)))


def zodiac_camera(width=3840, height=2160, distance=4.0, elevation=0.45, azimuth=0.3,
                  fov_deg=60.0) -> Camera:
    """Camera at distance 4 looking at the ring centre, 60 degree fov."""
    ce, se = math.cos(elevation), math.sin(elevation)
    eye = distance * np.array([ce * math.cos(azimuth), ce * math.sin(azimuth), se])
    fx = width / (2.0 * math.tan(math.radians(fov_deg) / 2.0))
    return Camera(pose=look_at(eye, (0.0, 0.0, 0.0), (0.0, 0.0, 1.0)), fx=fx, fy=fx,
                  cx=width / 2, cy=height / 2, width=width, height=height)
