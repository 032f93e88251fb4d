"""CUDA path (libnolf_b200.so via the reference-signature host mirror) vs the
reference goldens and the pinned C oracle.

Bar (BASELINE.json north_star): bit-exact hit flags / hit indices / PSH
addresses (checked through the oracle, which is itself pinned to the
reference's integers in test_oracle.py, and through depth bits, which encode
t_hit = t_near + (i*+0.5)*step exactly); pixels within 1e-3 in fp32.  The
fp32 CUDA MLP uses the oracle's sequential-FMA order, so in practice the GPU
matches the oracle to the last bit and the reference to ~1e-6."""

import dataclasses

import numpy as np
import pytest

from golden_util import asset, camera, case_asset, load, render_cases
from oracle import oracle as O
from paper_2303_04086_b200 import render as R
from paper_2303_04086_b200.model import Frame, RayRange, RenderCounters, orbit_camera

pytestmark = pytest.mark.gpu
TOL = 1e-3   # north_star: max abs error <= 1e-3 in fp32


def _assert_frame(rgba, depth, g_rgba, g_depth, tol=TOL):
    fin = np.isfinite(g_depth)
    assert np.array_equal(np.isfinite(depth), fin), "hit/miss pattern differs"
    assert np.array_equal(depth[fin], g_depth[fin]), "depth bits differ (hit index / t_hit)"
    err = np.abs(rgba.astype(np.float64) - g_rgba).max() if rgba.size else 0.0
    assert err <= tol, f"max |rgba err| {err}"
    return err


@pytest.mark.parametrize("case", render_cases())
def test_render_range_vs_reference(case):
    g = load(f"render_{case}.npz")
    a = case_asset(case, g)
    cam = camera(g)
    x0, y0, x1, y1 = (int(v) for v in g["rect"])
    cnt = RenderCounters()
    tile, instr = R.render_range(a, RayRange(cam, x0, y0, x1, y1), cnt)
    err = _assert_frame(tile.rgba.reshape(-1, 4), tile.depth.reshape(-1), g["rgba"], g["depth"])
    assert [cnt.fs_evals, cnt.fd_evals, cnt.hit_pixels, cnt.march_samples] == g["counters"].tolist()
    assert instr["rays"] == (x1 - x0) * (y1 - y0)
    # oracle agreement is tighter than the reference tolerance
    o_rgba, o_depth = O.render_rect(a, cam, (x0, y0, x1, y1))
    assert np.abs(tile.rgba - o_rgba).max() <= 1e-6
    assert np.array_equal(tile.depth, o_depth)
    print(case, "max err vs reference", err)


@pytest.mark.parametrize("name", ["rays_sphere", "rays_sphere_xform"])
def test_render_rays_vs_reference(name):
    g = load(f"{name}.npz")
    a = case_asset("sphere", g)
    cnt = RenderCounters()
    rgba, depth = R.render_rays(a, g["origins"], g["dirs"], cnt)
    _assert_frame(rgba, depth, g["rgba"], g["depth"])
    assert [cnt.fs_evals, cnt.fd_evals, cnt.hit_pixels, cnt.march_samples] == g["counters"].tolist()


def test_compose_vs_reference():
    g = load("compose.npz")
    n = len([k for k in g if k.startswith("in_rgba_")])
    for i in range(n):
        rgba, depth = g[f"in_rgba_{i}"], g[f"in_depth_{i}"]
        k, h, w = depth.shape
        frames = [Frame(w, h, rgba[j], depth[j]) for j in range(k)]
        out = R.compose(frames)
        np.testing.assert_array_equal(out.rgba, g[f"out_rgba_{i}"])
        np.testing.assert_array_equal(out.depth, g[f"out_depth_{i}"])


def _scene():
    g = load("scene.npz")
    names = {"sphere": "toy_sphere", "box": "toy_box", "two": "toy_two"}
    scene = [(asset(names[str(n)]), tr) for n, tr in zip(g["names"], g["transforms"])]
    return g, scene


def test_render_frame_and_compose_vs_reference():
    g, scene = _scene()
    cam = camera(g)
    frames = R.render_frame(scene, cam)
    for k, f in enumerate(frames):
        _assert_frame(f.rgba, f.depth, g["frame_rgba"][k], g["frame_depth"][k])
    out = R.compose(frames)
    _assert_frame(out.rgba, out.depth, g["rgba"], g["depth"])


@pytest.mark.parametrize("tile", [32, 17, 8])
def test_fused_scene_vs_reference(tile):
    g, scene = _scene()
    cam = camera(g)
    cnt = RenderCounters()
    out = R.render_scene(scene, cam, cnt, tile=tile)
    _assert_frame(out.rgba, out.depth, g["rgba"], g["depth"])
    # the fused path composes exactly what compose(render_frame) composes
    ref = R.compose(R.render_frame(scene, cam))
    np.testing.assert_array_equal(out.rgba, ref.rgba)
    np.testing.assert_array_equal(out.depth, ref.depth)


def test_partition_determinism():
    """Any tiling of a frame gives bit-identical pixels (test_renderer.py:38-48)."""
    a = asset("toy_sphere")
    cam = orbit_camera(0.4, 0.3, radius=2.0, size=48)
    full, _ = R.render_range(a, RayRange(cam, 0, 0, 48, 48))
    rgba = np.zeros_like(full.rgba)
    depth = np.zeros_like(full.depth)
    for ty in range(0, 48, 17):
        for tx in range(0, 48, 17):
            x1, y1 = min(tx + 17, 48), min(ty + 17, 48)
            t, _ = R.render_range(a, RayRange(cam, tx, ty, x1, y1))
            rgba[ty:y1, tx:x1] = t.rgba
            depth[ty:y1, tx:x1] = t.depth
    np.testing.assert_array_equal(full.rgba, rgba)
    np.testing.assert_array_equal(full.depth, depth)


def test_proxy_miss_and_empty_inputs():
    a = asset("toy_sphere")
    cnt = RenderCounters()
    rgba, depth = R.render_rays(a, np.array([[5.0, 5.0, 5.0]]), np.array([[0.0, 0.0, 1.0]]), cnt)
    assert np.all(rgba == 0) and np.isinf(depth[0]) and cnt.fs_evals == 0
    rgba, depth = R.render_rays(a, np.zeros((0, 3)), np.zeros((0, 3)))
    assert rgba.shape == (0, 4) and depth.shape == (0,)


def test_hitting_ray_queries_specular_once():
    a = asset("toy_sphere")
    cnt = RenderCounters()
    rgba, depth = R.render_rays(a, np.array([[-1.0, 0.5, 0.5]]), np.array([[1.0, 0.0, 0.0]]), cnt)
    assert cnt.fs_evals == 1 and cnt.hit_pixels == 1 and np.isfinite(depth[0])


def test_mutated_mlp_is_reuploaded():
    a = asset("toy_sphere")
    a2 = dataclasses.replace(a, specular_mlp=dataclasses.replace(
        a.specular_mlp, biases=[b.copy() for b in a.specular_mlp.biases]))
    cam = orbit_camera(0.8, 0.3, radius=2.0, size=32)
    t1, _ = R.render_range(a2, RayRange(cam, 0, 0, 32, 32))
    a2.specular_mlp.biases[-1][:3] += 2.0
    t2, _ = R.render_range(a2, RayRange(cam, 0, 0, 32, 32))
    assert np.abs(t1.rgba - t2.rgba).max() > 1e-3


def test_live_diffuse_eval_vs_reference():
    g = load("render_live_far.npz")
    a = case_asset("live", g)
    import torch
    from paper_2303_04086_b200 import _native as N
    dev = R.device_asset(a)
    p = torch.from_numpy(np.ascontiguousarray(g["shade_p"])).cuda()
    out = torch.empty((len(p), 4), dtype=torch.float32, device="cuda")
    N.check(N.lib().nolf_eval_diffuse(dev.handle, p.data_ptr(), len(p), out.data_ptr(),
                                      R._stream_ptr()))
    np.testing.assert_allclose(out.cpu().numpy(), g["diffuse"], rtol=0, atol=2e-6)


@pytest.mark.parametrize("tile", [32, 17, 8])
def test_fused_scene_encoded_frame(tile):
    """rgba8 + u16 depth written by the compose epilogue (encode_frame RAW,
    protocol.py:256-266): bit-equal to the oracle's encoder applied to the
    fused f32 frame, and within one rgba8 step / bit-equal depth vs the
    reference-encoded golden (tile 32 and 8 take the 4-slot vector path,
    tile 17 the per-slot path)."""
    import torch
    g, scene = _scene()
    enc = load("encode.npz")
    cam = camera(g)
    f32 = R.render_scene(scene, cam, tile=tile)
    r = R.SceneRenderer(scene)
    tiles = R.frame_tiles(cam.width, cam.height, tile)
    out = r.alloc(len(tiles), tile * tile, want_f32=False, want_u8=True)
    r.render([cam], torch.from_numpy(tiles).to(r.device), len(tiles), tile * tile, out, frame_layout=True)
    npx = cam.width * cam.height
    rgba8 = out["rgba8"][:npx].cpu().numpy().reshape(cam.height, cam.width, 4)
    depth16 = out["depth16"][:npx].cpu().numpy().view(np.uint16).reshape(cam.height, cam.width)
    e8, e16 = O.encode_frame(f32.rgba, f32.depth)
    np.testing.assert_array_equal(rgba8, e8)
    np.testing.assert_array_equal(depth16, e16)
    np.testing.assert_array_equal(depth16, enc["scene_depth16"])
    assert np.abs(rgba8.astype(int) - enc["scene_rgba8"].astype(int)).max() <= 1


@pytest.mark.parametrize("b,r", [(12, 3), (16, 3), (8, 8)])
def test_any_grid_matches_oracle(b, r):
    """The march has an integer sub-voxel path for power-of-two b and r (the
    reference defaults) and the general fp64 path otherwise: both must match
    the oracle bit for bit on depth / counters (rgba to 1e-6)."""
    from tools import synth
    from paper_2303_04086_b200.model import orbit_camera
    a = synth.make_asset("sphere", 5, b=b, r=r, psh_resolution=16, diffuse_levels=3,
                         diffuse_table=2 ** 10, shell_cameras_n=12, shell_image_size=16,
                         diffuse_shell_cameras=8, diffuse_shell_image=8)
    cam = orbit_camera(0.7, 0.4, radius=1.6, size=64)
    cnt, ocnt = RenderCounters(), RenderCounters()
    tile, _ = R.render_range(a, RayRange(cam, 0, 0, 64, 64), cnt)
    o_rgba, o_depth = O.render_rect(a, cam, (0, 0, 64, 64), ocnt)
    assert np.isfinite(o_depth).sum() > 100
    assert np.array_equal(tile.depth, o_depth)
    assert np.abs(tile.rgba - o_rgba).max() <= 1e-6
    assert (cnt.hit_pixels, cnt.march_samples) == (ocnt.hit_pixels, ocnt.march_samples)


def test_multi_camera_launch_equals_single_camera_launches():
    """One launch over the tiles of two cameras (the multi-user batch of
    BASELINE configs 3/5: compacted live chunks, per-camera frame bases)
    gives each camera's frame bit for bit as rendering it alone."""
    import torch
    from paper_2303_04086_b200.model import orbit_camera
    _, scene = _scene()
    cams = [orbit_camera(0.5, 0.6, radius=2.5, size=64, target=(0.2, 0.2, 0.25)),
            orbit_camera(2.0, 0.3, radius=2.2, size=64, target=(0.1, 0.3, 0.2))]
    r = R.SceneRenderer(scene)
    tiles = np.concatenate([R.frame_tiles(64, 64, 32, cam=c) for c in range(2)])
    out = r.alloc(len(tiles), 1024, want_f32=False, want_u8=True)
    r.render(cams, torch.from_numpy(tiles).to(r.device), len(tiles), 1024, out, frame_layout=True)
    both = out["rgba8"][:2 * 64 * 64].cpu().numpy().reshape(2, 64, 64, 4)
    both_d = out["depth16"][:2 * 64 * 64].cpu().numpy().view(np.uint16).reshape(2, 64, 64)
    for c in range(2):
        one = r.alloc(4, 1024, want_f32=False, want_u8=True)
        t1 = R.frame_tiles(64, 64, 32)
        r.render([cams[c]], torch.from_numpy(t1).to(r.device), len(t1), 1024, one, frame_layout=True)
        np.testing.assert_array_equal(both[c], one["rgba8"][:64 * 64].cpu().numpy().reshape(64, 64, 4))
        np.testing.assert_array_equal(both_d[c], one["depth16"][:64 * 64].cpu().numpy().view(np.uint16).reshape(64, 64))
    assert (both_d != 65535).sum() > 0


def test_prefilled_output_skips_only_unreachable_pixels():
    """NolfSceneOut.prefilled: with the frame pre-set to the miss encoding,
    the compose epilogue skips chunks no screen box reaches and the frame is
    bit-identical to a full write (multi-GPU frame composer, bench.py)."""
    import torch
    from paper_2303_04086_b200.model import orbit_camera
    _, scene = _scene()
    cam = orbit_camera(0.5, 0.6, radius=2.5, size=256, target=(0.2, 0.2, 0.25))
    r = R.SceneRenderer(scene)
    tiles = torch.from_numpy(R.frame_tiles(256, 256, 32)).to(r.device)
    full = r.alloc(len(tiles), 1024, want_f32=False, want_u8=True)
    r.render([cam], tiles, len(tiles), 1024, full, frame_layout=True)
    pre = r.alloc(len(tiles), 1024, want_f32=False, want_u8=True)
    pre["rgba8"].zero_()
    pre["depth16"].fill_(-1)
    r.render([cam], tiles, len(tiles), 1024, pre, frame_layout=True, prefilled=True)
    n = 256 * 256
    assert torch.equal(full["rgba8"][:n], pre["rgba8"][:n])
    assert torch.equal(full["depth16"][:n], pre["depth16"][:n])
    assert (full["depth16"][:n] != -1).sum().item() > 0


@pytest.mark.parametrize("seed", range(6))
def test_random_scene_matches_oracle(seed):
    """Randomised placements and cameras (rotation, non-unit uniform scale,
    overlap, assets partly behind the camera): the fused scene path with all
    its exact skipping (screen / chunk / warp culling, occupied-box clip,
    no-clip fast path, distance-field jumps, zero masks) against the oracle,
    which evaluates every fixed march step: depth bits and counters equal,
    rgba to 1e-6 (fp32 MLP)."""
    import math
    from paper_2303_04086_b200.model import orbit_camera
    rng = np.random.default_rng(100 + seed)
    names = ["toy_sphere", "toy_box", "toy_two", "toy_norefine"]
    scene = []
    for i in range(4):
        a = asset(names[rng.integers(len(names))])
        th, ph = rng.uniform(0, 2 * math.pi), rng.uniform(-1, 1)
        c, s_ = math.cos(th), math.sin(th)
        rot = np.array([[c, -s_, 0], [s_, c, 0], [0, 0, 1]]) @ np.array(
            [[1, 0, 0], [0, math.cos(ph), -math.sin(ph)], [0, math.sin(ph), math.cos(ph)]])
        m = np.eye(4)
        m[:3, :3] = rot * rng.uniform(0.3, 0.8)
        m[:3, 3] = rng.uniform(-0.8, 0.8, 3)
        scene.append((a, m))
    cam = orbit_camera(rng.uniform(0, 2 * math.pi), rng.uniform(-0.6, 0.9), radius=rng.uniform(1.2, 3.0),
                       size=64, target=tuple(rng.uniform(-0.2, 0.6, 3)))
    cnt = RenderCounters()
    out = R.render_scene(scene, cam, cnt, tile=32)
    rg, dp = [], []
    ocnt = RenderCounters()
    for a, m in scene:
        r_, d_ = O.render_rect(a, cam, (0, 0, 64, 64), ocnt, transform=m)
        rg.append(r_)
        dp.append(d_)
    o_rgba, o_depth = O.compose(np.stack(rg), np.stack(dp))
    assert np.array_equal(out.depth, o_depth), "depth bits differ from the every-step oracle"
    assert np.abs(out.rgba - o_rgba).max() <= 1e-6
    assert (cnt.hit_pixels, cnt.march_samples) == (ocnt.hit_pixels, ocnt.march_samples)


_FULL = {}


def _full_size(kind):
    """A reference-default asset (b=32, r=8, PSH N=64: power-of-two grid path)."""
    from tools import synth
    if kind not in _FULL:
        _FULL[kind] = synth.make_asset(kind, seed=7, shell_cameras_n=64, shell_image_size=32,
                                       diffuse_shell_cameras=16, diffuse_shell_image=16)
    return _FULL[kind]


@pytest.mark.parametrize("seed", range(3))
def test_random_full_size_scene_matches_oracle(seed):
    """As above with reference-default (b=32, r=8, N=64) assets: the integer
    sub-voxel path, long distance-field jumps and the zero masks at full
    resolution, against the every-step oracle."""
    import math
    from paper_2303_04086_b200.model import orbit_camera
    rng = np.random.default_rng(200 + seed)
    scene = []
    for kind in ("sphere", "box", "two"):
        m = np.eye(4)
        th = rng.uniform(0, 2 * math.pi)
        rot = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
        m[:3, :3] = rot * rng.uniform(0.4, 0.9)
        m[:3, 3] = rng.uniform(-0.6, 0.6, 3)
        scene.append((_full_size(kind), m))
    cam = orbit_camera(rng.uniform(0, 2 * math.pi), rng.uniform(-0.5, 0.8), radius=rng.uniform(1.5, 2.5),
                       size=96, target=tuple(rng.uniform(0.0, 0.5, 3)))
    cnt, ocnt = RenderCounters(), RenderCounters()
    out = R.render_scene(scene, cam, cnt, tile=32)
    rg, dp = [], []
    for a, m in scene:
        r_, d_ = O.render_rect(a, cam, (0, 0, 96, 96), ocnt, transform=m)
        rg.append(r_)
        dp.append(d_)
    o_rgba, o_depth = O.compose(np.stack(rg), np.stack(dp))
    assert np.isfinite(o_depth).sum() > 50
    assert np.array_equal(out.depth, o_depth), "depth bits differ from the every-step oracle"
    assert np.abs(out.rgba - o_rgba).max() <= 1e-6
    assert (cnt.hit_pixels, cnt.march_samples) == (ocnt.hit_pixels, ocnt.march_samples)


@pytest.mark.parametrize("size", [(256, 256), (200, 136)])
def test_sparse_frame_pack_and_host_scatter(size):
    """NolfSceneOut.pack (only the non-miss 8-pixel runs of live chunks leave
    the GPU) + nolf_host_scatter rebuild the encode_frame RAW frame on the
    host bit for bit, across frames (runs written before and missed now are
    reset)."""
    import torch
    from paper_2303_04086_b200 import _native as N
    from paper_2303_04086_b200.model import orbit_camera
    _, scene = _scene()
    W, H = size
    r = R.SceneRenderer(scene)
    tiles = R.frame_tiles(W, H, 32)
    tiles_dev = torch.from_numpy(tiles).to(r.device)
    n_chunks = len(tiles) * 1024 // 128
    host8 = np.zeros((H, W, 4), np.uint8)
    host16 = np.full((H, W), 65535, np.uint16)
    dirty = np.zeros(n_chunks, np.uint16)
    for az in (0.5, 1.7, 1.75):
        cam = orbit_camera(az, 0.6, radius=2.5, width=W, height=H, target=(0.2, 0.2, 0.25))
        dev = {"pack": torch.zeros(n_chunks * 16 * 48, dtype=torch.uint8, device=r.device),
               "pack_ids": torch.zeros(n_chunks * 3, dtype=torch.int32, device=r.device),
               "pack_count": torch.zeros(2, dtype=torch.int32, device=r.device),
               "counters": torch.zeros(4, dtype=torch.int64, device=r.device)}
        r.render([cam], tiles_dev, len(tiles), 1024, dev, frame_layout=True, prefilled=True)
        ref = r.alloc(len(tiles), 1024, want_f32=False, want_u8=True)
        r.render([cam], tiles_dev, len(tiles), 1024, ref, frame_layout=True)
        r.check()
        n_live, n_runs = (int(v) for v in dev["pack_count"].cpu().numpy())
        assert 0 < n_live < n_chunks and 0 < n_runs < 16 * n_live
        runs = dev["pack"][:max(n_runs, 1) * 48].cpu().numpy()
        heads = dev["pack_ids"][:n_live * 3].cpu().numpy().astype(np.uint32)
        tl = np.ascontiguousarray(tiles, np.int32)
        N.check(N.lib().nolf_host_scatter(runs.ctypes.data, heads.ctypes.data, n_live, tl.ctypes.data, len(tl), 1024,
                                          W, H, host8.ctypes.data, host16.ctypes.data, dirty.ctypes.data, 0))
        np.testing.assert_array_equal(host8.reshape(-1, 4), ref["rgba8"][:W * H].cpu().numpy())
        np.testing.assert_array_equal(host16.reshape(-1), ref["depth16"][:W * H].cpu().numpy().view(np.uint16))


def test_compose_any_number_of_frames():
    """nolf_compose with K = 100 frames (beyond the per-thread sort's 64):
    bit-equal to the oracle's farm.compose."""
    import torch
    rng = np.random.default_rng(9)
    K, P = 100, 4096
    a = rng.uniform(0, 1, (K, P)).astype(np.float32)
    a[rng.uniform(size=(K, P)) < 0.3] = 0
    rgba = np.concatenate([rng.uniform(0, 1, (K, P, 3)).astype(np.float32) * a[..., None], a[..., None]], -1)
    depth = np.where(a > 0, rng.choice([1.0, 1.5, 2.0], (K, P)), np.inf).astype(np.float32)
    o, d = R.compose_device(torch.from_numpy(rgba).cuda(), torch.from_numpy(depth).cuda())
    eo, ed = O.compose(rgba, depth)
    np.testing.assert_array_equal(o.cpu().numpy(), eo)
    np.testing.assert_array_equal(d.cpu().numpy(), ed)


def test_scene_with_more_than_64_instances():
    """70 placed assets in one fused launch (instance groups of 64, up to 255
    compose layers): equal to compose(render_frame) bit for bit, and to the
    every-step oracle in depth bits."""
    import math
    from paper_2303_04086_b200.model import orbit_camera
    names = ["toy_sphere", "toy_box", "toy_two"]
    scene = []
    for i in range(70):
        m = np.eye(4)
        m[:3, :3] *= 0.35
        th = 2 * math.pi * i / 35
        m[:3, 3] = [0.9 * math.cos(th), 0.9 * math.sin(th), 0.25 * (i // 35) - 0.1]
        scene.append((asset(names[i % 3]), m))
    cam = orbit_camera(0.4, 0.7, radius=3.0, size=64, target=(0.0, 0.0, 0.0))
    out = R.render_scene(scene, cam)
    ref = R.compose(R.render_frame(scene, cam))
    np.testing.assert_array_equal(out.rgba, ref.rgba)
    np.testing.assert_array_equal(out.depth, ref.depth)
    assert np.isfinite(out.depth).sum() > 200


def test_more_than_32_cameras_in_one_launch():
    """40 cameras' tiles in one launch == each camera alone (bitwise)."""
    import torch
    from paper_2303_04086_b200.model import orbit_camera
    _, scene = _scene()
    cams = [orbit_camera(0.15 * c, 0.5, radius=2.5, size=32, target=(0.2, 0.2, 0.25)) for c in range(40)]
    r = R.SceneRenderer(scene)
    tiles = np.concatenate([R.frame_tiles(32, 32, 32, cam=c) for c in range(40)])
    out = r.alloc(len(tiles), 1024, want_f32=False, want_u8=True)
    r.render(cams, torch.from_numpy(tiles).to(r.device), len(tiles), 1024, out, frame_layout=True)
    allf = out["rgba8"][:40 * 1024].cpu().numpy().reshape(40, 32, 32, 4)
    for c in (0, 17, 39):
        one = r.alloc(1, 1024, want_f32=False, want_u8=True)
        t1 = R.frame_tiles(32, 32, 32)
        r.render([cams[c]], torch.from_numpy(t1).to(r.device), 1, 1024, one, frame_layout=True)
        np.testing.assert_array_equal(allf[c], one["rgba8"][:1024].cpu().numpy().reshape(32, 32, 4))
    r.check()


def test_encode_frame_vs_reference():
    """render.encode_frame (protocol.encode_frame, protocol.py:256-279), RAW
    and ENC_DEFLATE, byte-equal to the reference's messages (encode.npz)."""
    from paper_2303_04086_b200.model import ENC_DEFLATE, ENC_RAW
    g, _ = _scene()
    enc = load("encode.npz")
    h, w = g["depth"].shape
    fr = Frame(width=w, height=h, rgba=g["rgba"], depth=g["depth"])
    raw = R.encode_frame(fr, ENC_RAW)
    assert raw.rgba == enc["scene_rgba8"].tobytes() and raw.depth == enc["scene_depth16"].astype("<u2").tobytes()
    z = R.encode_frame(fr, ENC_DEFLATE)
    assert z.encoding == ENC_DEFLATE and z.rgba == enc["scene_deflate_rgba"].tobytes()
    assert z.depth == enc["scene_deflate_depth"].tobytes()
    syn = R.encode_frame(Frame(width=16, height=16, rgba=enc["syn_rgba"], depth=enc["syn_depth"]), ENC_DEFLATE, 7.5)
    assert syn.rgba == enc["syn_deflate_rgba"].tobytes() and syn.depth == enc["syn_deflate_depth"].tobytes()


def test_prefilled_frame_with_chunk_state_over_frames():
    """NolfSceneOut.chunk_state: one frame buffer re-used across cameras is
    never cleared as a whole -- the library resets the chunks it wrote last
    time that are not live now -- and every frame equals a full render."""
    import torch
    from paper_2303_04086_b200.model import orbit_camera
    _, scene = _scene()
    r = R.SceneRenderer(scene)
    tiles = torch.from_numpy(R.frame_tiles(256, 256, 32)).to(r.device)
    n = 256 * 256
    buf = {"rgba8": torch.zeros((n, 4), dtype=torch.uint8, device=r.device),
           "depth16": torch.full((n,), -1, dtype=torch.int16, device=r.device),
           "chunk_state": torch.zeros(len(tiles) * 8, dtype=torch.int16, device=r.device),
           "counters": torch.zeros(4, dtype=torch.int64, device=r.device)}
    for az in (0.5, 1.3, 2.9, 0.6):
        cam = orbit_camera(az, 0.6, radius=2.5, size=256, target=(0.2, 0.2, 0.25))
        r.render([cam], tiles, len(tiles), 1024, buf, frame_layout=True, prefilled=True)
        full = r.alloc(len(tiles), 1024, want_f32=False, want_u8=True)
        r.render([cam], tiles, len(tiles), 1024, full, frame_layout=True)
        assert torch.equal(buf["rgba8"], full["rgba8"][:n]) and torch.equal(buf["depth16"], full["depth16"][:n])
    assert int((buf["chunk_state"] != 0).sum()) > 0
    r.check()


def test_multi_view_launch_vs_oracle():
    """One launch over two cameras' tiles (the multi-user batches of BASELINE
    configs 3 / 5) against the oracle's render_frame + compose of each
    camera: depth bits and counters equal, rgba <= 1e-6 (fp32 MLP)."""
    import torch
    from paper_2303_04086_b200.model import orbit_camera
    _, scene = _scene()
    cams = [orbit_camera(0.5, 0.6, radius=2.5, size=64, target=(0.2, 0.2, 0.25)),
            orbit_camera(2.6, -0.3, radius=2.0, size=64, target=(0.1, 0.3, 0.2))]
    r = R.SceneRenderer(scene)
    tiles = np.concatenate([R.frame_tiles(64, 64, 32, cam=c) for c in range(2)])
    out = r.alloc(len(tiles), 1024, want_f32=True, want_u8=False)
    r.render(cams, torch.from_numpy(tiles).to(r.device), len(tiles), 1024, out, frame_layout=True)
    r.check()
    got_rgba = out["rgba"][:2 * 4096].cpu().numpy().reshape(2, 64, 64, 4)
    got_depth = out["depth"][:2 * 4096].cpu().numpy().reshape(2, 64, 64)
    cnt = out["counters"].cpu().numpy()
    from paper_2303_04086_b200.model import RenderCounters
    oc = RenderCounters()
    for c, cam in enumerate(cams):
        rg, dp = [], []
        for a, m in scene:
            r_, d_ = O.render_rect(a, cam, (0, 0, 64, 64), oc, transform=m)
            rg.append(r_)
            dp.append(d_)
        o_rgba, o_depth = O.compose(np.stack(rg), np.stack(dp))
        assert np.array_equal(got_depth[c], o_depth)
        assert np.abs(got_rgba[c] - o_rgba).max() <= 1e-6
    assert (int(cnt[2]), int(cnt[3])) == (oc.hit_pixels, oc.march_samples)
