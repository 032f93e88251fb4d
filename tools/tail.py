"""March tail of one rank's shard (diagnostic; needs the -DNOLF_STATS build).

Renders rank R's tile rows of an N-GPU partition on ONE GPU (what that rank
marches), then reads the per-CTA globaltimer spans of the last march launch:
the active-CTA profile over time and the heaviest CTAs.

usage: NOLF_LIB=.../libnolf_stats.so python tools/tail.py --config 4 --world 4 --rank 0
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import ctypes
    import torch
    import bench
    from paper_2303_04086_b200 import _native as N
    from paper_2303_04086_b200.dist import partition, shard_tiles
    from paper_2303_04086_b200.render import SceneRenderer, frame_tiles
    argv = sys.argv[1:]
    world = int(argv[argv.index("--world") + 1]) if "--world" in argv else 4
    rank = int(argv[argv.index("--rank") + 1]) if "--rank" in argv else 0
    argv = [a for i, a in enumerate(argv) if a not in ("--world", "--rank") and
            (i == 0 or argv[i - 1] not in ("--world", "--rank"))]
    sys.argv = [sys.argv[0]] + argv
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    scene, views, W, H, desc = bench.workload(args)
    n_views = len(views(0))
    R = SceneRenderer(scene)
    R.mlp_mode(N.MLP_BF16)
    T = args.tile
    stride = T * T
    tiles = np.concatenate([frame_tiles(W, H, T, cam=v) for v in range(n_views)])
    parts = partition(tiles, world, T, by_rows=True, weights=None)
    mine, n_max = shard_tiles(tiles, world, rank, parts)
    my_tiles = torch.from_numpy(mine).to(dev)
    out = R.alloc(n_max, stride, want_f32=False, want_u8=True)
    cams = [R.camera_array(views(k)) for k in range(12)]
    R.reserve(cams, n_max * stride)
    for k in range(12):
        R.render(cams[k], my_tiles, n_max, stride, out)
    torch.cuda.synchronize()
    n = 1 << 20
    st = (ctypes.c_ulonglong * n)()
    en = (ctypes.c_ulonglong * n)()
    N.lib().nolf_stats_cta(st, en, n)          # resets the end stamps
    wk = (ctypes.c_uint * (4 * n))()
    N.lib().nolf_stats_work(wk, n)
    R.render(cams[11], my_tiles, n_max, stride, out)
    torch.cuda.synchronize()
    N.lib().nolf_stats_cta(st, en, n)
    N.lib().nolf_stats_work(wk, n)
    work = np.frombuffer(wk, np.uint32).reshape(n, 4)
    s = np.frombuffer(st, np.uint64).astype(np.int64)
    e = np.frombuffer(en, np.uint64).astype(np.int64)
    ok = (s > 0) & (e > s)
    work = work[ok]
    s, e = s[ok], e[ok]
    t0 = s.min()
    s, e = (s - t0) / 1e3, (e - t0) / 1e3     # us
    d = e - s
    live = d > 1.0                               # CTAs past the live list exit at once
    print(f"{desc}: rank {rank}/{world}: {ok.sum()} CTAs, march span {e.max():.1f} us, "
          f"last start {s.max():.1f} us, sum of durations {d.sum() / 148:.1f} us per SM")
    print(f"  {live.sum()} CTAs marched a chunk; duration percentiles (us):",
          {q: round(float(np.percentile(d[live], q)), 1) for q in (50, 90, 99, 99.9, 100)})
    grid = np.linspace(0, e.max(), 21)
    act = [int(((s <= g) & (e > g)).sum()) for g in grid]
    print("  active CTAs over time:", " ".join(f"{g:.0f}:{a}" for g, a in zip(grid, act)))
    top = np.argsort(-d)[:12]
    print("  heaviest CTAs (start us, duration us, warp-instance passes, max lane iterations of one march, "
          "max lane iterations, max lane instances):")
    for i in top:
        print("   ", round(float(s[i]), 1), round(float(d[i]), 1), work[i].tolist())
    med = np.argsort(d)[len(d) // 2]
    print("  median CTA:", round(float(d[med]), 1), work[med].tolist(),
          " corr(duration, max lane iterations) =", round(float(np.corrcoef(d[live], work[live][:, 2])[0, 1]), 3),
          " corr(duration, passes) =", round(float(np.corrcoef(d[live], work[live][:, 0])[0, 1]), 3))


if __name__ == "__main__":
    main()
