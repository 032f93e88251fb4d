"""GPU farm workers on N GPUs (torchrun, NCCL): every rank replays the
reference master's dispatches (tests/golden/dispatch.json), renders its
workers' tasks on its GPU, rank 0 gathers the tiles and composes; checked
against the recorded dispatch log and compose(render_frame) on rank 0.

usage: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/farm_check.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_farm import CASES, run_case  # noqa: E402
from paper_2303_04086_b200 import render as R  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
out = []
for idx, rec in enumerate(CASES):
    logs, frames, scene, cam = run_case(rec, world, rank)
    ok_log = logs == rec["ticks"]
    res = {"case": idx, "dispatch_log_equal": ok_log}
    if rank == 0:
        ref = R.compose(R.render_frame(scene, cam))
        res["frames"] = len(frames)
        res["frames_bitwise_equal"] = all(np.array_equal(f.frame.rgba, ref.rgba) and
                                          np.array_equal(f.frame.depth, ref.depth) for f in frames)
    out.append(res)
if rank == 0:
    print(json.dumps({"world": world, "cases": out,
                      "pass": all(r["dispatch_log_equal"] and r["frames_bitwise_equal"] and r["frames"] for r in out)}))
dist.barrier()
dist.destroy_process_group()
