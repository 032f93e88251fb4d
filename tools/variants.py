"""Build A/B variants of libnolf_b200.so (extra -D flags) next to the in-tree
library: paper_2303_04086_b200/variants/libnolf_<name>.so (git-ignored; they
travel to the GPU box with the snapshot).  Select one with NOLF_LIB=<path>.

usage: python tools/variants.py name=-DFLAG[,-DFLAG2] [name2=...]
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_04086_b200 import build as B  # noqa: E402

OUT = os.path.join(ROOT, "paper_2303_04086_b200", "variants")


def build(name, flags):
    os.makedirs(OUT, exist_ok=True)
    so = os.path.join(OUT, f"libnolf_{name}.so")
    cmd = ["nvcc", *B.NVCC_FLAGS, *flags, os.path.join(B.HERE, "csrc", "nolf_capi.cu"), "-o", so]
    subprocess.run(cmd, check=True)
    return so


if __name__ == "__main__":
    jobs = []
    for a in sys.argv[1:]:
        name, _, fl = a.partition("=")
        jobs.append((name, [f for f in fl.split(",") if f]))
    with ThreadPoolExecutor(len(jobs)) as ex:
        for so in ex.map(lambda j: build(*j), jobs):
            print(so)
