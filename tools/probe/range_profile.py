import os, sys, time
import numpy as np
ROOT = "/root/repo"
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_util import asset
from paper_2303_04086_b200 import render as R, _native as N
from paper_2303_04086_b200.model import RayRange, orbit_camera
import cProfile, pstats
a = asset("toy_sphere")
cam = orbit_camera(0.8, 0.3, radius=2.0, size=256)
for _ in range(5): R.render_range(a, RayRange(cam, 96, 96, 128, 128))
t=time.perf_counter()
for _ in range(200): R.render_range(a, RayRange(cam, 96, 96, 128, 128))
print("per call us", (time.perf_counter()-t)/200*1e6)
t=time.perf_counter()
for _ in range(200): R._fingerprint(a, 0)
print("fingerprint us", (time.perf_counter()-t)/200*1e6)
t=time.perf_counter()
for _ in range(200): R._instance(a)
print("_instance us", (time.perf_counter()-t)/200*1e6)
t=time.perf_counter()
for _ in range(200): R.check_device_errors()
print("check_device_errors (idle) us", (time.perf_counter()-t)/200*1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(200): R.render_range(a, RayRange(cam, 96, 96, 128, 128))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
