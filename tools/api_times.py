"""Per-call wall time of the public API (solve_pyramid, float64 host arrays) on C3,
with the previous result alive and with results dropped (pinned output pool reuse)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
from paper_1909_07545_b200 import synth as S
from paper_1909_07545_b200.solver import solve_pyramid, _CACHE
rig, prm, desc, ss = bench.workload("c3")
sc = S.default_scene()
i0 = S.render_device(sc, rig.cam0, supersample=ss)[0].cpu().numpy().astype(np.float64)
i1 = S.render_device(sc, rig.cam1, pose=rig.pose, supersample=ss)[0].cpu().numpy().astype(np.float64)
for _ in range(5):
    r = solve_pyramid(i0, i1, rig, prm)
ts = []
for _ in range(20):
    t = time.perf_counter(); r = solve_pyramid(i0, i1, rig, prm); ts.append((time.perf_counter() - t) * 1e3)
print("per-call ms:", [round(x, 2) for x in ts])
eng = next(iter(_CACHE.values())); print("pool sets:", len(eng._out_pool))
del r
ts = []
for _ in range(20):
    t = time.perf_counter(); solve_pyramid(i0, i1, rig, prm); ts.append((time.perf_counter() - t) * 1e3)
print("results dropped at once:", [round(x, 2) for x in ts])
