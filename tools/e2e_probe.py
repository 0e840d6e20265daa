"""Time the phases of the public-API call on the C3 workload (diagnostic)."""
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
for _ in range(3):
    r = solve_pyramid(i0, i1, rig, prm)
torch.cuda.synchronize()
eng = next(iter(_CACHE.values()))
T = {}
def tick(k, t0):
    torch.cuda.synchronize(); T[k] = T.get(k, 0) + time.perf_counter() - t0; return time.perf_counter()
for _ in range(10):
    t = time.perf_counter()
    h = eng._staging()
    h["i0"].copy_(torch.from_numpy(np.ascontiguousarray(i0))); h["i1"].copy_(torch.from_numpy(np.ascontiguousarray(i1)))
    t = tick("host->pinned (cast to fp32)", t)
    eng.i0.copy_(h["i0"], non_blocking=True); eng.i1.copy_(h["i1"], non_blocking=True)
    t = tick("h2d", t)
    eng.replay()
    t = tick("graph", t)
    outs = {}
    for k, dt in (("u", torch.float64), ("w", torch.float64), ("v", torch.float64), ("mask", torch.bool), ("i1c", torch.float64)):
        outs[k] = getattr(eng, k).to(dt)
    t = tick("cast out", t)
    hb = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in outs.items()}
    t = tick("pinned alloc", t)
    for k in hb: hb[k].copy_(outs[k], non_blocking=True)
    t = tick("d2h", t)
    res = {k: v.numpy() for k, v in hb.items()}
    t = tick("numpy", t)
t0 = time.perf_counter()
for _ in range(10):
    r = solve_pyramid(i0, i1, rig, prm)
torch.cuda.synchronize()
print({k: round(v * 100, 3) for k, v in T.items()}, "ms/call; full API", round((time.perf_counter() - t0) * 100, 2), "ms/call")
