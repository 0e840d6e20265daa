"""Phases of one public-API call on the C3 pair (diagnostic): host -> pinned
staging, H2D, graph replay, D2H of the five outputs; then the full API."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
from paper_1909_07545_b200.solver import solve_pyramid, _CACHE

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
rig, prm = bench.product_rig("c3"), bench.product_params("c3")
h0, h1 = bench.load_c3_pair()
i0, i1 = h0.astype(np.float64), h1.astype(np.float64)
for _ in range(3):
    r = solve_pyramid(i0, i1, rig, prm, precision=prec)
torch.cuda.synchronize()
eng = next(iter(_CACHE.values()))[0]
T = {}
def tick(k, t0):
    torch.cuda.synchronize(); T[k] = T.get(k, 0) + time.perf_counter() - t0; return time.perf_counter()
hb = {k: torch.empty(tuple(getattr(eng, k).shape), dtype=dt, pin_memory=True) for k, dt in eng._OUT}
for _ in range(10):
    t = time.perf_counter()
    h = eng._staging()
    h["i0"].copy_(torch.from_numpy(i0)); h["i1"].copy_(torch.from_numpy(i1))
    t = tick("host->pinned", t)
    eng.i0.copy_(h["i0"], non_blocking=True); eng.i1.copy_(h["i1"], non_blocking=True)
    t = tick("h2d", t)
    eng.replay()
    t = tick("graph", t)
    for k, dt in eng._OUT:
        src = getattr(eng, k)
        src = src.view(torch.bool) if dt == torch.bool else src.to(dt)
        hb[k].copy_(src, non_blocking=True)
    t = tick("d2h", t)
t0 = time.perf_counter()
for _ in range(10):
    r = solve_pyramid(i0, i1, rig, prm, precision=prec)
torch.cuda.synchronize()
full = (time.perf_counter() - t0) * 100
t0 = time.perf_counter()
for _ in range(10):
    r = eng.solve(i0, i1)
torch.cuda.synchronize()
print(prec, {k: round(v * 100, 3) for k, v in T.items()}, "ms/call; full API", round(full, 2),
      "ms/call; eng.solve", round((time.perf_counter() - t0) * 100, 2), "ms/call")

# where does the API call spend its time beyond eng.solve?
import paper_1909_07545_b200.solver as SV
made = []
orig_init = SV.Solver.__init__
def counting_init(self, *a, **k):
    made.append(1)
    return orig_init(self, *a, **k)
SV.Solver.__init__ = counting_init
pools = []
ts = []
for _ in range(10):
    t = time.perf_counter()
    r = solve_pyramid(i0, i1, rig, prm, precision=prec)
    ts.append(round((time.perf_counter() - t) * 1e3, 2))
    pools.append([len(e._out_pool) for v in SV._CACHE.values() for e in v])
print("per-call ms", ts, "engines built", len(made), "pool sizes", pools[-1], "cache keys", len(SV._CACHE))
