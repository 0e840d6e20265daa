"""Per-call wall time of the public API (solve_pyramid, float64 host arrays) on
the C3 pair: 60 calls with the previous result alive (bench.py's e2e pattern),
printing every call so outliers can be located."""
import gc, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
from paper_1909_07545_b200.solver import solve_pyramid
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
rig, prm = bench.product_rig("c3"), bench.product_params("c3")
h0, h1 = bench.load_c3_pair()
x0, x1 = h0.astype(np.float64), h1.astype(np.float64)
for _ in range(5):
    r = solve_pyramid(x0, x1, rig, prm, precision=prec)
ts = []
for _ in range(60):
    t = time.perf_counter(); r = solve_pyramid(x0, x1, rig, prm, precision=prec)
    ts.append(round((time.perf_counter() - t) * 1e3, 2))
print(prec, "per-call ms:", ts)
print("median", np.median(ts), "max", max(ts), "at", int(np.argmax(ts)), "gc counts", gc.get_count())
