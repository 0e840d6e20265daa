"""Per-level cost of the C3 frame from graph-replayed solves with 1..5 pyramid
levels: T(L) - T(L-1) is the cost of the level added at the coarse end."""
import sys
from dataclasses import replace
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_1909_07545_b200 import synth as S
from paper_1909_07545_b200.solver import Solver

rig, prm, desc, ss = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c3")
import os
if os.environ.get("PD_ITERS"):  # cost model: per-warp fixed part vs per-cycle part
    prm = replace(prm, pd_iters=int(os.environ["PD_ITERS"]))
sc = S.default_scene()
i0 = S.render_device(sc, rig.cam0, supersample=ss)[0]
i1 = S.render_device(sc, rig.cam1, pose=rig.pose, supersample=ss)[0]
T = {}
import os
prec = os.environ.get("PREC", "fp32")
for L in range(1, prm.pyramid_levels + 1):
    p = replace(prm, pyramid_levels=L)
    eng = Solver(rig, p, precision=prec)
    eng.i0.copy_(i0); eng.i1.copy_(i1)
    if os.environ.get("NOGRAPH"):
        eng.replay = eng.run
    else:
        eng.capture()
    for _ in range(3):
        eng.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        eng.replay()
    e1.record()
    torch.cuda.synchronize()
    T[L] = e0.elapsed_time(e1) / 10
    del eng
shapes = Solver.__init__.__globals__["pyramid_shapes"](rig.cam0.height, rig.cam0.width, prm.pyramid_levels, prm.pyramid_scale, prm.min_width)
prev = 0.0
for L in range(1, prm.pyramid_levels + 1):
    h, w = shapes[L - 1]
    print(f"levels={L} total {T[L]:7.3f} ms; level {w}x{h}: {T[L] - prev:7.3f} ms ({(T[L]-prev)/prm.warp_iters*1e3:6.1f} us/warp)")
    prev = T[L]
