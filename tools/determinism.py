"""Run-to-run determinism of the float64 C3 frame: N graph replays (default 20)
must give bit-identical u, w, v (a race in an exchange or a missing barrier
shows up as a differing replay)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_1909_07545_b200.solver import Solver

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rig, prm = bench.product_rig("c3"), bench.product_params("c3")
i0, i1 = bench.load_c3_pair()
eng = Solver(rig, prm, precision="fp64")
eng.i0.copy_(torch.as_tensor(i0, device="cuda")); eng.i1.copy_(torch.as_tensor(i1, device="cuda"))
eng.capture()
ref = None
bad = 0
for k in range(n):
    eng.replay()
    torch.cuda.synchronize()
    out = [t.cpu().numpy().copy() for t in (eng.u, eng.w, eng.v)]
    if ref is None:
        ref = out
    elif not all(np.array_equal(a, b) for a, b in zip(ref, out)):
        bad += 1
print(f"{n} C3 float64 replays: {n - bad} bit-identical to the first, {bad} differ")
sys.exit(1 if bad else 0)
