"""Per-level split of the float64 C3 frame into the warp prologue (sampling +
linearisation) and the primal-dual launches, from the native phase timer
(CUDA events around each warp's phases, direct enqueue, so launch gaps count)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_1909_07545_b200.solver import Solver

rig, prm, desc, ss = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c3")
i0, i1 = bench.load_c3_pair()
eng = Solver(rig, prm, precision="fp64")
eng.i0.copy_(torch.as_tensor(i0, device="cuda")); eng.i1.copy_(torch.as_tensor(i1, device="cuda"))
eng.run(); torch.cuda.synchronize()
for lvl in range(prm.pyramid_levels):
    eng.time_phases(lvl)
    t = eng.time_phases(lvl)
    nw = t["warps"]
    if nw == 0:  # k64_level: the whole level is one launch
        print(f"level {t['w']}x{t['h']}: one whole-level launch (k64_level)")
        continue
    print(f"level {t['w']}x{t['h']}: prologue {t['sample_ms'] * 1e3 / nw:7.1f} us/warp, "
          f"PD {t['pd_ms'] * 1e3 / nw:7.1f} us/warp ({t['pd_launches_per_warp']} launches)")
