"""C3 at full size against the pinned CPU oracle (test-infrastructure use only):
the fp32 production path and the fp64 parity path vs oracle/fs_oracle.pyramid_solve
(~8 min of single-core NumPy). Writes the error statistics; the `-m gpu` suite keeps
the fast proxy (fp32 vs fp64 path, tests/test_gpu_configs.py)."""
import sys, time
from pathlib import Path
R = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(R)); sys.path.insert(0, str(R / "tests"))
import numpy as np
from test_gpu_configs import _render_pair
from oracle import fs_oracle as O
from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
from paper_1909_07545_b200.solver import SolverParams, solve_pyramid

cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5,
                    fov=np.pi, xi=0.9)
rig = StereoRig(cam, cam, RelativePose.from_displacement((0.08, 0.02, 0.03),
                                                         rotvec=(0.01, 0.03, -0.02)))
prm = SolverParams()
i0, i1 = _render_pair(rig, ss=1)
r32 = solve_pyramid(i0, i1, rig, prm, precision="fp32")
r64 = solve_pyramid(i0, i1, rig, prm, precision="fp64")
t0 = time.time()
sol = O.pyramid_solve(i0, i1, rig, prm)
print(f"C3 1024^2 unified 6-DoF, N=50 K=10, 5 levels; oracle {time.time() - t0:.0f} s on 1 core")
print("mask identical (fp32, fp64):", bool(np.array_equal(r32.mask, sol.mask)),
      bool(np.array_equal(r64.mask, sol.mask)), "; mask px", int(sol.mask.sum()))
for name, r in (("fp32 path", r32), ("fp64 path", r64)):
    e = np.abs(r.u - sol.u)[sol.mask]
    ew = np.linalg.norm(r.w - sol.w, axis=-1)[sol.mask]
    print(f"{name}: u err median {np.median(e):.3e} p99 {np.percentile(e, 99):.3e} "
          f"max {e.max():.3e}; > 0.1 px {int((e > 0.1).sum())}, > 1 px {int((e > 1).sum())}; "
          f"|w err| median {np.median(ew):.3e} p99 {np.percentile(ew, 99):.3e}")
    print(f"  i1_calibrated max err {np.max(np.abs(r.i1_calibrated - sol.i1c)):.3e}")
