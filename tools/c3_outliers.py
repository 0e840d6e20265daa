"""Where the fp32 path departs from the fp64 parity path at C3 (N=50): count and location of |du| > 0.1 px."""
import sys, numpy as np
from pathlib import Path
R = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(R)); sys.path.insert(0, str(R / 'tests'))
from test_gpu_configs import _render_pair
from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
from paper_1909_07545_b200 import fields as F
cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5, fov=np.pi, xi=0.9)
rig = StereoRig(cam, cam, RelativePose.from_displacement((0.08, 0.02, 0.03), rotvec=(0.01, 0.03, -0.02)))
prm = SolverParams()
i0, i1 = _render_pair(rig, ss=1)
r32 = solve_pyramid(i0, i1, rig, prm, precision="fp32"); r64 = solve_pyramid(i0, i1, rig, prm, precision="fp64")
e = np.abs(r32.u - r64.u); e[~r64.mask] = 0
ys, xs = np.nonzero(e > 1.0)
print("px > 1:", len(ys), "px > 0.1:", int((e > 0.1).sum()), "of", int(r64.mask.sum()))
for y, x in list(zip(ys, xs))[:20]:
    print(y, x, round(float(e[y, x]), 3), round(float(r64.u[y, x]), 3), round(float(r32.u[y, x]), 3))
m = e > 0.1
if m.any():
    ys, xs = np.nonzero(m)
    print("bbox >0.1:", ys.min(), ys.max(), xs.min(), xs.max())
    # distance from image centre (FOV edge?) and from the epipole (845.5, 595.0)
    r = np.hypot(xs - 511.5, ys - 511.5); de = np.hypot(xs - 845.5, ys - 595.0)
    print("radius from centre: min", r.min().round(1), "median", np.median(r).round(1), "max", r.max().round(1))
    print("dist from epipole: min", de.min().round(1), "median", np.median(de).round(1))
    h = np.histogram(de, bins=[0, 5, 10, 20, 50, 100, 200, 2000])[0]; print("epipole-distance histogram", h)
    h = np.histogram(r, bins=[0, 100, 200, 300, 400, 450, 500, 520, 600])[0]; print("radius histogram", h)
