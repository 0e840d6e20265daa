"""Fraction of C3 finest-level mask pixels whose 4x4 bicubic stencil is fully valid
(mask and traj_ok): the share of samples on the packed fast path."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
from paper_1909_07545_b200 import fields as F, camera as Cm, solver as Sv
rig, prm, desc, ss = bench.workload("c3")
m0 = Cm.fov_mask(rig.cam0)
i1c_ok = F.calibrate_second_image(np.zeros((rig.cam1.height, rig.cam1.width)), rig)[1]
mask = m0 & i1c_ok
dirs, tok = F.generate_trajectory_field(F.translation_only_rig(rig), prm.epsilon_scale)
def full(m):
    h, w = m.shape
    f = np.zeros_like(m)
    ok = np.ones((h - 3, w - 3), bool)
    for a in range(4):
        for b in range(4):
            ok &= m[a:h - 3 + a, b:w - 3 + b]
    f[1:h - 2, 1:w - 2] = ok
    return f
fm, ft = full(mask), full(tok)
print("mask frac", mask.mean(), "traj_ok frac in mask", tok[mask].mean())
print("full16 mask", fm[mask].mean(), "full16 traj", ft[mask].mean(), "both", (fm & ft)[mask].mean())
