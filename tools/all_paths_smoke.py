"""Small solves through every kernel family (memory-safety smoke):
TMA path, cluster path, pair fallback,
fp64 blocked path, depth, evaluation."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1909_07545_b200 import evaluate, fields, synth as S
from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
for (w, h) in [(256, 192), (258, 130)]:  # TMA path + cluster; w % 4 != 0: pair fallback
    cam = UnifiedCamera(width=w, height=h, fx=110.0, fy=110.0, cx=(w - 1) / 2, cy=(h - 1) / 2,
                        fov=np.pi, xi=0.9)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.1, 0.01, 0), rotvec=(0, 0.02, 0)))
    sc = S.default_scene()
    i0, _, _ = S.render(sc, rig.cam0)
    i1, _, _ = S.render(sc, rig.cam1, pose=rig.pose)
    prm = SolverParams(warp_iters=2, pd_iters=10, pyramid_levels=3, min_width=30)
    r = solve_pyramid(i0, i1, rig, prm, collect_diagnostics=True)
    r64 = solve_pyramid(i0, i1, rig, prm, precision="fp64", collect_diagnostics=True)
    cal, ok = fields.generate_calibration_field(rig)
    corr, cok = fields.compose_with_calibration(r.w, cal, ok)
    d, dok = evaluate.depth_from_correspondence(rig, corr, cok & r.mask)
    gt = S.make_ground_truth(sc, rig)
    rep = evaluate.make_report(corr, gt.correspondence, gt.covisibility & cok & r.mask)
    print(w, h, float(np.abs(r.u - r64.u)[r.mask].max()), rep.valid_count)
print("ok")
