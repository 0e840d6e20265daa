"""Print the reference acceptance numbers (criteria 06-08) for the B200 path."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1909_07545_b200 import evaluate, fields, synth as S
from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
rig = S.default_rig(); sc = S.default_scene()
i0, _, _ = S.render(sc, rig.cam0, supersample=2)
i1, _, _ = S.render(sc, rig.cam1, pose=rig.pose, supersample=2)
gt = S.make_ground_truth(sc, rig)
cal, cal_ok = fields.generate_calibration_field(rig)
for prec in ("fp32", "fp64"):
    for n, du in [(2, 0.2), (5, 0.2), (10, 0.2), (50, 0.2), (50, 0.1), (50, 1.0)]:
        res = solve_pyramid(i0, i1, rig, SolverParams(warp_iters=n, du_max=du), precision=prec)
        corr, ok = fields.compose_with_calibration(res.w, cal, cal_ok)
        rep = evaluate.make_report(corr, gt.correspondence, gt.covisibility & ok & res.mask)
        print(f"{prec} N={n:2d} du_max={du}: tau>1 {rep.pct_bad[1.0]:.2f}%  tau>3 {rep.pct_bad[3.0]:.2f}%"
              f"  tau>5 {rep.pct_bad[5.0]:.2f}%  median {rep.median_error_px:.3f}px  n={rep.valid_count}")
