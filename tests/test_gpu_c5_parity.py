"""C5 geometry against the oracle (BASELINE config 5): 2048^2
unified (xi=0.9) pair, 7 levels (min_width 32), K=10, with the reference's own
TGV regulariser (the config's Huber-TV has no reference) at a
reduced warp count N=2 so the NumPy oracle finishes in about two minutes on the
GPU box's host. Both GPU paths: north-star gate median <= 1e-3 px, p99 <= 1e-2
px on the solve mask; the default float64 path also within 1e-6 px max."""

import numpy as np
import pytest

from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu


def test_c5_tgv_parity_reduced_warps():
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    cam = UnifiedCamera(width=2048, height=2048, fx=910.0, fy=910.0, cx=1023.5, cy=1023.5,
                        fov=np.pi, xi=0.9)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.1, 0, 0),
                                                             rotvec=(0, 0.02, 0.005)))
    sc = S.default_scene()
    i0 = S.render_device(sc, rig.cam0)[0].double().cpu().numpy()
    i1 = S.render_device(sc, rig.cam1, pose=rig.pose)[0].double().cpu().numpy()
    prm = SolverParams(warp_iters=2, pd_iters=10, pyramid_levels=7, min_width=32,
                       regularizer="tgv")
    sol = O.pyramid_solve(i0, i1, rig, prm)
    assert sol.mask.shape == (2048, 2048)
    for precision in ("fp64", "fp32"):
        res = solve_pyramid(i0, i1, rig, prm, precision=precision)
        np.testing.assert_array_equal(res.mask, sol.mask)
        e = np.abs(res.u - sol.u)[sol.mask]
        med, p99, mx = float(np.median(e)), float(np.percentile(e, 99)), float(e.max())
        print(f"C5 TGV N=2 [{precision}] vs oracle: median {med:.3e} p99 {p99:.3e} "
              f"max {mx:.3e}; u range {sol.u[sol.mask].min():.2f}..{sol.u[sol.mask].max():.2f}")
        assert med <= 1e-3 and p99 <= 1e-2, (precision, med, p99)
        if precision == "fp64":
            assert mx <= 1e-6, mx
