"""North-star parity gate at the headline config, in suite: C3 at full size.

BASELINE config 3: the 1024^2 unified (xi=0.9) pair under the
6-DoF pose, reference defaults N=50 warps x K=10, 5 levels. Inputs and the
expected answer are the REFERENCE's own: `synth.render(..., supersample=2)`
rounded to float32 (tests/golden/c3_pair.npz) and `fisheyestereo.solve_pyramid`
run on exactly those values (tests/golden/c3_solution.npz), both made by
oracle/make_c3_fixture.py in the build container (457 s of reference time).

Gate (north star): disparity within 1e-3 px median and 1e-2 px p99 absolute
error on the reference's solve mask, mask identical. The default float64 path
must pass; the float32 path is measured and its numbers printed (it holds the
median gate but not the p99 gate at N=50)."""

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

MEDIAN_TOL, P99_TOL = 1e-3, 1e-2


def _c3():
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import SolverParams
    cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5,
                        fov=np.pi, xi=0.9)
    pose = RelativePose.from_displacement((0.08, 0.02, 0.03), rotvec=(0.01, 0.03, -0.02))
    return StereoRig(cam, cam, pose), SolverParams()


@pytest.fixture(scope="module")
def c3():
    with np.load(ROOT / "tests" / "golden" / "c3_pair.npz") as z:
        i0, i1 = z["i0"].astype(np.float64), z["i1"].astype(np.float64)
    with np.load(ROOT / "tests" / "golden" / "c3_solution.npz") as z:
        ref = {k: z[k] for k in z.files}
    return i0, i1, ref


def _stats(u, ref):
    e = np.abs(np.asarray(u, np.float64) - ref["u"].astype(np.float64))[ref["mask"]]
    return float(np.median(e)), float(np.percentile(e, 99)), float(e.max()), e


def test_c3_default_fp64_path_matches_reference(c3):
    from paper_1909_07545_b200.solver import solve_pyramid
    i0, i1, ref = c3
    rig, prm = _c3()
    res = solve_pyramid(i0, i1, rig, prm)  # the drop-in default: float64
    np.testing.assert_array_equal(res.mask, ref["mask"])
    med, p99, mx, e = _stats(res.u, ref)
    print(f"C3 fp64 vs reference: u err median {med:.3e} p99 {p99:.3e} max {mx:.3e}; "
          f"> 0.1 px {int((e > 0.1).sum())} of {e.size}")
    assert med <= MEDIAN_TOL and p99 <= P99_TOL, (med, p99, mx)
    # the calibrated second image (reference float64, stored rounded to float32)
    assert np.max(np.abs(res.i1_calibrated - ref["i1c"].astype(np.float64))) <= 1e-6
    assert np.isfinite(res.u).all() and np.isfinite(res.w).all()


def test_c3_fp32_path_median_gate_and_recorded_p99(c3):
    """The float32 path: median gate asserted; p99 printed (measured ~3e-2 px
    in round 1: the N=50 warp loop amplifies fp32 rounding)."""
    from paper_1909_07545_b200.solver import solve_pyramid
    i0, i1, ref = c3
    rig, prm = _c3()
    res = solve_pyramid(i0, i1, rig, prm, precision="fp32")
    np.testing.assert_array_equal(res.mask, ref["mask"])
    med, p99, mx, e = _stats(res.u, ref)
    print(f"C3 fp32 vs reference: u err median {med:.3e} p99 {p99:.3e} max {mx:.3e}; "
          f"> 0.1 px {int((e > 0.1).sum())} of {e.size} (p99 gate {P99_TOL} not asserted)")
    assert med <= MEDIAN_TOL, med
