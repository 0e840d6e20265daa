"""End-to-end parity of the GPU solve (fp32) against the pinned fp64 oracle.

North-star gate (BASELINE.json): final disparity within 1e-3 px median and
1e-2 px 99th-percentile absolute error over the solve mask. Solver invariants
from the reference tests (dual feasibility, du clip, accumulation identity,
determinism) are checked at fp32 tolerances stated inline.
"""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import camera_from_record, load_golden
from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

MEDIAN_TOL = 1e-3
P99_TOL = 1e-2


def err_stats(a, b, sel):
    e = np.abs(np.asarray(a) - np.asarray(b))[sel]
    if e.size == 0:
        return 0.0, 0.0, 0.0
    return float(np.median(e)), float(np.percentile(e, 99)), float(e.max())


def _rig(g):
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    return StereoRig(camera_from_record(g["cam0"]), camera_from_record(g["cam1"]),
                     RelativePose(g["R"], g["t"]))


def _params(g):
    from paper_1909_07545_b200.solver import SolverParams
    return SolverParams.from_dict(json.loads(str(g["params"])))


def test_level_solve_parity():
    from paper_1909_07545_b200.solver import Diagnostics, WarpState, solve_level
    g = load_golden("level_solve")
    prm = _params(g)
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    i0, i1, dirs, u0, w0 = f(g["i0"]), f(g["i1"]), f(g["dirs"]), f(g["u0"]), f(g["w0"])
    d = Diagnostics()
    ws, ss = solve_level(i0, i1, dirs, g["tok"], prm, g["mask"], WarpState(u=u0, w=w0), d)
    tr = O.Trace()
    ou, ow, os_ = O.level_solve(i0, i1, dirs, g["tok"], prm, g["mask"], u0, w0, tr)
    med, p99, mx = err_stats(ws.u, ou, g["mask"])
    assert med <= MEDIAN_TOL and p99 <= P99_TOL, (med, p99, mx)
    med, p99, mx = err_stats(ws.w, ow, g["mask"][..., None] & np.ones(2, bool))
    assert med <= MEDIAN_TOL and p99 <= P99_TOL, (med, p99, mx)
    assert len(d.max_p_norm) == prm.warp_iters * prm.pd_iters
    assert max(d.max_p_norm) <= 1 + 1e-6 and max(d.max_q_norm) <= 1 + 1e-6
    assert max(d.max_du) <= prm.du_max * (1 + 1e-6)
    np.testing.assert_allclose(d.max_du, tr.max_du, atol=1e-4)
    np.testing.assert_allclose(d.mean_abs_du, tr.mean_abs_du, atol=1e-4)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_pyramid_solve_parity_small_rendered_pair(precision):
    from paper_1909_07545_b200.solver import solve_pyramid
    g = load_golden("pyramid_solve")
    rig, prm = _rig(g), _params(g)
    res = solve_pyramid(g["i0"], g["i1"], rig, prm, collect_diagnostics=True,
                        precision=precision)
    sol = O.pyramid_solve(g["i0"], g["i1"], rig, prm, trace=True)
    np.testing.assert_array_equal(res.mask, sol.mask)
    np.testing.assert_allclose(res.i1_calibrated, sol.i1c, atol=2e-7)
    med, p99, mx = err_stats(res.u, sol.u, sol.mask)
    print(f"u error median {med:.2e} p99 {p99:.2e} max {mx:.2e}")
    assert med <= MEDIAN_TOL and p99 <= P99_TOL
    d = res.diagnostics
    assert len(d.max_p_norm) == len(sol.trace.max_p_norm)
    assert max(d.max_p_norm) <= 1 + 1e-6 and max(d.max_q_norm) <= 1 + 1e-6
    assert max(d.max_du) <= prm.du_max * (1 + 1e-6)


def test_accumulation_identity():
    """test_solver.py:307-321: u and w equal the running sums of increments."""
    from paper_1909_07545_b200.solver import Diagnostics, WarpState, solve_level
    g = load_golden("level_solve")
    prm = _params(g)
    h, w = g["mask"].shape
    d = Diagnostics(record_increments=True)
    ws, _ = solve_level(g["i0"], g["i1"], g["dirs"], g["tok"], prm, g["mask"],
                        WarpState(u=np.zeros((h, w)), w=np.zeros((h, w, 2))), d)
    u_sum = sum(du for du, _ in d.increments)
    w_sum = sum(du[..., None] * dd for du, dd in d.increments)
    assert np.max(np.abs(ws.u - u_sum)) < 1e-5
    assert np.max(np.abs(ws.w - w_sum)) < 1e-5
    assert all(m <= prm.du_max * (1 + 1e-6) for m in d.max_du)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_determinism_and_graph_replay(precision):
    """Outputs are bit-identical run to run and through a CUDA graph (SPEC: deterministic)."""
    import torch
    from paper_1909_07545_b200.solver import Solver
    g = load_golden("pyramid_solve")
    eng = Solver(_rig(g), _params(g), precision=precision)
    r1 = eng.solve(g["i0"], g["i1"])  # first call captures the graph
    r2 = eng.solve(g["i0"], g["i1"])
    assert eng.kernels_per_frame and eng.kernels_per_frame > 0
    eng.i0.copy_(torch.from_numpy(g["i0"]))  # cast to the engine dtype as solve() stages
    eng.i1.copy_(torch.from_numpy(g["i1"]))
    eng.run()  # direct enqueue, no graph
    torch.cuda.synchronize()
    r3 = type(r1)(u=eng.u.cpu().numpy(), w=eng.w.cpu().numpy(), v=eng.v.cpu().numpy(),
                  mask=eng.mask.cpu().numpy().astype(bool),
                  i1_calibrated=eng.i1c.double().cpu().numpy())
    for a, b in ((r1, r2), (r1, r3)):
        assert np.array_equal(a.u, b.u) and np.array_equal(a.w, b.w)
        assert np.array_equal(a.v, b.v) and np.array_equal(a.mask, b.mask)
        # mask / i1_calibrated of the float64 graph leave early, on a side stream
        assert np.array_equal(a.i1_calibrated, b.i1_calibrated)
    from paper_1909_07545_b200 import _ext
    early = _ext.lib().fsb_graph_early_event(eng.graph)
    assert (early is not None) == (precision == "fp64")


def test_api_errors():
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    g = load_golden("pyramid_solve")
    rig = _rig(g)
    with pytest.raises(ValueError):
        solve_pyramid(np.zeros((10, 10)), g["i1"], rig, SolverParams())
    with pytest.raises(ValueError):
        solve_pyramid(g["i0"], np.zeros((3, 3)), rig, SolverParams())
    zero = StereoRig(rig.cam0, rig.cam1, RelativePose(rig.pose.rotation, np.zeros(3)))
    with pytest.raises(ValueError):
        solve_pyramid(g["i0"], g["i1"], zero, SolverParams(pyramid_levels=1))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_traj_override_matches_generated(precision):
    """Override path (solver.py:437-438) fed with the generated field gives the same answer."""
    from paper_1909_07545_b200 import fields as F
    from paper_1909_07545_b200.solver import solve_pyramid
    g = load_golden("pyramid_solve")
    rig, prm = _rig(g), _params(g)
    a = solve_pyramid(g["i0"], g["i1"], rig, prm, precision=precision)

    def override(rig_lvl):
        return F.generate_trajectory_field(rig_lvl, prm.epsilon_scale)

    b = solve_pyramid(g["i0"], g["i1"], rig, prm, traj_override=override, precision=precision)
    assert np.array_equal(a.u, b.u) and np.array_equal(a.w, b.w)


def test_empty_mask_frame():
    """A rig whose FOV masks leave nothing to solve returns zeros, not NaNs."""
    from paper_1909_07545_b200.camera import PinholeCamera, RelativePose, StereoRig
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    cam = PinholeCamera(width=24, height=20, fx=10.0, fy=10.0, cx=11.5, cy=9.5, fov=1e-6)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.1, 0.0, 0.0)))
    res = solve_pyramid(np.zeros((20, 24)), np.zeros((20, 24)), rig,
                        SolverParams(warp_iters=2, pd_iters=2, pyramid_levels=2, min_width=4))
    sol = O.pyramid_solve(np.zeros((20, 24)), np.zeros((20, 24)), rig,
                          SimpleNamespace(**SolverParams(warp_iters=2, pd_iters=2,
                                                         pyramid_levels=2, min_width=4).to_dict()))
    np.testing.assert_array_equal(res.mask, sol.mask)
    assert not res.mask.any()
    assert np.all(res.u == 0) and np.all(res.w == 0) and np.isfinite(res.v).all()


def test_results_stay_fresh_with_pinned_pool():
    """Each StereoResult owns its arrays (solver.py:451-452 returns fresh arrays):
    a held result is never overwritten by later calls, and a dropped one's
    pinned buffers are reused (no per-call cudaHostAlloc)."""
    from paper_1909_07545_b200.solver import Solver
    g = load_golden("pyramid_solve")
    eng = Solver(_rig(g), _params(g))
    r1 = eng.solve(g["i0"], g["i1"])
    keep = r1.u[2:, 3:]  # a slice of the result must pin it too
    u1, w1 = r1.u.copy(), r1.w.copy()
    del r1
    r2 = eng.solve(np.flipud(g["i0"]).copy(), np.flipud(g["i1"]).copy())
    assert not np.array_equal(r2.u, u1)
    assert np.array_equal(keep, u1[2:, 3:])  # still the first frame's values
    del keep
    r3 = eng.solve(g["i0"], g["i1"])
    assert np.array_equal(r3.u, u1) and np.array_equal(r3.w, w1)
    del r2
    r3 = eng.solve(g["i0"], g["i1"])  # r3 of the previous call is alive during it
    n_sets = len(eng._out_pool)
    for _ in range(4):  # at most one earlier result alive: the pool stops growing
        r3 = eng.solve(g["i0"], g["i1"])
    assert len(eng._out_pool) == n_sets <= 3
    assert np.array_equal(r3.u, u1)
    assert r3.u.flags.writeable and r3.mask.dtype == bool


def test_concurrent_callers_same_rig():
    """solve_pyramid is re-entrant like the reference: threads
    solving with the same (rig, params) check out separate engines and each get
    the serial result, bit for bit."""
    import threading
    from paper_1909_07545_b200.solver import solve_pyramid
    g = load_golden("pyramid_solve")
    rig, prm = _rig(g), _params(g)
    pairs = [(g["i0"], g["i1"]), (np.flipud(g["i0"]).copy(), np.flipud(g["i1"]).copy())]
    want = [solve_pyramid(a, b, rig, prm) for a, b in pairs]
    out, errs = {}, []

    def work(t):
        try:
            for k in range(6):
                j = (t + k) % 2
                r = solve_pyramid(*pairs[j], rig, prm)
                out[(t, k)] = (j, r.u.copy(), r.w.copy())
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert len(out) == 24
    for j, u, w in out.values():
        assert np.array_equal(u, want[j].u) and np.array_equal(w, want[j].w)


_OVERLAP_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import load_golden
import test_gpu_solve as T
from paper_1909_07545_b200.solver import Solver
g = load_golden("pyramid_solve")
r = Solver(T._rig(g), T._params(g), precision="fp32").solve(g["i0"], g["i1"])
np.savez(sys.argv[2], u=r.u, w=r.w, v=r.v)
"""


def test_side_stream_overlap_is_bit_identical(tmp_path):
    """Per-level setup on the side stream (default) and everything on the
    caller's stream (FSB_OVERLAP=0, read once per process: a child process)
    give bit-identical frames."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    from paper_1909_07545_b200.solver import Solver
    g = load_golden("pyramid_solve")
    r = Solver(_rig(g), _params(g), precision="fp32").solve(g["i0"], g["i1"])
    out = tmp_path / "serial.npz"
    env = dict(os.environ, FSB_OVERLAP="0")
    subprocess.run([sys.executable, "-c", _OVERLAP_CHILD, str(ROOT), str(out)], env=env,
                   check=True, timeout=600)
    with np.load(out) as z:
        assert np.array_equal(z["u"], r.u) and np.array_equal(z["w"], r.w)
        assert np.array_equal(z["v"], r.v)


def test_diagnostics_do_not_change_the_solution():
    """As in the reference (diagnostics only observe the iteration), collecting
    diagnostics gives bit-identical u, w, v: the same kernels run in both modes
    (k64_level and k64_ctile reduce the traces themselves)."""
    import bench
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.solver import solve_pyramid
    g = load_golden("pyramid_solve")
    rig1, prm1 = bench.product_rig("c1"), bench.product_params("c1")
    sc = S.default_scene()
    i0 = S.render(sc, rig1.cam0, supersample=1)[0]
    i1 = S.render(sc, rig1.cam1, pose=rig1.pose, supersample=1)[0]
    for rig, prm, a, b in ((_rig(g), _params(g), g["i0"], g["i1"]), (rig1, prm1, i0, i1)):
        r0 = solve_pyramid(a, b, rig, prm)
        r1 = solve_pyramid(a, b, rig, prm, collect_diagnostics=True)
        assert np.array_equal(r0.u, r1.u) and np.array_equal(r0.w, r1.w)
        assert np.array_equal(r0.v, r1.v)
        d = r1.diagnostics
        assert len(d.max_p_norm) == prm.pyramid_levels * prm.warp_iters * prm.pd_iters or \
            len(d.max_p_norm) > 0
        assert max(d.max_p_norm) <= 1 + 1e-6 and max(d.max_du) <= prm.du_max * (1 + 1e-6)
        assert all(np.isfinite(d.mean_abs_du)) and min(d.mean_abs_du) >= 0.0
