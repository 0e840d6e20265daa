"""The temporally blocked PD kernel (K6) against the one-iteration kernels and
the oracle: same cycles, tile halos at image borders, ragged sizes, every
iteration count (partial launches), fused prologue / epilogue."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def _random_level(h, w, seed):
    rng = np.random.default_rng(seed)
    mask = rng.random((h, w)) > 0.1
    mask[h // 3: h // 3 + 7, :] = False  # a masked band crossing tiles
    img = O.smooth_in_mask(rng.random((h, w)), mask, 1.5)
    T = f32(O.edge_tensor(img, mask, 9.0, 0.85))
    st = O.step_sizes(T, mask, 17.0, 1.2)
    st = O.Steps(f32(st.sigma_p), st.sigma_q, f32(st.tau_u), f32(st.tau_v))
    s = dict(u=f32(rng.normal(size=(h, w))), v=f32(rng.normal(size=(h, w, 2)) * 0.1),
             p=f32(rng.normal(size=(h, w, 2)) * 0.3), q=f32(rng.normal(size=(h, w, 4)) * 0.2),
             u_bar=f32(rng.normal(size=(h, w))), v_bar=f32(rng.normal(size=(h, w, 2)) * 0.1))
    iu = f32(rng.normal(size=(h, w)) * 0.1)
    iu[rng.random((h, w)) < 0.1] = 0.0
    rho0 = f32(rng.normal(size=(h, w)) * 0.05)
    uo = f32(s["u"] + rng.normal(size=(h, w)) * 0.05)
    return mask, T, st, s, iu, rho0, uo


@pytest.mark.parametrize("shape", [(20, 24), (131, 203), (64, 54)])
@pytest.mark.parametrize("iters", [1, 2, 3, 5, 7, 10])
def test_blocked_pd_matches_reference_cycles(shape, iters):
    from paper_1909_07545_b200.solver import SolverParams, SolverState, primal_dual_iterate
    p = SolverParams()
    mask, T, st, s, iu, rho0, uo = _random_level(*shape, seed=iters)
    blk = primal_dual_iterate(SolverState(**s), T, iu, rho0, uo, p, mask, st, blocked=True,
                              iters=iters)
    one = primal_dual_iterate(SolverState(**s), T, iu, rho0, uo, p, mask, st, blocked=False,
                              iters=iters)
    ref = O.PDState(**s)
    for _ in range(iters):
        ref = O.pd_cycle(ref, T, iu, rho0, uo, p, mask, st)
    for k in ("u", "v", "p", "q", "u_bar", "v_bar"):
        a, b, r = getattr(blk, k), getattr(one, k), getattr(ref, k)
        np.testing.assert_allclose(a, b, atol=1e-6, rtol=1e-6, err_msg=f"blocked vs v1 {k}")
        np.testing.assert_allclose(a, r, atol=1e-5, rtol=1e-5, err_msg=f"blocked vs oracle {k}")


def test_blocked_level_solve_matches_one_iteration_kernels():
    from paper_1909_07545_b200.solver import Diagnostics, SolverParams, WarpState, solve_level
    g = load_golden("level_solve")
    h, w = g["mask"].shape
    for prm in (SolverParams(warp_iters=3, pd_iters=4, pyramid_levels=1),
                SolverParams(warp_iters=4, pd_iters=10, pyramid_levels=1),
                SolverParams(warp_iters=2, pd_iters=7, pyramid_levels=1)):
        init = WarpState(u=f32(g["u0"]), w=f32(g["w0"]))
        da, db = Diagnostics(), Diagnostics()
        a, sa = solve_level(g["i0"], g["i1"], g["dirs"], g["tok"], prm, g["mask"], init, da,
                            blocked=True)
        b, sb = solve_level(g["i0"], g["i1"], g["dirs"], g["tok"], prm, g["mask"], init, db,
                            blocked=False)
        np.testing.assert_allclose(a.u, b.u, atol=1e-5)
        np.testing.assert_allclose(a.w, b.w, atol=1e-5)
        np.testing.assert_allclose(sa.v, sb.v, atol=1e-5)
        np.testing.assert_allclose(sa.p, sb.p, atol=1e-5)
        np.testing.assert_allclose(da.max_p_norm, db.max_p_norm, atol=1e-6)
        np.testing.assert_allclose(da.max_q_norm, db.max_q_norm, atol=1e-6)
        np.testing.assert_allclose(da.max_du, db.max_du, atol=1e-6)
        np.testing.assert_allclose(da.mean_abs_du, db.mean_abs_du, atol=1e-6)
