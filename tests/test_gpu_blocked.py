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
        # packed FFMA2 cycles vs the scalar one-cycle kernels: fp32 round-off of
        # up to 40 cycles on unit-ball duals (observed <= 1.2e-5)
        np.testing.assert_allclose(sa.p, sb.p, atol=5e-5)
        np.testing.assert_allclose(da.max_p_norm, db.max_p_norm, atol=1e-6)
        np.testing.assert_allclose(da.max_q_norm, db.max_q_norm, atol=1e-6)
        np.testing.assert_allclose(da.max_du, db.max_du, atol=1e-6)
        np.testing.assert_allclose(da.mean_abs_du, db.mean_abs_du, atol=1e-6)


def _random_pair(h, w, seed):
    rng = np.random.default_rng(seed)
    mask = np.ones((h, w), bool)
    yy, xx = np.mgrid[0:h, 0:w]
    mask &= (xx - w / 2) ** 2 / (0.48 * w) ** 2 + (yy - h / 2) ** 2 / (0.48 * h) ** 2 < 1.0
    base = O.smooth_in_mask(rng.random((h, w + 8)), np.ones((h, w + 8), bool), 1.2)
    i0 = f32(base[:, 4:w + 4])
    i1 = f32(base[:, 2:w + 2] + 0.01 * rng.normal(size=(h, w)))  # ~2 px shift
    ang = 0.2 * np.sin(yy / max(h, 1) * 3.0)
    dirs = f32(np.stack([np.cos(ang), np.sin(ang)], -1))
    tok = mask.copy()
    tok[:, :2] = False
    return i0, i1, dirs, tok, mask


# Level shapes on the whole-level cluster path (<= 16 rows per CTA, <= 16 warps),
# including ragged bands and widths that are not multiples of 64, and on the
# TMA path with its mask-tile work list (96x160, 200x256, 300x212: the elliptic
# mask leaves whole tiles outside it, which the work list skips).
@pytest.mark.parametrize("shape", [(64, 64), (128, 128), (37, 50), (17, 130), (250, 40),
                                   (96, 160), (200, 256), (300, 212)])
def test_level_solve_paths_match_v1_and_oracle(shape):
    from paper_1909_07545_b200.solver import Diagnostics, SolverParams, WarpState, solve_level
    h, w = shape
    i0, i1, dirs, tok, mask = _random_pair(h, w, seed=h * w)
    prm = SolverParams(warp_iters=3, pd_iters=6, pyramid_levels=1)
    rng = np.random.default_rng(1)
    init = WarpState(u=f32(rng.normal(size=(h, w)) * 0.3), w=f32(rng.normal(size=(h, w, 2)) * 0.3))
    da, db = Diagnostics(), Diagnostics()
    a, sa = solve_level(i0, i1, dirs, tok, prm, mask, init, da, blocked=True)
    b, sb = solve_level(i0, i1, dirs, tok, prm, mask, init, db, blocked=False)
    for k in ("u", "w"):
        np.testing.assert_allclose(getattr(a, k), getattr(b, k), atol=1e-5, err_msg=k)
    for k in ("u", "v", "p", "q", "u_bar", "v_bar"):
        np.testing.assert_allclose(getattr(sa, k), getattr(sb, k), atol=1e-5, err_msg=k)
    for k in ("max_p_norm", "max_q_norm", "max_du", "mean_abs_du"):
        np.testing.assert_allclose(getattr(da, k), getattr(db, k), atol=1e-6, err_msg=k)
    ref = O.level_solve(i0, i1, dirs, tok, prm, mask, init.u, init.w)
    err = np.abs(a.u - ref[0])[mask]
    assert np.median(err) < 1e-5 and np.percentile(err, 99) < 1e-3, (np.median(err), err.max())
