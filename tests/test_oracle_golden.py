"""Pin the CPU oracle (oracle/fs_oracle.py) to the reference's own outputs.

The fixtures in tests/golden were produced by running the reference
implementation (oracle/make_golden.py). The oracle must reproduce them to the
last bit for every stage (tolerance 0 except where noted) — this is what makes
it a trustworthy checker for the GPU path.
"""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import camera_from_record, load_golden
from oracle import fs_oracle as O

CAMS = ["pinhole", "unified", "equidistant", "kb"]


def same(a, b, tol=0.0):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    if a.dtype == bool or tol == 0.0:
        np.testing.assert_array_equal(a, b)
    else:
        np.testing.assert_allclose(a, b, rtol=tol, atol=tol)


@pytest.mark.parametrize("name", CAMS)
def test_lens_models(name):
    g = load_golden(f"camera_{name}")
    cam = camera_from_record(g["cam"])
    same(O.fov_mask(cam), g["mask"])
    rx, ry, rz, ok = O.unproject(cam, g["pix"][:, 0], g["pix"][:, 1])
    same(ok, g["rays_ok"])
    same(np.stack([rx, ry, rz], -1), g["rays"])
    px, py, pok = O.project(cam, g["pts"][:, 0], g["pts"][:, 1], g["pts"][:, 2])
    same(pok, g["proj_ok"])
    same(np.stack([px, py], -1), g["proj"])


def _rig(g):
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    return StereoRig(camera_from_record(g["cam0"]), camera_from_record(g["cam1"]),
                     RelativePose(g["R"], g["t"]))


@pytest.mark.parametrize("name", ["unified", "kb"])
def test_calibration(name):
    g = load_golden(f"calib_{name}")
    rig = _rig(g)
    cal, ok = O.calibration_field(rig)
    same(ok, g["cal_ok"])
    same(cal, g["cal"])
    i1c, cok = O.calibrate(g["i1"], rig)
    same(cok, g["i1c_ok"])
    same(i1c, g["i1c"])


@pytest.mark.parametrize("name", ["pinhole", "unified_epipole", "unified", "equidistant", "kb"])
@pytest.mark.parametrize("eps", [0.1, 0.05])
def test_trajectory_field(name, eps):
    g = load_golden(f"traj_{name}_{eps}")
    d, ok = O.trajectory_field(camera_from_record(g["cam"]), g["t"], float(g["eps"]))
    same(ok, g["ok"])
    same(d, g["dirs"])


@pytest.mark.parametrize("c", [1, 2])
def test_bicubic(c):
    g = load_golden(f"bicubic_c{c}")
    v, ok = O.bicubic(g["field"], g["pos"], g["mask"])
    same(ok, g["ok"])
    np.testing.assert_array_equal(np.isnan(v), np.isnan(g["vals"]))
    same(np.nan_to_num(v), np.nan_to_num(g["vals"]))


def test_grad_div():
    g = load_golden("graddiv")
    same(O.grad_fwd(g["u"], g["mask"]), g["grad"])
    same(O.div_bwd(g["p"], g["mask"]), g["div"])


def test_smoothing_matches_scipy_gaussian():
    g = load_golden("smooth")
    for k in range(4):
        out = O.smooth_in_mask(g[f"f{k}"], g[f"m{k}"], float(g[f"s{k}"]))
        same(out, g[f"out{k}"])


def test_pyramid_and_upsample():
    g = load_golden("pyramid")
    fs, ms = O.build_levels(g["img"], g["mask"], 4, 2.0, 5)
    assert len(fs) == int(g["n"])
    for i in range(len(fs)):
        same(ms[i], g[f"m{i}"])
        same(fs[i], g[f"f{i}"])
    u2, w2 = O.lift_state(g["up_u"], g["up_w"], ms[1], ms[2].shape, ms[2])
    same(u2, g["up_u_out"])
    same(w2, g["up_w_out"])


def test_tensor_steps_pd():
    g = load_golden("pd")
    prm = SimpleNamespace(lam=5.0, alpha0=17.0, alpha1=1.2, beta=9.0, eta=0.85, theta=1.0)
    T = O.edge_tensor(g["image"], g["mask"], prm.beta, prm.eta)
    same(T, g["T"])
    st = O.step_sizes(T, g["mask"], prm.alpha0, prm.alpha1)
    same(st.sigma_p, g["sigma_p"])
    same(st.tau_u, g["tau_u"])
    same(st.tau_v, g["tau_v"])
    s = O.PDState(u=g["u"], v=g["v"], p=g["p"], q=g["q"], u_bar=g["u_bar"], v_bar=g["v_bar"])
    out = O.pd_cycle(s, T, g["iu"], g["rho0"], g["u_omega"], prm, g["mask"], st)
    for k in ("u", "v", "p", "q", "u_bar", "v_bar"):
        same(getattr(out, k), g[f"out_{k}"])


def test_shrink():
    g = load_golden("shrink")
    same(O.shrink(g["u_hat"], g["rho"], g["iu"], g["tau"], float(g["lam"])), g["out"])


def _params(g):
    return SimpleNamespace(**json.loads(str(g["params"])))


def test_level_solve():
    g = load_golden("level_solve")
    tr = O.Trace()
    u, w, s = O.level_solve(g["i0"], g["i1"], g["dirs"], g["tok"], _params(g), g["mask"],
                            g["u0"], g["w0"], tr)
    same(u, g["u"])
    same(w, g["w"])
    same(s.v, g["v"])
    same(s.p, g["p"])
    same(s.q, g["q"])
    same(tr.max_p_norm, g["max_p"])
    same(tr.max_q_norm, g["max_q"])
    same(tr.max_du, g["max_du"])
    same(tr.mean_abs_du, g["mean_du"])


def test_pyramid_solve():
    g = load_golden("pyramid_solve")
    sol = O.pyramid_solve(g["i0"], g["i1"], _rig(g), _params(g), trace=True)
    same(sol.mask, g["mask"])
    same(sol.i1c, g["i1c"])
    same(sol.u, g["u"])
    same(sol.w, g["w"])
    same(sol.v, g["v"])
    same(sol.trace.max_p_norm, g["max_p"])
    same(sol.trace.max_du, g["max_du"])
    same(sol.trace.mean_abs_du, g["mean_du"])


@pytest.mark.parametrize("name", ["unified", "kb"])
def test_depth_chain(name):
    """compose_with_calibration, depth_from_correspondence (with and without a
    cap) and triangulate_midpoint against the reference."""
    g = load_golden(f"depth_{name}")
    rig = _rig(g)
    full, fok = O.compose_calibration(g["wv"], g["cal"], g["cal_ok"])
    same(fok, g["full_ok"])
    same(full, g["full"])
    d, dok = O.depth_from_corr(rig, g["full"], g["valid"])
    same(dok, g["depth_ok"])
    np.testing.assert_allclose(d, g["depth"], rtol=1e-12, atol=0)
    d2, dok2 = O.depth_from_corr(rig, g["full"], g["valid"], depth_cap=2.0)
    same(dok2, g["depth_cap2_ok"])
    np.testing.assert_allclose(d2, g["depth_cap2"], rtol=1e-12, atol=0)
    t, tok = O.triangulate(rig, g["x0"], g["x1"])
    same(tok, g["tri_ok"])
    np.testing.assert_allclose(t, g["tri"], rtol=1e-12, atol=0)
    assert np.isnan(t[~tok]).all()
