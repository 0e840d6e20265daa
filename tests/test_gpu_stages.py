"""Per-stage parity: libfsb200 (sm_100a) vs the pinned CPU oracle.

Inputs are the golden fixtures' seeded inputs; the oracle runs on exactly the
values the GPU sees (fp32-rounded where the device stores fp32). Tolerances
are the SURVEY §8c per-stage gates: trajectory field <= 1e-5 abs (fp64 compute,
fp32 store), fp64-accumulated gathers ~ fp32 output rounding, fp32 stencils
<= 1e-5 relative.
"""

import numpy as np
import pytest

from conftest import camera_from_record, load_golden
from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu

CAMS = ["pinhole", "unified", "equidistant", "kb"]


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("name", CAMS)
def test_lens_models(name):
    from paper_1909_07545_b200 import camera as K
    g = load_golden(f"camera_{name}")
    cam = camera_from_record(g["cam"])
    np.testing.assert_array_equal(K.fov_mask(cam), O.fov_mask(cam))
    rays, ok = K.unproject(cam, g["pix"])
    rx, ry, rz, ook = O.unproject(cam, g["pix"][:, 0], g["pix"][:, 1])
    np.testing.assert_array_equal(ok, ook)
    np.testing.assert_allclose(rays[ok], np.stack([rx, ry, rz], -1)[ok], atol=1e-13, rtol=0)
    assert np.isnan(rays[~ok]).all()
    pix, pok = K.project(cam, g["pts"])
    px, py, opk = O.project(cam, g["pts"][:, 0], g["pts"][:, 1], g["pts"][:, 2])
    np.testing.assert_array_equal(pok, opk)
    np.testing.assert_allclose(pix[pok], np.stack([px, py], -1)[pok], atol=1e-10, rtol=1e-13)


def _rig(g):
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    return StereoRig(camera_from_record(g["cam0"]), camera_from_record(g["cam1"]),
                     RelativePose(g["R"], g["t"]))


@pytest.mark.parametrize("name", ["unified", "kb"])
def test_calibration(name):
    from paper_1909_07545_b200 import fields as F
    g = load_golden(f"calib_{name}")
    rig = _rig(g)
    cal, ok = F.generate_calibration_field(rig)
    ocal, ook = O.calibration_field(rig)
    np.testing.assert_array_equal(ok, ook)
    np.testing.assert_allclose(cal, ocal, atol=1e-10, rtol=0)
    i1 = f32(g["i1"])
    i1c, cok, _, _ = F.calibrate_second_image(i1, rig)
    oi1c, ocok = O.calibrate(i1, rig)
    np.testing.assert_array_equal(cok, ocok)
    np.testing.assert_allclose(i1c, oi1c, atol=2e-7, rtol=0)  # f64 taps, f32 store


@pytest.mark.parametrize("name", ["pinhole", "unified_epipole", "unified", "equidistant", "kb"])
@pytest.mark.parametrize("eps", [0.1, 0.05])
def test_trajectory_field(name, eps):
    """North-star gate: trajectory field within 1e-5 absolute."""
    from paper_1909_07545_b200 import fields as F
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    g = load_golden(f"traj_{name}_{eps}")
    cam = camera_from_record(g["cam"])
    rig = StereoRig(cam, cam, RelativePose(np.eye(3), g["t"]))
    d, ok = F.generate_trajectory_field(rig, epsilon_scale=eps)
    od, ook = O.trajectory_field(cam, g["t"], eps)
    np.testing.assert_array_equal(ok, ook)
    assert np.max(np.abs(d - od)) <= 1e-5
    if name == "pinhole":  # fields.py:91-96 snapping: exactly (-1, 0)
        assert np.all(d[ok][:, 0] == -1.0) and np.all(d[ok][:, 1] == 0.0)


def test_trajectory_zero_baseline_and_rotation_rejected():
    from paper_1909_07545_b200 import fields as F
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    cam = camera_from_record(load_golden("camera_unified")["cam"])
    with pytest.raises(ValueError):
        F.generate_trajectory_field(StereoRig(cam, cam, RelativePose()))
    with pytest.raises(ValueError):
        F.generate_trajectory_field(StereoRig(cam, cam, RelativePose.from_displacement(
            (0.1, 0, 0), rotvec=(0, 0.01, 0))))


@pytest.mark.parametrize("c", [1, 2])
@pytest.mark.parametrize("acc64", [True, False])
def test_bicubic(c, acc64):
    from paper_1909_07545_b200.rasters import sample_bicubic
    g = load_golden(f"bicubic_c{c}")
    field = f32(g["field"])
    v, ok = sample_bicubic(field, g["pos"], g["mask"], acc64=acc64)
    ov, ook = O.bicubic(field, g["pos"], g["mask"])
    np.testing.assert_array_equal(ok, ook)
    assert np.isnan(v[~ok]).all()
    tol = 1e-6 if acc64 else 1e-5
    np.testing.assert_allclose(v[ok], ov[ok], atol=tol, rtol=0)


def test_bicubic_reference_unit_cases():
    """Reference test_rasters.py:13-80 known answers, on the GPU sampler."""
    from paper_1909_07545_b200.rasters import pixel_grid, sample_bicubic
    full = np.ones((16, 16), bool)
    v, ok = sample_bicubic(np.full((16, 16), 0.7), np.array([[3.2, 5.7], [0, 0], [14.9, 14.9]]),
                           full)
    assert ok.all() and np.allclose(v, 0.7, atol=1e-7)
    f = np.random.default_rng(0).normal(size=(16, 16)).astype(np.float32)
    v, ok = sample_bicubic(f, np.array([[7.0, 9.0], [0.0, 0.0], [15.0, 15.0]]), full)
    assert ok.all() and np.array_equal(v, [f[9, 7], f[0, 0], f[15, 15]])
    v, ok = sample_bicubic(np.ones((16, 16)), np.array([8.0, 8.0]), np.zeros((16, 16), bool))
    assert not ok and np.isnan(v)
    v, ok = sample_bicubic(np.ones((16, 16)), np.array([40.0, 2.0]), full)
    assert not ok
    fld = np.zeros((16, 16)); fld[8, 8] = 4.0
    m = np.zeros((16, 16), bool); m[8, 8] = True
    v, ok = sample_bicubic(fld, np.array([8.3, 7.9]), m)
    assert ok and v == 4.0
    g = pixel_grid(32, 32)
    v, ok = sample_bicubic(2.0 * g[:, :, 0] + 3.0 * g[:, :, 1], np.array([10.5, 4.25]),
                           np.ones((32, 32), bool))
    assert ok and abs(float(v) - 33.75) < 1e-5


def test_grad_div_and_adjointness():
    from paper_1909_07545_b200.rasters import divergence, gradient
    g = load_golden("graddiv")
    u, p = f32(g["u"]), f32(g["p"])
    np.testing.assert_allclose(gradient(u, g["mask"]), O.grad_fwd(u, g["mask"]), atol=1e-6)
    np.testing.assert_allclose(divergence(p, g["mask"]), O.div_bwd(p, g["mask"]), atol=1e-6)
    rng = np.random.default_rng(7)
    for _ in range(20):  # criterion 02 (test_acceptance.py:103-115), fp32 tolerance
        uu = f32(rng.normal(size=(32, 32)))
        pp = f32(rng.normal(size=(32, 32, 2)))
        m = rng.random((32, 32)) > 0.35
        lhs = float(np.sum(gradient(uu, m) * pp))
        rhs = -float(np.sum(uu * divergence(pp, m)))
        assert abs(lhs - rhs) <= 1e-4 * max(1.0, abs(lhs))


def test_smoothing():
    from paper_1909_07545_b200.rasters import smooth_masked
    g = load_golden("smooth")
    for k in range(4):
        f = f32(g[f"f{k}"])
        out = smooth_masked(f, g[f"m{k}"], float(g[f"s{k}"]))
        np.testing.assert_allclose(out, O.smooth_in_mask(f, g[f"m{k}"], float(g[f"s{k}"])),
                                   atol=1e-7, rtol=0)


def test_pyramid_and_upsample():
    from paper_1909_07545_b200.rasters import build_pyramid, upsample_state
    g = load_golden("pyramid")
    img = f32(g["img"])
    pyr = build_pyramid(img, g["mask"], 4, 2.0, 5)
    fs, ms = O.build_levels(img, g["mask"], 4, 2.0, 5)
    assert pyr.num_levels == len(fs)
    for a, b, ma, mb in zip(pyr.fields, fs, pyr.masks, ms):
        np.testing.assert_array_equal(ma, mb)
        np.testing.assert_allclose(a, b, atol=2e-7, rtol=0)
    uu, ww = f32(g["up_u"]), f32(g["up_w"])
    u2, w2 = upsample_state(uu, ww, ms[1], ms[2].shape, ms[2])
    ou, ow = O.lift_state(uu, ww, ms[1], ms[2].shape, ms[2])
    np.testing.assert_allclose(u2, ou, atol=1e-6, rtol=0)
    np.testing.assert_allclose(w2, ow, atol=1e-6, rtol=0)


def test_tensor_and_steps():
    from paper_1909_07545_b200.solver import SolverParams, compute_tensor, precondition_steps
    g = load_golden("pd")
    im = f32(g["image"])
    p = SolverParams()
    T = compute_tensor(im, p.beta, p.eta, g["mask"])
    oT = O.edge_tensor(im, g["mask"], p.beta, p.eta)
    np.testing.assert_allclose(T, oT, atol=1e-7, rtol=0)
    st = precondition_steps(oT, g["mask"], p)
    ost = O.step_sizes(f32(oT), g["mask"], p.alpha0, p.alpha1)
    for k in ("sigma_p", "tau_u", "tau_v"):
        np.testing.assert_allclose(getattr(st, k), getattr(ost, k), rtol=1e-7)


def test_pd_iteration():
    from paper_1909_07545_b200.solver import SolverParams, SolverState, primal_dual_iterate
    g = load_golden("pd")
    p = SolverParams()
    T = f32(g["T"])
    st = O.step_sizes(T, g["mask"], p.alpha0, p.alpha1)
    st = O.Steps(f32(st.sigma_p), st.sigma_q, f32(st.tau_u), f32(st.tau_v))
    s = {k: f32(g[k]) for k in ("u", "v", "p", "q", "u_bar", "v_bar")}
    args = (f32(g["iu"]), f32(g["rho0"]), f32(g["u_omega"]))
    out = primal_dual_iterate(SolverState(**s), T, *args, p, g["mask"], steps=st)
    ref = O.pd_cycle(O.PDState(**s), T, *args, p, g["mask"], st)
    for k in ("u", "v", "p", "q", "u_bar", "v_bar"):
        a, b = getattr(out, k), getattr(ref, k)
        np.testing.assert_allclose(a, b, atol=2e-6, rtol=2e-6, err_msg=k)
    assert np.linalg.norm(out.p, axis=-1).max() <= 1 + 1e-6
    assert np.linalg.norm(out.q, axis=-1).max() <= 1 + 1e-6


def test_pd_stationary_at_zero_data():
    """test_solver.py:189-200: exact zeros stay exact in fp32."""
    from paper_1909_07545_b200.solver import (SolverParams, SolverState, compute_tensor,
                                              primal_dual_iterate)
    mask = np.ones((20, 20), bool)
    t = compute_tensor(np.full((20, 20), 0.5), 9.0, 0.85, mask)
    u0 = np.full((20, 20), 1.7)
    z2 = np.zeros((20, 20, 2))
    s = SolverState(u=u0.copy(), v=z2, p=z2, q=np.zeros((20, 20, 4)), u_bar=u0.copy(), v_bar=z2)
    for _ in range(5):
        s = primal_dual_iterate(s, t, np.zeros((20, 20)), np.zeros((20, 20)), u0,
                                SolverParams(), mask)
    assert np.array_equal(s.u, np.float32(u0))
    assert np.all(s.p == 0) and np.all(s.q == 0) and np.all(s.v == 0)


def test_thresholding():
    from paper_1909_07545_b200.solver import thresholding_step
    g = load_golden("shrink")
    out = thresholding_step(g["u_hat"], g["rho"], g["iu"], g["tau"], float(g["lam"]))
    np.testing.assert_allclose(out, g["out"], atol=1e-15, rtol=1e-15)
    # reference test_solver.py:128-153 known answers
    assert np.isclose(thresholding_step(2.0, 1.5, 2.0, 0.25, 1.0), 1.5, atol=1e-12)
    assert np.isclose(thresholding_step(2.0, 0.4, 2.0, 0.25, 1.0), 1.8, atol=1e-12)
    assert float(thresholding_step(1.3, 0.0, 2.0, 0.25, 1.0)) == 1.3
    assert float(thresholding_step(1.3, 0.7, 0.0, 0.25, 1.0)) == 1.3


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("amp", [0.0, 1.5, 6.0])
def test_warp_linearize_stage_gate_fp64(kind, amp):
    """SURVEY §8(c) per-stage gate of K5 on the float64 path: i1w, dirs, I_u and
    rho0 each within 1e-6 of the oracle (oracle/fs_oracle.linearize =
    solver.py:332-346 + 192-202) with validity identical, for a zero, a small
    and a large random warp field (the large one drives stencils across the mask
    edge into every fallback branch), with both prologue kernels (kind 0 masked
    gathers, kind 1 NaN-encoded texels)."""
    from paper_1909_07545_b200.solver import warp_linearize64
    g = load_golden("level_solve")
    h, w = g["mask"].shape
    rng = np.random.default_rng(int(10 * amp) + kind)
    wv = amp * rng.standard_normal((h, w, 2))
    got = warp_linearize64(g["i0"], g["i1"], g["mask"], g["dirs"], g["tok"], wv, kind)
    ref = O.linearize(g["i0"], g["i1"], g["dirs"], g["tok"], g["mask"], wv)
    m = g["mask"]
    i1w, wok, dirs, dok, iu, rho0 = got
    ri1w, rwok, rdirs, rdok, riu, rrho0 = ref
    np.testing.assert_array_equal(wok & m, rwok & m)
    np.testing.assert_array_equal(dok, rdok)
    assert np.max(np.abs(np.where(m & rwok, i1w - ri1w, 0.0))) <= 1e-6
    assert np.max(np.abs(dirs - rdirs)) <= 1e-6
    assert np.max(np.abs(iu - riu)) <= 1e-6
    assert np.max(np.abs(rho0 - rrho0)) <= 1e-6
    # the gate is met with orders of margin: same operation order as the oracle
    assert max(np.max(np.abs(iu - riu)), np.max(np.abs(dirs - rdirs))) <= 1e-12
    if amp > 0:  # the field really exercises partial stencils
        assert (rwok & m).sum() < m.sum() or (rdok != m).any()
