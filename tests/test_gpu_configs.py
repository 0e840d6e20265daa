"""GPU renderer parity and end-to-end parity on the BASELINE configurations.

The renderer (input generator) is checked against the reference's own renders
(tests/golden/render.npz). The solve is checked against the pinned oracle on
GPU-rendered inputs at the sizes the oracle finishes in seconds (C1 at full
size; C2 geometry at full size), and at the headline 1024^2 size (C3) through
size-independent invariants, the per-level trajectory fields against the oracle
and the fp32 / fp64 paths against the oracle.
"""

import numpy as np
import pytest

from conftest import camera_from_record, load_golden
from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu


def test_render_matches_reference():
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.camera import RelativePose
    g = load_golden("render")
    cams = {n: camera_from_record(load_golden(f"camera_{n}")["cam"])
            for n in ("unified", "kb", "pinhole", "equidistant")}
    sc = S.default_scene()
    extra = S.Scene(primitives=(
        S.Plane(point=(0.0, 0.0, 2.0), normal=(0.1, 0.0, -1.0), texture=S.Checkerboard(period=0.3)),
        S.Sphere(center=(-0.3, 0.2, 1.2), radius=0.3,
                 texture=S.SineGrating(wavelength=0.2, direction=(1.0, 1.0, 0.0))),
        S.Box(lo=(0.2, -0.5, 0.9), hi=(0.6, -0.1, 1.4), texture=S.ValueNoise(scale=0.1, octaves=2,
                                                                             seed=3))))
    cases = [(sc, cams["unified"], None, 2),
             (sc, cams["kb"], RelativePose.from_displacement((0.1, 0, 0), rotvec=(0, .03, 0)), 1),
             (extra, cams["pinhole"], None, 3),
             (S.reseed_scene(sc, 5), cams["equidistant"], None, 1)]
    for k, (scene, cam, pose, ss) in enumerate(cases):
        img, depth, hit = S.render(scene, cam, pose=pose, supersample=ss)
        ref_hit = g[f"hit{k}"]
        assert np.mean(hit == ref_hit) >= 0.999
        both = hit & ref_hit
        close = np.abs(img - g[f"img{k}"])[both] <= 1e-5
        assert close.mean() >= 0.995, (k, close.mean())
        np.testing.assert_allclose(depth[both], g[f"depth{k}"][both], rtol=1e-6, atol=1e-6)


def _c1():
    """BASELINE config 1: 320^2 equidistant, pure x baseline."""
    from paper_1909_07545_b200.camera import PolynomialFisheyeCamera, RelativePose, StereoRig
    from paper_1909_07545_b200.solver import SolverParams
    cam = PolynomialFisheyeCamera(width=320, height=320, fx=100.0, fy=100.0, cx=159.5, cy=159.5,
                                  fov=np.pi, k=(1.0, 0.0, 0.0, 0.0))
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.1, 0.0, 0.0)))
    return rig, SolverParams(warp_iters=5, pd_iters=10, pyramid_levels=3)


def _c2():
    """BASELINE config 2 geometry: 640x480 Kannala-Brandt."""
    from paper_1909_07545_b200.camera import PolynomialFisheyeCamera, RelativePose, StereoRig
    from paper_1909_07545_b200.solver import SolverParams
    kw = dict(width=640, height=480, fx=200.0, fy=200.0, cy=239.5, fov=np.deg2rad(163.0),
              k=(1.0, 0.03, -0.006, 0.001))
    rig = StereoRig(PolynomialFisheyeCamera(cx=319.5, **kw), PolynomialFisheyeCamera(cx=320.5, **kw),
                    RelativePose.from_displacement((0.064, 0, 0), rotvec=(0.002, 0.004, 0.001)))
    return rig, SolverParams(warp_iters=10, pd_iters=10, pyramid_levels=5, min_width=40)


def _render_pair(rig, ss=2):
    from paper_1909_07545_b200 import synth as S
    scene = S.default_scene()
    i0, _, _ = S.render(scene, rig.cam0, supersample=ss)
    i1, _, _ = S.render(scene, rig.cam1, pose=rig.pose, supersample=ss)
    return i0, i1


def _parity(rig, prm, i0, i1, precision="fp32", p99_tol=1e-2, sol=None):
    from paper_1909_07545_b200.solver import solve_pyramid
    res = solve_pyramid(i0, i1, rig, prm, collect_diagnostics=True, precision=precision)
    sol = sol if sol is not None else O.pyramid_solve(i0, i1, rig, prm)
    np.testing.assert_array_equal(res.mask, sol.mask)
    e = np.abs(res.u - sol.u)[sol.mask]
    med, p99, mx = float(np.median(e)), float(np.percentile(e, 99)), float(e.max())
    print(f"[{precision}] u err median {med:.3e} p99 {p99:.3e} max {mx:.3e}; "
          f"u range {sol.u.max():.2f}")
    assert med <= 1e-3 and (p99_tol is None or p99 <= p99_tol)
    d = res.diagnostics
    assert max(d.max_p_norm) <= 1 + 1e-6 and max(d.max_q_norm) <= 1 + 1e-6
    assert max(d.max_du) <= prm.du_max * (1 + 1e-6)
    return res, sol


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c1_end_to_end_parity(precision):
    rig, prm = _c1()
    i0, i1 = _render_pair(rig)
    _parity(rig, prm, i0, i1, precision=precision)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c2_kannala_brandt_end_to_end_parity(precision):
    rig, prm = _c2()
    i0, i1 = _render_pair(rig, ss=1)
    _parity(rig, prm, i0, i1, precision=precision)


def test_degenerates_to_rectified():
    """Criterion 05 (test_acceptance.py:165-191): on a pinhole pair the fisheye
    pipeline equals hard-coded horizontal directions."""
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    rig = S.pinhole_rig(width=240, height=240, f=200.0, baseline=0.1)
    scene = S.Scene(primitives=(
        S.Plane(point=(0.0, 0.0, 2.2), normal=(0.0, 0.0, -1.0),
                texture=S.ValueNoise(scale=0.5, octaves=4, seed=5, lo=0.05, hi=0.95,
                                     persistence=0.65)),
        S.Sphere(center=(0.3, -0.25, 1.4), radius=0.35,
                 texture=S.ValueNoise(scale=0.1, octaves=4, seed=23, lo=0.1, hi=0.9,
                                      persistence=0.65))))
    i0, _, _ = S.render(scene, rig.cam0, supersample=2)
    i1, _, _ = S.render(scene, rig.cam1, pose=rig.pose, supersample=2)

    def horizontal(rig_lvl):
        h, w = rig_lvl.cam0.height, rig_lvl.cam0.width
        d = np.zeros((h, w, 2))
        d[:, :, 0] = -1.0
        return d, rig_lvl.cam0.fov_mask()

    prm = SolverParams(warp_iters=10, pyramid_levels=4, min_width=30)
    a = solve_pyramid(i0, i1, rig, prm)
    b = solve_pyramid(i0, i1, rig, prm, traj_override=horizontal)
    assert np.max(np.abs(a.u - b.u)) <= 1e-6
    assert np.max(np.linalg.norm(a.w - b.w, axis=-1)) <= 1e-6
    # rectified oracle: 4 px disparity plane (test_solver.py:387-399) sanity
    assert np.isfinite(a.u).all()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_rectified_constant_disparity(precision):
    """test_solver.py:387-399: fronto plane at f*b/4 gives 4 px of disparity."""
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.rasters import gradient
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    rig = S.pinhole_rig(width=240, height=240, f=300.0, baseline=0.1)
    scene = S.plane_scene(depth=300.0 * 0.1 / 4.0,
                          texture=S.ValueNoise(scale=1.7, octaves=4, seed=9, lo=0.05, hi=0.95,
                                               persistence=0.65))
    i0, _, _ = S.render(scene, rig.cam0, supersample=2)
    i1, _, _ = S.render(scene, rig.cam1, pose=rig.pose, supersample=2)
    res = solve_pyramid(i0, i1, rig, SolverParams(warp_iters=10, pyramid_levels=4, min_width=30),
                        precision=precision)
    g = np.linalg.norm(gradient(i0, res.mask), axis=-1)
    textured = res.mask & (g > 0.02)
    assert np.mean(np.abs(res.u[textured] - 4.0) < 0.5) >= 0.95


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c3_headline_invariants(precision):
    """C3 (1024^2 unified, 6-DoF, reference defaults N=50 K=10): size-independent
    properties — determinism, dual feasibility, du clip, finite output, and
    agreement of the calibrated image with the oracle (fp64 taps)."""
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import Solver, SolverParams
    cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5,
                        fov=np.pi, xi=0.9)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.08, 0.02, 0.03),
                                                             rotvec=(0.01, 0.03, -0.02)))
    i0, i1 = _render_pair(rig, ss=1)
    prm = SolverParams()
    eng = Solver(rig, prm, collect_diagnostics=True, precision=precision)
    r1 = eng.solve(i0, i1)
    r2 = eng.solve(i0, i1)
    assert np.array_equal(r1.u, r2.u) and np.array_equal(r1.w, r2.w)
    d = r1.diagnostics
    assert len(d.max_p_norm) == 5 * 50 * 10
    assert max(d.max_p_norm) <= 1 + 1e-6 and max(d.max_q_norm) <= 1 + 1e-6
    assert max(d.max_du) <= prm.du_max * (1 + 1e-6)
    assert np.isfinite(r1.u).all() and np.isfinite(r1.w).all()
    assert 0.6 < r1.mask.mean() < 0.9
    i1c, ok = O.calibrate(i1, rig)
    np.testing.assert_array_equal(ok & O.fov_mask(rig.cam0), r1.mask)
    np.testing.assert_allclose(r1.i1_calibrated, i1c, atol=2e-7)


def test_c3_full_size_trajectory_fields():
    """North-star trajectory gate at the headline config (C3, 1024^2, 6-DoF
    unified rig): the trajectory field of EVERY pyramid level (1024^2 .. 64^2,
    the residual rig of fields.py:159-167 on cam0.scaled_to, solver.py:435-441)
    within 1e-5 of the fp64 oracle, validity identical. The full-size C3
    disparity gate against the reference is tests/test_gpu_c3_parity.py."""
    from paper_1909_07545_b200 import fields as F
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.rasters import pyramid_shapes
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5,
                        fov=np.pi, xi=0.9)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.08, 0.02, 0.03),
                                                             rotvec=(0.01, 0.03, -0.02)))
    prm = SolverParams()
    res_rig = F.translation_only_rig(rig)
    shapes = pyramid_shapes(1024, 1024, prm.pyramid_levels, prm.pyramid_scale, prm.min_width)
    assert len(shapes) == 5
    for shp in shapes:
        c = res_rig.cam0.scaled_to(shp)
        lrig = StereoRig(c, c, res_rig.pose)
        d, ok = F.generate_trajectory_field(lrig, epsilon_scale=prm.epsilon_scale)
        od, ook = O.trajectory_field(c, res_rig.pose.translation, prm.epsilon_scale)
        np.testing.assert_array_equal(ok, ook)
        assert np.max(np.abs(d - od)[ok]) <= 1e-5, shp


def test_n50_parity_on_acceptance_geometry():
    """The reference acceptance setup (default_rig 400^2, default_scene, reference
    defaults N=50 x K=10, 4 levels, du_max 0.1 = criterion 06).

    fp64 path (the default): north-star gate median <= 1e-3 px, p99 <= 1e-2 px
    (it reproduces the reference to round-off). fp32 path: only the median gate
    is asserted; its p99 is printed — rounding ANY one quantity of the fp64
    reference to fp32 already gives p99 ~2e-2 at N=50
    (profiles/r01_precision_study.txt), so fp32 misses the p99
    gate here by construction and is not the default."""
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.solver import SolverParams
    rig = S.default_rig()
    i0, i1 = _render_pair(rig, ss=2)
    prm = SolverParams(du_max=0.1)
    sol = O.pyramid_solve(i0, i1, rig, prm)
    _parity(rig, prm, i0, i1, precision="fp64", p99_tol=1e-2, sol=sol)
    _parity(rig, prm, i0, i1, precision="fp32", p99_tol=None, sol=sol)


def test_fp64_path_reproduces_oracle_to_roundoff():
    """The float64 path on the golden pair and on C1: disparity and warp
    agree with the fp64 oracle to ~1e-9 (same algorithm, same operation order)."""
    import json
    from conftest import load_golden
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    g = load_golden("pyramid_solve")
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    rig = StereoRig(camera_from_record(g["cam0"]), camera_from_record(g["cam1"]),
                    RelativePose(g["R"], g["t"]))
    prm = SolverParams.from_dict(json.loads(str(g["params"])))
    res = solve_pyramid(g["i0"], g["i1"], rig, prm, precision="fp64", collect_diagnostics=True)
    np.testing.assert_array_equal(res.mask, g["mask"])
    assert np.max(np.abs(res.u - g["u"])) <= 1e-8
    assert np.max(np.abs(res.w - g["w"])) <= 1e-8
    assert np.max(np.abs(res.i1_calibrated - g["i1c"])) <= 1e-12
    np.testing.assert_allclose(res.diagnostics.max_du, g["max_du"], atol=1e-7)
    rig1, prm1 = _c1()
    i0, i1 = _render_pair(rig1)
    r1 = solve_pyramid(i0, i1, rig1, prm1, precision="fp64")
    s1 = O.pyramid_solve(i0, i1, rig1, prm1)
    assert np.max(np.abs(r1.u - s1.u)[s1.mask]) <= 1e-8


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_odd_size_pipeline_parity(precision):
    """A 322x241 unified pair: width % 4 != 0 selects the non-TMA pair kernel
    fallback, ragged pyramid shapes and partial tiles at every level."""
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import SolverParams
    cam0 = UnifiedCamera(width=322, height=241, fx=140.0, fy=141.0, cx=160.3, cy=120.2,
                         fov=np.pi, xi=0.9)
    cam1 = UnifiedCamera(width=322, height=241, fx=140.0, fy=141.0, cx=161.0, cy=119.8,
                         fov=np.pi, xi=0.9)
    rig = StereoRig(cam0, cam1, RelativePose.from_displacement((0.1, 0.01, 0.0),
                                                               rotvec=(0.0, 0.02, 0.005)))
    prm = SolverParams(warp_iters=8, pd_iters=10, pyramid_levels=3, min_width=40)
    i0, i1 = _render_pair(rig)
    _parity(rig, prm, i0, i1, precision=precision)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c5_headline_invariants(precision):
    """C5 (2048^2 unified, 7 levels, N=20 x K=10, Huber-TV): the size-independent
    invariants (determinism, feasible duals, v = 0 for the TV-type regulariser,
    clipped increments, finite output)."""
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import Solver, SolverParams
    cam = UnifiedCamera(width=2048, height=2048, fx=910.0, fy=910.0, cx=1023.5, cy=1023.5,
                        fov=np.pi, xi=0.9)
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.1, 0, 0), rotvec=(0, 0.02, 0.005)))
    sc = S.default_scene()
    i0 = S.render_device(sc, rig.cam0)[0].double().cpu().numpy()
    i1 = S.render_device(sc, rig.cam1, pose=rig.pose)[0].double().cpu().numpy()
    prm = SolverParams(warp_iters=20, pd_iters=10, pyramid_levels=7, min_width=32,
                       regularizer="huber")
    eng = Solver(rig, prm, collect_diagnostics=True, precision=precision)
    r1 = eng.solve(i0, i1)
    r2 = eng.solve(i0, i1)
    assert np.array_equal(r1.u, r2.u) and np.array_equal(r1.w, r2.w)
    d = r1.diagnostics
    assert len(d.max_p_norm) == 7 * 20 * 10
    assert max(d.max_p_norm) <= 1 + 1e-6 and max(d.max_q_norm) == 0.0
    assert max(d.max_du) <= prm.du_max * (1 + 1e-6)
    assert not r1.v.any()
    assert np.isfinite(r1.u).all() and np.isfinite(r1.w).all()
    assert 0.6 < r1.mask.mean() < 0.9


@pytest.mark.parametrize("shape", [(12, 10), (9, 40), (40, 9), (1, 64)])
def test_tiny_and_degenerate_shapes(shape):
    """Single-level solves on tiny / one-pixel-wide images (cluster path, empty
    interiors, no right or lower neighbours) against the oracle."""
    from paper_1909_07545_b200.camera import PinholeCamera, RelativePose, StereoRig
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    h, w = shape
    cam = PinholeCamera(width=w, height=h, fx=8.0, fy=8.0, cx=(w - 1) / 2.0, cy=(h - 1) / 2.0,
                        fov=np.deg2rad(150.0))
    rig = StereoRig(cam, cam, RelativePose.from_displacement((0.1, 0.0, 0.0)))
    rng = np.random.default_rng(h * 100 + w)
    i0 = rng.random((h, w))
    i1 = np.roll(i0, 1, axis=1) * 0.9 + 0.05
    prm = SolverParams(warp_iters=3, pd_iters=4, pyramid_levels=1, min_width=1)
    res = solve_pyramid(i0, i1, rig, prm, collect_diagnostics=True, precision="fp32")
    sol = O.pyramid_solve(i0, i1, rig, prm)
    np.testing.assert_array_equal(res.mask, sol.mask)
    if sol.mask.any():
        e = np.abs(res.u - sol.u)[sol.mask]
        assert np.median(e) <= 1e-4 and e.max() <= 1e-3
    assert np.isfinite(res.u).all() and np.isfinite(res.w).all()
    r64 = solve_pyramid(i0, i1, rig, prm, precision="fp64")
    assert np.max(np.abs(r64.u - sol.u)) <= 1e-9


def test_noisy_render_matches_reference():
    """render(noise_sigma > 0): GPU ray casting plus the reference's own numpy
    noise stream (default_rng(noise_seed)), clipped inside the hit mask."""
    from paper_1909_07545_b200 import synth as S
    g = load_golden("render_noise")
    cam = camera_from_record(load_golden("camera_unified")["cam"])
    img, _, hit = S.render(S.default_scene(), cam, noise_sigma=0.02, noise_seed=23, supersample=2)
    assert np.mean(hit == g["hit"]) >= 0.999
    both = hit & g["hit"]
    assert (np.abs(img - g["img"])[both] <= 1e-5).mean() >= 0.995
    assert (img[~hit] == 0).all()


@pytest.mark.parametrize("seed", range(6))
def test_randomized_configurations(seed):
    """Randomised rigs (all three lens models), sizes (incl. widths that are not
    multiples of 4), pyramid depths, N / K / du_max and regularisers: the fp64
    path reproduces the oracle to round-off, the fp32 path to the parity gate."""
    from paper_1909_07545_b200.camera import (PinholeCamera, PolynomialFisheyeCamera,
                                              RelativePose, StereoRig, UnifiedCamera)
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    rng = np.random.default_rng(1000 + seed)
    w = int(rng.integers(70, 180)); h = int(rng.integers(60, 150))
    f = float(rng.uniform(0.35, 0.55)) * w
    kind = ["unified", "kb", "pinhole"][seed % 3]
    kw = dict(width=w, height=h, fx=f, fy=f * rng.uniform(0.97, 1.03), cx=(w - 1) / 2 + rng.uniform(-2, 2),
              cy=(h - 1) / 2 + rng.uniform(-2, 2))
    if kind == "unified":
        cam = UnifiedCamera(fov=np.pi, xi=float(rng.uniform(0.6, 1.0)), **kw)
    elif kind == "kb":
        cam = PolynomialFisheyeCamera(fov=np.deg2rad(170.0),
                                      k=(1.0, float(rng.uniform(-0.02, 0.04)), -0.004, 0.0005), **kw)
    else:
        cam = PinholeCamera(fov=np.deg2rad(110.0), **kw)
    t = (float(rng.uniform(0.05, 0.12)), float(rng.uniform(-0.02, 0.02)), float(rng.uniform(-0.02, 0.02)))
    rv = tuple(float(x) for x in rng.uniform(-0.02, 0.02, 3))
    rig = StereoRig(cam, cam, RelativePose.from_displacement(t, rotvec=rv))
    prm = SolverParams(warp_iters=int(rng.integers(2, 7)), pd_iters=int(rng.integers(3, 12)),
                       du_max=float(rng.uniform(0.1, 0.4)), pyramid_levels=int(rng.integers(1, 4)),
                       min_width=30, regularizer=["tgv", "tgv", "tv", "huber"][seed % 4])
    i0, i1 = _render_pair(rig, ss=1)
    sol = O.pyramid_solve(i0, i1, rig, prm)
    r64 = solve_pyramid(i0, i1, rig, prm, precision="fp64")
    np.testing.assert_array_equal(r64.mask, sol.mask)
    assert np.max(np.abs(r64.u - sol.u)) <= 1e-8
    assert np.max(np.abs(r64.w - sol.w)) <= 1e-8
    r32 = solve_pyramid(i0, i1, rig, prm, precision="fp32")
    np.testing.assert_array_equal(r32.mask, sol.mask)
    if sol.mask.any():
        e = np.abs(r32.u - sol.u)[sol.mask]
        assert np.median(e) <= 1e-3 and np.percentile(e, 99) <= 1e-2, (np.median(e), np.percentile(e, 99))


def test_ragged_size_cluster_kernels_parity():
    """A 614x452 unified pair (even width, not a multiple of 32; height not a
    multiple of 8; >= 512^2 pixels): the finest level runs k64_ctile with
    regions and CTA tiles hanging over the right and bottom edges, 307x226
    (odd width) the k64_tile fallback, 77x57 the whole-level k64_level with a
    partly filled cluster. Without diagnostics (the default kernels) and with
    them (the DIAG variants, no k64_level), against the oracle."""
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    cam0 = UnifiedCamera(width=614, height=452, fx=262.0, fy=263.0, cx=306.4, cy=225.6,
                         fov=np.pi, xi=0.9)
    cam1 = UnifiedCamera(width=614, height=452, fx=262.0, fy=263.0, cx=307.1, cy=225.1,
                         fov=np.pi, xi=0.9)
    rig = StereoRig(cam0, cam1, RelativePose.from_displacement((0.1, 0.01, 0.0),
                                                               rotvec=(0.0, 0.02, 0.005)))
    prm = SolverParams(warp_iters=3, pd_iters=10, pyramid_levels=4, min_width=40)
    i0, i1 = _render_pair(rig)
    sol = O.pyramid_solve(i0, i1, rig, prm)
    for diag in (False, True):
        res = solve_pyramid(i0, i1, rig, prm, collect_diagnostics=diag, precision="fp64")
        np.testing.assert_array_equal(res.mask, sol.mask)
        err = float(np.max(np.abs(res.u - sol.u)[sol.mask]))
        werr = float(np.max(np.abs(res.w - sol.w)[sol.mask]))
        print(f"diag={diag}: u max err {err:.3e}, w max err {werr:.3e}")
        assert err <= 1e-8 and werr <= 1e-8
