"""TV-L1 / Huber-TV on the GPU (parity unpinned against the TGV-only reference;
pinned against the oracle's restatement, see tests/test_regularizers.py)."""

import numpy as np
import pytest

from oracle import fs_oracle as O

pytestmark = pytest.mark.gpu


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def _pair(h, w, seed):
    from test_gpu_blocked import _random_pair
    return _random_pair(h, w, seed)


# cluster path (64x64), TMA path with its tile work list (200x256)
@pytest.mark.parametrize("shape", [(64, 64), (200, 256)])
@pytest.mark.parametrize("reg", ["tv", "huber"])
def test_level_solve_variants_match_v1_and_oracle(shape, reg):
    from paper_1909_07545_b200.solver import Diagnostics, SolverParams, WarpState, solve_level
    h, w = shape
    i0, i1, dirs, tok, mask = _pair(h, w, seed=h + w)
    prm = SolverParams(warp_iters=3, pd_iters=6, pyramid_levels=1, regularizer=reg,
                       huber_eps=0.05)
    rng = np.random.default_rng(2)
    init = WarpState(u=f32(rng.normal(size=(h, w)) * 0.3), w=f32(rng.normal(size=(h, w, 2)) * 0.3))
    da, db = Diagnostics(), Diagnostics()
    a, sa = solve_level(i0, i1, dirs, tok, prm, mask, init, da, blocked=True)
    b, sb = solve_level(i0, i1, dirs, tok, prm, mask, init, db, blocked=False)
    for st in (sa, sb):
        assert not st.v.any() and not st.q.any()
        assert np.linalg.norm(st.p, axis=-1).max() <= 1.0 + 1e-6
    np.testing.assert_allclose(a.u, b.u, atol=1e-5)
    np.testing.assert_allclose(a.w, b.w, atol=1e-5)
    np.testing.assert_allclose(sa.p, sb.p, atol=1e-5)
    np.testing.assert_allclose(da.max_p_norm, db.max_p_norm, atol=1e-6)
    ref = O.level_solve(i0, i1, dirs, tok, prm, mask, init.u, init.w)
    err = np.abs(a.u - ref[0])[mask]
    assert np.median(err) < 1e-5 and np.percentile(err, 99) < 1e-3, (np.median(err), err.max())


@pytest.mark.parametrize("reg", ["tv", "huber"])
def test_fp64_variant_reproduces_oracle(reg):
    import json
    from conftest import camera_from_record, load_golden
    from paper_1909_07545_b200.camera import RelativePose, StereoRig
    from paper_1909_07545_b200.solver import SolverParams, solve_pyramid
    g = load_golden("pyramid_solve")
    rig = StereoRig(camera_from_record(g["cam0"]), camera_from_record(g["cam1"]),
                    RelativePose(g["R"], g["t"]))
    d = json.loads(str(g["params"]))
    d.update(regularizer=reg, huber_eps=0.05)
    prm = SolverParams.from_dict(d)
    res = solve_pyramid(g["i0"], g["i1"], rig, prm, precision="fp64")
    sol = O.pyramid_solve(g["i0"], g["i1"], rig, prm)
    assert np.max(np.abs(res.u - sol.u)[sol.mask]) <= 1e-8
    assert not res.v.any()
    r32 = solve_pyramid(g["i0"], g["i1"], rig, prm, precision="fp32")
    e = np.abs(r32.u - sol.u)[sol.mask]
    assert np.median(e) <= 1e-3 and np.percentile(e, 99) <= 1e-2


@pytest.mark.parametrize("reg", ["tgv", "tv", "huber"])
def test_energy_decreases_from_zero_init(reg):
    """test_solver.py:408-417 on the reference's small fisheye rig, per variant."""
    from paper_1909_07545_b200 import synth as S
    from paper_1909_07545_b200.camera import RelativePose, StereoRig, UnifiedCamera
    from paper_1909_07545_b200.fields import calibrate_second_image
    from paper_1909_07545_b200.solver import SolverParams, energy, solve_pyramid
    cam0 = UnifiedCamera(width=200, height=200, fx=100.0, fy=100.0, cx=99.5, cy=99.5,
                         fov=np.pi, xi=0.9)
    cam1 = UnifiedCamera(width=200, height=200, fx=100.0, fy=100.0, cx=100.0, cy=99.7,
                         fov=np.pi, xi=0.9)
    rig = StereoRig(cam0, cam1, RelativePose.from_displacement((0.1, 0.0, 0.0),
                                                              rotvec=(0.0, 0.02, 0.005)))
    scene = S.Scene(primitives=(S.Sphere(center=(0.0, 0.0, 0.0), radius=5.0,
                                         texture=S.ValueNoise(scale=1.0, octaves=3, seed=11,
                                                              lo=0.2, hi=0.9)),))
    i0, _, _ = S.render(scene, rig.cam0, supersample=2)
    i1, _, _ = S.render(scene, rig.cam1, pose=rig.pose, supersample=2)
    prm = SolverParams(warp_iters=8, pyramid_levels=3, min_width=40, regularizer=reg)
    res = solve_pyramid(i0, i1, rig, prm)
    i1c, _, _, _ = calibrate_second_image(i1, rig)
    z2 = np.zeros(i0.shape + (2,))
    e0 = energy(i0, i1c, res.mask, np.zeros_like(i0), z2, z2, prm)
    e1 = energy(i0, i1c, res.mask, res.u, res.v, res.w, prm)
    assert e1 < e0, (e0, e1)
