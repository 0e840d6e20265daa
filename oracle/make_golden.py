"""Generate tests/golden/*.npz by running the REFERENCE implementation.

TEST INFRASTRUCTURE ONLY. Run in the build container (the reference is not on
the GPU box):

    python oracle/make_golden.py            # reads /root/reference/pkg/src

Each fixture stores seeded inputs and the reference's own outputs for one
stage of the dense-mapping path; tests/test_oracle_golden.py pins the oracle
(oracle/fs_oracle.py) against them, and the GPU parity tests reuse the inputs.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF))
    import fisheyestereo  # noqa: F401
    from fisheyestereo import camera, fields, rasters, solver, synth
    return camera, fields, rasters, solver, synth


def cameras(camera):
    """Small test cameras of every model (shapes chosen non-square)."""
    H, W = 40, 48
    return {
        "pinhole": camera.PinholeCamera(width=W, height=H, fx=30.0, fy=31.0, cx=23.5, cy=19.5,
                                        fov=np.deg2rad(100.0)),
        "unified": camera.UnifiedCamera(width=W, height=H, fx=20.0, fy=20.5, cx=23.2, cy=19.6,
                                        fov=np.pi, xi=0.9),
        "equidistant": camera.PolynomialFisheyeCamera(width=W, height=H, fx=15.0, fy=15.0,
                                                      cx=23.5, cy=19.5, fov=np.pi,
                                                      k=(1.0, 0.0, 0.0, 0.0)),
        "kb": camera.PolynomialFisheyeCamera(width=W, height=H, fx=15.0, fy=14.5, cx=24.0,
                                             cy=19.5, fov=np.deg2rad(163.0),
                                             k=(1.0, 0.03, -0.006, 0.001)),
    }


def cam_record(c) -> str:
    d = {"model": c.model, "width": c.width, "height": c.height, "fx": c.fx, "fy": c.fy,
         "cx": c.cx, "cy": c.cy, "fov": c.fov}
    if c.model == "unified":
        d["xi"] = c.xi
    if c.model == "polynomial":
        d["k"] = list(c.k)
    return json.dumps(d)


def main() -> int:
    camera, fields, rasters, solver, synth = _ref()
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(20190917)
    cams = cameras(camera)

    # ---- lens models: fov mask, unproject, project
    for name, c in cams.items():
        pix = np.concatenate([rng.uniform(-10, 58, size=(300, 2)),
                              np.array([[c.cx, c.cy], [0.0, 0.0], [47.0, 39.0]])])
        rays, rok = c.unproject(pix)
        pts = rng.normal(size=(300, 3))
        pts[:100, 2] = np.abs(pts[:100, 2]) + 0.1
        pts[-1] = 0.0
        pts[-2] = (0.0, 0.0, 1.0)
        px, pok = c.project(pts)
        np.savez_compressed(OUT / f"camera_{name}.npz", cam=cam_record(c), mask=c.fov_mask(),
                            pix=pix, rays=rays, rays_ok=rok, pts=pts, proj=px, proj_ok=pok)

    # ---- calibration field + calibrated image on two rigs
    for name, (c0, c1, pose) in {
        "unified": (cams["unified"],
                    camera.UnifiedCamera(width=48, height=40, fx=20.0, fy=20.5, cx=24.0, cy=19.9,
                                         fov=np.pi, xi=0.9),
                    camera.RelativePose.from_displacement((0.1, 0.0, 0.0),
                                                          rotvec=(0.0, 0.03, 0.01))),
        "kb": (cams["kb"], cams["kb"],
               camera.RelativePose.from_displacement((0.064, 0, 0), rotvec=(0.002, 0.004, 0.001))),
    }.items():
        rig = camera.StereoRig(c0, c1, pose)
        cal, cok = fields.generate_calibration_field(rig)
        i1 = rng.random((c1.height, c1.width)).astype(np.float32).astype(np.float64)
        i1c, ok, _, _ = solver.calibrate_second_image(i1, rig)
        np.savez_compressed(OUT / f"calib_{name}.npz", cam0=cam_record(c0), cam1=cam_record(c1),
                            R=pose.rotation, t=pose.translation, cal=cal, cal_ok=cok, i1=i1,
                            i1c=i1c, i1c_ok=ok)

    # ---- trajectory fields (incl. an in-image epipole and the pinhole snap)
    traj_cases = {
        "pinhole": (cams["pinhole"], (-0.1, 0.0, 0.0)),
        "unified_epipole": (cams["unified"], (0.02, -0.01, 0.08)),
        "unified": (cams["unified"], (-0.1, 0.015, 0.0)),
        "equidistant": (cams["equidistant"], (-0.1, 0.0, 0.0)),
        "kb": (cams["kb"], (-0.064, 0.001, 0.002)),
    }
    for name, (c, t) in traj_cases.items():
        rig = camera.StereoRig(c, c, camera.RelativePose(np.eye(3), np.array(t, dtype=float)))
        for eps in (0.1, 0.05):
            d, ok = fields.generate_trajectory_field(rig, epsilon_scale=eps)
            np.savez_compressed(OUT / f"traj_{name}_{eps}.npz", cam=cam_record(c),
                                t=np.array(t, dtype=float), eps=eps, dirs=d, ok=ok)

    # ---- bicubic sampling with every fallback branch
    for C in (1, 2):
        f = rng.normal(size=(12, 15) if C == 1 else (12, 15, 2))
        m = rng.random((12, 15)) > 0.3
        pos = rng.uniform(-3.5, 17.5, size=(600, 2))
        pos[:20] = np.round(pos[:20])  # exact nodes
        pos[20, 0] = np.nan
        pos[21, 1] = np.inf
        vals, ok = rasters.sample_bicubic(f, pos, m)
        np.savez_compressed(OUT / f"bicubic_c{C}.npz", field=f, mask=m, pos=pos, vals=vals, ok=ok)

    # ---- gradient / divergence
    u = rng.normal(size=(9, 11))
    p = rng.normal(size=(9, 11, 2))
    m = rng.random((9, 11)) > 0.25
    np.savez_compressed(OUT / "graddiv.npz", u=u, p=p, mask=m, grad=rasters.gradient(u, m),
                        div=rasters.divergence(p, m))

    # ---- smoothing (incl. a tiny image for repeated reflection)
    cases = {}
    for k, (h, w, s) in enumerate([(17, 13, 1.0), (20, 24, 1.5), (3, 2, 1.0), (1, 7, 1.0)]):
        f = rng.random((h, w))
        mm = rng.random((h, w)) > 0.2
        cases[f"f{k}"] = f
        cases[f"m{k}"] = mm
        cases[f"s{k}"] = np.array(s)
        cases[f"out{k}"] = rasters.smooth_masked(f, mm, s)
    np.savez_compressed(OUT / "smooth.npz", **cases)

    # ---- pyramid + upsample (odd sizes)
    img = rng.random((37, 53))
    mm = rasters.circular_mask(37, 53, (26.0, 18.0), 20.0)
    pyr = rasters.build_pyramid(img, mm, levels=4, scale=2.0, min_width=5)
    rec = {"img": img, "mask": mm, "n": np.array(pyr.num_levels)}
    for i, (ff, mk) in enumerate(zip(pyr.fields, pyr.masks)):
        rec[f"f{i}"] = ff
        rec[f"m{i}"] = mk
    uu = rng.normal(size=pyr.masks[1].shape)
    ww = rng.normal(size=pyr.masks[1].shape + (2,))
    u2, w2 = rasters.upsample_state(uu, ww, pyr.masks[1], pyr.masks[2].shape, pyr.masks[2])
    rec.update(up_u=uu, up_w=ww, up_u_out=u2, up_w_out=w2)
    np.savez_compressed(OUT / "pyramid.npz", **rec)

    # ---- tensor + steps + one PD iteration
    h, w = 20, 24
    mk = rng.random((h, w)) > 0.15
    im = rasters.smooth_masked(rng.random((h, w)), mk, 1.0)
    params = solver.SolverParams()
    T = solver.compute_tensor(im, params.beta, params.eta, mk)
    st = solver.precondition_steps(T, mk, params)
    state = solver.SolverState(u=rng.normal(size=(h, w)), v=rng.normal(size=(h, w, 2)) * 0.1,
                               p=rng.normal(size=(h, w, 2)) * 0.4,
                               q=rng.normal(size=(h, w, 4)) * 0.3,
                               u_bar=rng.normal(size=(h, w)), v_bar=rng.normal(size=(h, w, 2)) * 0.1)
    iu = rng.normal(size=(h, w)) * 0.1
    iu[rng.random((h, w)) < 0.1] = 0.0
    rho0 = rng.normal(size=(h, w)) * 0.05
    u_om = state.u + rng.normal(size=(h, w)) * 0.05
    out = solver.primal_dual_iterate(state, T, iu, rho0, u_om, params, mk, st)
    np.savez_compressed(OUT / "pd.npz", image=im, mask=mk, T=T, sigma_p=st.sigma_p,
                        tau_u=st.tau_u, tau_v=st.tau_v, u=state.u, v=state.v, p=state.p,
                        q=state.q, u_bar=state.u_bar, v_bar=state.v_bar, iu=iu, rho0=rho0,
                        u_omega=u_om, out_u=out.u, out_v=out.v, out_p=out.p, out_q=out.q,
                        out_u_bar=out.u_bar, out_v_bar=out.v_bar)

    # ---- thresholding draws (criterion 01 style)
    n = 2000
    tau = rng.uniform(0.02, 1.0, n)
    lam = 0.7
    g = rng.uniform(-2.0, 2.0, n)
    g[rng.random(n) < 0.05] = 0.0
    rho = rng.uniform(-2.0, 2.0, n)
    uh = rng.uniform(-1.0, 1.0, n)
    np.savez_compressed(OUT / "shrink.npz", tau=tau, lam=lam, iu=g, rho=rho, u_hat=uh,
                        out=solver.thresholding_step(uh, rho, g, tau, lam))

    # ---- a rendered pair: level solve + full pyramid solve (with diagnostics)
    scene = synth.default_scene()
    c0 = camera.UnifiedCamera(width=64, height=60, fx=32.0, fy=32.0, cx=31.5, cy=29.5,
                              fov=np.pi, xi=0.9)
    c1 = camera.UnifiedCamera(width=64, height=60, fx=32.0, fy=32.0, cx=32.0, cy=29.7,
                              fov=np.pi, xi=0.9)
    pose = camera.RelativePose.from_displacement((0.1, 0.0, 0.0), rotvec=(0.0, 0.03, 0.008))
    rig = camera.StereoRig(c0, c1, pose)
    i0, _, _ = synth.render(scene, c0, supersample=2)
    i1, _, _ = synth.render(scene, c1, pose=pose, supersample=2)
    i0 = i0.astype(np.float32).astype(np.float64)
    i1 = i1.astype(np.float32).astype(np.float64)
    prm = solver.SolverParams(warp_iters=4, pd_iters=5, pyramid_levels=2, min_width=20)
    res = solver.solve_pyramid(i0, i1, rig, prm, collect_diagnostics=True)
    d = res.diagnostics
    np.savez_compressed(OUT / "pyramid_solve.npz", cam0=cam_record(c0), cam1=cam_record(c1),
                        R=pose.rotation, t=pose.translation, i0=i0, i1=i1,
                        params=json.dumps(prm.to_dict()), u=res.u, w=res.w, v=res.v,
                        mask=res.mask, i1c=res.i1_calibrated,
                        max_p=np.array(d.max_p_norm), max_q=np.array(d.max_q_norm),
                        max_du=np.array(d.max_du), mean_du=np.array(d.mean_abs_du))

    # level solve on the finest level inputs of that pair
    rig_t = fields.translation_only_rig(rig)
    dirs, tok = fields.generate_trajectory_field(rig_t, 0.1)
    lp = solver.SolverParams(warp_iters=3, pd_iters=4, pyramid_levels=1)
    di = solver.Diagnostics()
    u0 = rng.normal(size=res.mask.shape) * 0.3
    w0 = rng.normal(size=res.mask.shape + (2,)) * 0.3
    ws, ss = solver.solve_level(i0, res.i1_calibrated, dirs, tok, lp, res.mask,
                                solver.WarpState(u=u0.copy(), w=w0.copy()), di)
    np.savez_compressed(OUT / "level_solve.npz", i0=i0, i1=res.i1_calibrated, dirs=dirs,
                        tok=tok, mask=res.mask, u0=u0, w0=w0, params=json.dumps(lp.to_dict()),
                        u=ws.u, w=ws.w, v=ss.v, p=ss.p, q=ss.q,
                        max_p=np.array(di.max_p_norm), max_q=np.array(di.max_q_norm),
                        max_du=np.array(di.max_du), mean_du=np.array(di.mean_abs_du))
    # ---- renderer (GPU input generator) on every primitive / texture kind
    sc = synth.default_scene()
    extra = synth.Scene(primitives=(
        synth.Plane(point=(0.0, 0.0, 2.0), normal=(0.1, 0.0, -1.0),
                    texture=synth.Checkerboard(period=0.3)),
        synth.Sphere(center=(-0.3, 0.2, 1.2), radius=0.3,
                     texture=synth.SineGrating(wavelength=0.2, direction=(1.0, 1.0, 0.0))),
        synth.Box(lo=(0.2, -0.5, 0.9), hi=(0.6, -0.1, 1.4),
                  texture=synth.ValueNoise(scale=0.1, octaves=2, seed=3))))
    rec = {}
    k = 0
    for scene, c, pose_, ss in [
            (sc, cams["unified"], None, 2),
            (sc, cams["kb"], camera.RelativePose.from_displacement((0.1, 0, 0), rotvec=(0, .03, 0)), 1),
            (extra, cams["pinhole"], None, 3),
            (synth.reseed_scene(sc, 5), cams["equidistant"], None, 1)]:
        img, dep, hit = synth.render(scene, c, pose=pose_, supersample=ss)
        rec[f"img{k}"] = img
        rec[f"depth{k}"] = dep
        rec[f"hit{k}"] = hit
        k += 1
    np.savez_compressed(OUT / "render.npz", **rec)

    # ---- post-solve depth: compose_with_calibration, depth_from_correspondence,
    # triangulate_midpoint (own rng: the fixtures above keep their streams)
    from fisheyestereo import evaluate
    rd = np.random.default_rng(1909)
    for name, (c0, c1, pose) in {
        "unified": (cams["unified"],
                    camera.UnifiedCamera(width=48, height=40, fx=20.0, fy=20.5, cx=24.0, cy=19.9,
                                         fov=np.pi, xi=0.9),
                    camera.RelativePose.from_displacement((0.1, 0.0, 0.0),
                                                          rotvec=(0.0, 0.03, 0.01))),
        "kb": (cams["kb"], cams["kb"],
               camera.RelativePose.from_displacement((0.064, 0.01, 0.0),
                                                     rotvec=(0.002, 0.004, 0.001))),
    }.items():
        rig = camera.StereoRig(c0, c1, pose)
        cal, cok = fields.generate_calibration_field(rig)
        wv = rd.uniform(-4.0, 1.0, size=(c0.height, c0.width, 2))
        wv[..., 1] *= 0.2
        full, fok = fields.compose_with_calibration(wv, cal, cok)
        valid = fok & c0.fov_mask()
        depth, dok = evaluate.depth_from_correspondence(rig, full, valid)
        depth_c, dok_c = evaluate.depth_from_correspondence(rig, full, valid, depth_cap=2.0)
        pts = rd.uniform(-1.5, 1.5, size=(400, 3))
        pts[:, 2] = rd.uniform(0.3, 5.0, size=400)
        x0, ok0 = rig.cam0.project(pts)
        x1, ok1 = rig.cam1.project(pose.transform(pts))
        sel = ok0 & ok1
        x0, x1 = x0[sel], x1[sel]
        x1[:5] = x0[:5]  # zero-disparity / parallel-ray cases
        x1[5:10] += rd.normal(size=(5, 2)) * 3.0  # inconsistent pairs
        tri, tok = camera.triangulate_midpoint(rig, x0, x1)
        np.savez_compressed(OUT / f"depth_{name}.npz", cam0=cam_record(c0), cam1=cam_record(c1),
                            R=pose.rotation, t=pose.translation, cal=cal, cal_ok=cok, wv=wv,
                            full=full, full_ok=fok, valid=valid, depth=depth, depth_ok=dok,
                            depth_cap2=depth_c, depth_cap2_ok=dok_c, x0=x0, x1=x1, tri=tri,
                            tri_ok=tok)

    # ---- ground truth of a rendered pair (synth.make_ground_truth)
    rec = {}
    for k, (scene, c0, c1, pose) in enumerate([
            (synth.default_scene(), cams["unified"],
             camera.UnifiedCamera(width=48, height=40, fx=20.0, fy=20.5, cx=24.0, cy=19.9,
                                  fov=np.pi, xi=0.9),
             camera.RelativePose.from_displacement((0.1, 0.02, 0.0), rotvec=(0.0, 0.03, 0.01))),
            (extra, cams["kb"], cams["kb"],
             camera.RelativePose.from_displacement((0.3, 0.0, 0.05), rotvec=(0.01, 0.0, 0.02)))]):
        rig = camera.StereoRig(c0, c1, pose)
        gt = synth.make_ground_truth(scene, rig)
        rec[f"cam0_{k}"] = cam_record(c0)
        rec[f"cam1_{k}"] = cam_record(c1)
        rec[f"R_{k}"] = pose.rotation
        rec[f"t_{k}"] = pose.translation
        rec[f"depth0_{k}"] = gt.depth0
        rec[f"corr_{k}"] = gt.correspondence
        rec[f"covis_{k}"] = gt.covisibility
    np.savez_compressed(OUT / "ground_truth.npz", **rec)

    # ---- evaluate.make_report and the PFM writer
    from fisheyestereo import formats
    import tempfile
    re_ = np.random.default_rng(98)
    h, w = 37, 53
    w_gt = re_.normal(size=(h, w, 2)) * 5.0
    w_est = w_gt + re_.normal(size=(h, w, 2)) * re_.choice([0.3, 2.0, 8.0], size=(h, w, 1))
    valid = re_.random((h, w)) > 0.2
    d_gt = re_.uniform(0.5, 6.0, size=(h, w))
    d_est = d_gt + re_.normal(size=(h, w)) * 0.1
    d_est[::7, ::5] = np.nan
    d_est[1::9, ::4] = -1.0
    taus = (0.5, 1.0, 3.0, 5.0)
    rep = evaluate.make_report(w_est, w_gt, valid, taus, d_est, d_gt)
    rep0 = evaluate.make_report(w_est, w_gt, valid & False, taus)
    err = evaluate.correspondence_error(w_est, w_gt, valid)
    with tempfile.TemporaryDirectory() as td:
        formats.write_pfm(f"{td}/a.pfm", d_gt)
        formats.write_vector_pfm(f"{td}/b.pfm", w_gt, third=valid)
        pfm1 = np.frombuffer(open(f"{td}/a.pfm", "rb").read(), dtype=np.uint8)
        pfm3 = np.frombuffer(open(f"{td}/b.pfm", "rb").read(), dtype=np.uint8)
    np.savez_compressed(OUT / "report.npz", w_est=w_est, w_gt=w_gt, valid=valid, d_est=d_est,
                        d_gt=d_gt, taus=np.array(taus), err=err, report=rep.to_json(),
                        report_empty=rep0.to_json(), pfm1=pfm1, pfm3=pfm3)

    # ---- rig JSON schema (camera.rig_to_dict / rig_from_dict)
    rigs = [camera.StereoRig(cams["kb"], cams["unified"],
                             camera.RelativePose.from_displacement((0.1, 0.02, -0.01),
                                                                   rotvec=(0.01, -0.02, 0.03))),
            camera.StereoRig(cams["pinhole"], cams["equidistant"],
                             camera.RelativePose.from_displacement((-0.05, 0.0, 0.0)))]
    np.savez_compressed(OUT / "rig_json.npz",
                        rigs=np.array([json.dumps(camera.rig_to_dict(r), sort_keys=True)
                                       for r in rigs]))

    # ---- a noisy render (sensor noise drawn from numpy's default_rng(seed))
    img, dep, hit = synth.render(synth.default_scene(), cams["unified"], noise_sigma=0.02,
                                 noise_seed=23, supersample=2)
    np.savez_compressed(OUT / "render_noise.npz", img=img, hit=hit)

    # ---- epipolar curve tracing (acceptance criterion 04 helpers)
    rt = np.random.default_rng(404)
    rec = {}
    for k, (c, t) in enumerate([(cams["unified"], (-0.1, 0.015, 0.0)),
                                (cams["kb"], (-0.064, 0.001, 0.002))]):
        rigk = camera.StereoRig(c, c, camera.RelativePose(np.eye(3), np.array(t, dtype=float)))
        d, ok = fields.generate_trajectory_field(rigk)
        starts = np.stack([rt.uniform(2, c.width - 3, 40), rt.uniform(2, c.height - 3, 40)], -1)
        verts, alive = fields.trace_epipolar_curves(d, ok, starts, 15.0, 0.7)
        one = fields.trace_epipolar_curve(d, ok, starts[0], 9.0, 0.5)
        rig_c = camera.StereoRig(c, c, camera.RelativePose.from_displacement(
            (0.1, 0.02, 0.0), rotvec=(0.0, 0.03, 0.01)))
        x0 = np.array([c.cx + 3.0, c.cy - 2.0])
        depths = np.geomspace(0.3, 50.0, 25)
        sw, swok = fields.depth_swept_curve(rig_c, x0, depths)
        rec.update({f"cam_{k}": cam_record(c), f"t_{k}": np.array(t, dtype=float),
                    f"dirs_{k}": d, f"ok_{k}": ok, f"starts_{k}": starts, f"verts_{k}": verts,
                    f"alive_{k}": alive, f"one_{k}": one, f"R_{k}": rig_c.pose.rotation,
                    f"tr_{k}": rig_c.pose.translation, f"x0_{k}": x0, f"depths_{k}": depths,
                    f"swept_{k}": sw, f"swept_ok_{k}": swok})
    np.savez_compressed(OUT / "trace.npz", **rec)

    total = sum(f.stat().st_size for f in OUT.glob("*.npz"))
    print(f"wrote {len(list(OUT.glob('*.npz')))} fixtures, {total / 1024:.0f} KiB -> {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
