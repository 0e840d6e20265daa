"""Where does fp32 lose parity at N=50? (diagnostic study, CPU, build container)

Runs the pinned fp64 oracle on the reference acceptance pair (default_rig 400^2,
N=50, K=10, du_max=0.1) with float32 rounding injected at chosen points and
reports |du| statistics against the pure fp64 run.
"""
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
from oracle import fs_oracle as O  # noqa: E402

f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
_LEVEL = {"coarse": False}


def run(i0, i1, rig, prm, mode):
    orig_cycle, orig_lin, orig_level = O.pd_cycle, O.linearize, O.level_solve
    orig_T, orig_st = O.edge_tensor, O.step_sizes

    def cycle(s, *a, **k):
        s = orig_cycle(s, *a, **k)
        if "coarse32" in mode and _LEVEL["coarse"]:  # float32 state on the coarse levels only
            s = O.PDState(*(f32(getattr(s, f)) for f in ("u", "v", "p", "q", "u_bar", "v_bar")))
        if "state" in mode:
            s = O.PDState(*(f32(getattr(s, f)) for f in ("u", "v", "p", "q", "u_bar", "v_bar")))
        if "pq" in mode:  # only the duals stored as float32
            s = O.PDState(u=s.u, v=s.v, p=f32(s.p), q=f32(s.q), u_bar=s.u_bar, v_bar=s.v_bar)
        if "vv" in mode:  # only the second-order primal v, v_bar as float32
            s = O.PDState(u=s.u, v=f32(s.v), p=s.p, q=s.q, u_bar=s.u_bar, v_bar=f32(s.v_bar))
        return s

    def tensor(*a, **k):
        T = orig_T(*a, **k)
        return f32(T) if "consts" in mode or ("coarse32" in mode and _LEVEL["coarse"]) else T

    def steps(*a, **k):
        st = orig_st(*a, **k)
        if "consts" in mode or ("coarse32" in mode and _LEVEL["coarse"]):
            st = O.Steps(sigma_p=f32(st.sigma_p), sigma_q=st.sigma_q, tau_u=f32(st.tau_u),
                         tau_v=f32(st.tau_v))
        return st

    def lin(i0_, i1_, traj, tok, mask, w):
        c32 = "coarse32" in mode and _LEVEL["coarse"]
        if "w" in mode.split("+") or c32:
            w = f32(w)
        out = orig_lin(i0_, i1_, traj, tok, mask, w)
        if "gath" in mode or c32:
            i1w, wok, dirs, dok, iu, rho0 = out
            out = (f32(i1w), wok, f32(dirs), dok, f32(iu), f32(rho0))
        return out

    def level(i0_, i1_, traj, tok, prm_, mask, u0, w0, tr=None):
        _LEVEL["coarse"] = mask.shape != i0.shape
        if "coarse32" in mode and _LEVEL["coarse"]:
            u0, w0 = f32(u0), f32(w0)
        out = orig_level(i0_, i1_, traj, tok, prm_, mask, u0, w0, tr)
        if "coarse32" in mode and _LEVEL["coarse"]:
            out = (f32(out[0]), f32(out[1]), out[2])
        return out

    O.pd_cycle, O.linearize = cycle, lin
    O.level_solve = level
    O.edge_tensor, O.step_sizes = tensor, steps
    try:
        return O.pyramid_solve(i0, i1, rig, prm)
    finally:
        O.pd_cycle, O.linearize = orig_cycle, orig_lin
        O.level_solve = orig_level
        O.edge_tensor, O.step_sizes = orig_T, orig_st


def main():
    import os
    from fisheyestereo import synth
    modes = sys.argv[1:] or ["", "state", "w", "gath", "state+w+gath"]
    N = 50
    prm = SimpleNamespace(lam=5.0, alpha0=17.0, alpha1=1.2, beta=9.0, eta=0.85, warp_iters=N,
                          pd_iters=10, du_max=0.1, pyramid_levels=5, pyramid_scale=2.0,
                          min_width=50, epsilon_scale=0.1, tensor_sigma=1.0, theta=1.0)
    if os.environ.get("STUDY") == "c3":  # the C3 pair and rig, reference defaults
        import bench
        from fisheyestereo import camera
        d = np.load(ROOT / "tests" / "golden" / "c3_pair.npz")
        i0, i1 = d["i0"].astype(np.float64), d["i1"].astype(np.float64)
        cam = camera.UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5,
                                   cy=511.5, fov=np.pi, xi=0.9)
        rig = camera.StereoRig(cam, cam, camera.RelativePose.from_displacement(
            (0.08, 0.02, 0.03), rotvec=(0.01, 0.03, -0.02)))
        prm.du_max = 0.2
    else:
        rig = synth.default_rig()
        sc = synth.default_scene()
        i0 = f32(synth.render(sc, rig.cam0, supersample=2)[0])
        i1 = f32(synth.render(sc, rig.cam1, pose=rig.pose, supersample=2)[0])
    ref = run(i0, i1, rig, prm, "")
    for m in modes[1:] if modes[0] == "" else modes:
        s = run(i0, i1, rig, prm, m)
        e = np.abs(s.u - ref.u)[ref.mask]
        print(f"{m:14s} median {np.median(e):.2e} p99 {np.percentile(e, 99):.2e} "
              f"max {e.max():.2e}", flush=True)


if __name__ == "__main__":
    main()
