"""ctypes binding of libfsb200.so (include/fsb200.h).

The library is the only compute path: if it is missing, or no CUDA device is
present when a compute entry point is called, this module raises — there is no
CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# FSB_LIB=checked loads the checked debug build (build.py --checked)
LIB_PATH = Path(__file__).resolve().parent / (
    "libfsb200_checked.so" if os.environ.get("FSB_LIB") == "checked" else "libfsb200.so")

FSB_OK = 0
FSB_EINVAL = -1
FSB_ENOSPC = -2
FSB_EDOMAIN = -3

CAM_MODELS = {"pinhole": 0, "unified": 1, "polynomial": 2}

# Every symbol declared in include/fsb200.h (checked by tests/test_abi.py).
EXPORTED = (
    "fsb_fov_mask", "fsb_fov_mask_scratch_bytes", "fsb_unproject", "fsb_project",
    "fsb_unproject_scratch_bytes", "fsb_calibration_field", "fsb_calibrate_second_image",
    "fsb_calibrate_scratch_bytes", "fsb_trace_epipolar_curves", "fsb_compose_calibration", "fsb_triangulate_midpoint",
    "fsb_triangulate_scratch_bytes", "fsb_depth_from_correspondence", "fsb_trajectory_field", "fsb_trajectory_field_f64", "fsb_trajectory_scratch_bytes",
    "fsb_sample_bicubic", "fsb_gradient", "fsb_divergence", "fsb_smooth_masked",
    "fsb_smooth_scratch_bytes", "fsb_pyramid_shapes", "fsb_downsample_area",
    "fsb_upsample_state", "fsb_compute_tensor", "fsb_precondition_steps", "fsb_level_partials", "fsb_level_tiles", "fsb_level_setup", "fsb_warp_linearize",
    "fsb_pd_iterate", "fsb_thresholding_step", "fsb_warp_finish", "fsb_solve_level", "fsb_diag_counts",
    "fsb_solve_pyramid_workspace_bytes", "fsb_solve_pyramid",
    "fsb_solve_pyramid_f64_workspace_bytes", "fsb_solve_pyramid_f64", "fsb_render", "fsb_graph_create", "fsb_graph_create_f64", "fsb_graph_launch", "fsb_graph_destroy", "fsb_graph_early_event", "fsb_stream_wait_event",
    "fsb_warp_linearize_f64_scratch_bytes", "fsb_warp_linearize_f64",
    "fsb_phase_timer_create", "fsb_phase_timer_read", "fsb_phase_timer_destroy",
    "fsb_solve_pyramid_f64_timed",
    "fsb_ground_truth", "fsb_error_report", "fsb_error_report_scratch_bytes", "fsb_version",
)


class FsbCamera(C.Structure):
    _fields_ = [("model", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("reserved", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("fov", C.c_double),
                ("xi", C.c_double), ("k", C.c_double * 4)]


class FsbRig(C.Structure):
    _fields_ = [("cam0", FsbCamera), ("cam1", FsbCamera), ("rotation", C.c_double * 9),
                ("translation", C.c_double * 3)]


class FsbParams(C.Structure):
    _fields_ = [("lam", C.c_double), ("alpha0", C.c_double), ("alpha1", C.c_double),
                ("beta", C.c_double), ("eta", C.c_double), ("warp_iters", C.c_int32),
                ("pd_iters", C.c_int32), ("du_max", C.c_double),
                ("pyramid_levels", C.c_int32), ("min_width", C.c_int32),
                ("pyramid_scale", C.c_double), ("epsilon_scale", C.c_double),
                ("tensor_sigma", C.c_double), ("theta", C.c_double),
                ("regularizer", C.c_int32), ("reserved", C.c_int32), ("huber_eps", C.c_double)]


class FsbDiag(C.Structure):
    _fields_ = [("max_p_norm", C.c_void_p), ("max_q_norm", C.c_void_p),
                ("max_du", C.c_void_p), ("mean_abs_du", C.c_void_p),
                ("max_du_f64", C.c_void_p)]


class FsbLevel(C.Structure):
    _fields_ = [("h", C.c_int32), ("w", C.c_int32)] + [
        (name, C.c_void_p) for name in (
            "i0", "i1", "mask", "traj", "traj_ok", "tensor", "steps", "u", "u_bar", "v",
            "v_bar", "p", "q", "wv", "u_omega", "iu", "rho0", "i1w", "i1w_ok", "dirs",
            "dir_ok", "partials", "state_b", "packed", "full16", "maskf", "tiles")]


class FsbPrim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tex_kind", C.c_int32), ("octaves", C.c_int32),
                ("reserved", C.c_int32), ("seed", C.c_int64), ("geom", C.c_double * 7),
                ("tex", C.c_double * 8)]


class FsbError(RuntimeError):
    """A CUDA launch failed inside libfsb200."""


_lib = None


def lib() -> C.CDLL:
    """Load libfsb200.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1909_07545_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp, sz, i32, i64, dbl = C.c_void_p, C.c_size_t, C.c_int32, C.c_int64, C.c_double
        P = C.POINTER
        sig = {
            "fsb_fov_mask": (C.c_int, [P(FsbCamera), vp, vp, sz, vp]),
            "fsb_fov_mask_scratch_bytes": (sz, [P(FsbCamera)]),
            "fsb_unproject": (C.c_int, [P(FsbCamera), vp, i64, vp, vp, vp, sz, vp]),
            "fsb_project": (C.c_int, [P(FsbCamera), vp, i64, vp, vp, vp]),
            "fsb_unproject_scratch_bytes": (sz, []),
            "fsb_calibration_field": (C.c_int, [P(FsbRig), vp, vp, vp, sz, vp]),
            "fsb_calibrate_second_image": (C.c_int, [P(FsbRig), vp, vp, vp, vp, vp, sz, vp]),
            "fsb_calibrate_scratch_bytes": (sz, [P(FsbRig)]),
            "fsb_compose_calibration": (C.c_int, [vp, vp, vp, i32, i32, vp, vp, vp]),
            "fsb_trace_epipolar_curves": (C.c_int, [vp, vp, i32, i32, vp, i64, i32, dbl, dbl, vp,
                                                    vp, vp]),
            "fsb_triangulate_midpoint": (C.c_int, [P(FsbRig), vp, vp, i64, dbl, vp, vp, vp, sz,
                                                   vp]),
            "fsb_triangulate_scratch_bytes": (sz, []),
            "fsb_depth_from_correspondence": (C.c_int, [P(FsbRig), vp, vp, i32, i32, dbl, vp, vp,
                                                        vp, sz, vp]),
            "fsb_trajectory_field": (C.c_int, [P(FsbCamera), P(C.c_double), dbl, dbl, vp, vp,
                                               vp, sz, vp]),
            "fsb_trajectory_field_f64": (C.c_int, [P(FsbCamera), P(C.c_double), dbl, dbl, vp, vp,
                                               vp, sz, vp]),
            "fsb_trajectory_scratch_bytes": (sz, [P(FsbCamera)]),
            "fsb_sample_bicubic": (C.c_int, [vp, i32, i32, i32, vp, vp, i64, vp, vp, i32, vp]),
            "fsb_gradient": (C.c_int, [vp, vp, i32, i32, vp, vp]),
            "fsb_divergence": (C.c_int, [vp, vp, i32, i32, vp, vp]),
            "fsb_smooth_masked": (C.c_int, [vp, vp, i32, i32, dbl, vp, vp, sz, vp]),
            "fsb_smooth_scratch_bytes": (sz, [i32, i32]),
            "fsb_pyramid_shapes": (C.c_int, [i32, i32, i32, dbl, i32, P(C.c_int32), i32]),
            "fsb_downsample_area": (C.c_int, [vp, vp, i32, i32, vp, vp, i32, i32, vp]),
            "fsb_upsample_state": (C.c_int, [vp, vp, vp, i32, i32, vp, i32, i32, vp, vp, vp]),
            "fsb_compute_tensor": (C.c_int, [vp, vp, i32, i32, dbl, dbl, vp, vp, sz, vp]),
            "fsb_precondition_steps": (C.c_int, [vp, vp, i32, i32, P(FsbParams), vp, vp, sz,
                                                 vp]),
            "fsb_level_partials": (sz, [i32, i32]),
            "fsb_level_tiles": (sz, [i32, i32]),
            "fsb_level_setup": (C.c_int, [P(FsbLevel), P(FsbParams), vp, sz, vp]),
            "fsb_warp_linearize": (C.c_int, [P(FsbLevel), vp]),
            "fsb_pd_iterate": (C.c_int, [P(FsbLevel), P(FsbParams), i32, vp, vp, vp]),
            "fsb_thresholding_step": (C.c_int, [vp, vp, vp, vp, dbl, i64, vp, vp]),
            "fsb_warp_finish": (C.c_int, [P(FsbLevel), P(FsbParams), vp, vp, vp]),
            "fsb_solve_level": (C.c_int, [P(FsbLevel), P(FsbParams), P(FsbDiag), i64, i64, vp,
                                          sz, vp]),
            "fsb_diag_counts": (C.c_int, [i32, i32, P(FsbParams), P(C.c_int64), P(C.c_int64)]),
            "fsb_solve_pyramid_workspace_bytes": (sz, [P(FsbRig), P(FsbParams)]),
            "fsb_solve_pyramid": (C.c_int, [P(FsbRig), P(FsbParams), vp, vp, vp, vp, vp, sz,
                                            vp, vp, vp, vp, vp, P(FsbDiag), vp]),
            "fsb_solve_pyramid_f64_workspace_bytes": (sz, [P(FsbRig), P(FsbParams)]),
            "fsb_solve_pyramid_f64": (C.c_int, [P(FsbRig), P(FsbParams), vp, vp, vp, vp, vp, sz,
                                                vp, vp, vp, vp, vp, P(FsbDiag), vp]),
            "fsb_render": (C.c_int, [P(FsbCamera), P(C.c_double), P(C.c_double), vp, i32, i32,
                                     vp, vp, vp, vp]),
            "fsb_graph_create": (C.c_int, [P(FsbRig), P(FsbParams), vp, vp, vp, vp, vp, sz, vp,
                                           vp, vp, vp, vp, P(FsbDiag), vp, P(C.c_void_p),
                                           P(C.c_int64)]),
            "fsb_ground_truth": (C.c_int, [P(FsbRig), vp, i32, dbl, vp, vp, vp, vp, sz, vp]),
            "fsb_error_report": (C.c_int, [vp, vp, vp, i64, vp, i32, vp, vp, vp, vp, vp, sz, vp]),
            "fsb_error_report_scratch_bytes": (sz, [i64]),
            "fsb_graph_create_f64": (C.c_int, [P(FsbRig), P(FsbParams), vp, vp, vp, vp, vp, sz,
                                               vp, vp, vp, vp, vp, P(FsbDiag), vp,
                                               P(C.c_void_p), P(C.c_int64)]),
            "fsb_warp_linearize_f64_scratch_bytes": (sz, [i32, i32]),
            "fsb_warp_linearize_f64": (C.c_int, [i32, i32] + [vp] * 13 + [sz, i32, vp]),
            "fsb_phase_timer_create": (C.c_int, [i32, i32, P(C.c_void_p)]),
            "fsb_phase_timer_read": (C.c_int, [vp, P(C.c_double), P(C.c_double), P(C.c_int32),
                                               P(C.c_int32), P(C.c_int32), P(C.c_int32)]),
            "fsb_phase_timer_destroy": (C.c_int, [vp]),
            "fsb_solve_pyramid_f64_timed": (C.c_int, [P(FsbRig), P(FsbParams), vp, vp, vp, sz,
                                                      vp, vp, vp, vp, vp, vp, vp]),
            "fsb_graph_launch": (C.c_int, [vp, vp]),
            "fsb_graph_destroy": (C.c_int, [vp]),
            "fsb_graph_early_event": (C.c_void_p, [vp]),
            "fsb_stream_wait_event": (C.c_int, [vp, vp]),
            "fsb_version": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == FSB_OK:
        return
    if rc in (FSB_EINVAL, FSB_EDOMAIN):
        msg = {FSB_EINVAL: "invalid argument", FSB_EDOMAIN: "trajectory field undefined "
               "(zero baseline or rotated rig)"}[rc]
        raise ValueError(f"{what}: {msg}")
    if rc == FSB_ENOSPC:
        raise RuntimeError(f"{what}: workspace too small")
    raise FsbError(f"{what}: CUDA error {rc}")


# ---------------------------------------------------------------- conversions

def camera_struct(cam) -> FsbCamera:
    """Pack any reference-compatible camera (duck-typed on `model` and the
    CameraBase fields, camera.py:47-190) into the C struct."""
    model = getattr(cam, "model", None)
    if model not in CAM_MODELS:
        raise ValueError(f"unknown camera model {model!r}")
    c = FsbCamera()
    c.model = CAM_MODELS[model]
    c.width = int(cam.width)
    c.height = int(cam.height)
    c.fx, c.fy, c.cx, c.cy, c.fov = (float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                                     float(cam.fov))
    c.xi = float(getattr(cam, "xi", 0.0)) if model == "unified" else 0.0
    k = tuple(getattr(cam, "k", (1.0, 0.0, 0.0, 0.0))) if model == "polynomial" else (0, 0, 0, 0)
    for i in range(4):
        c.k[i] = float(k[i])
    return c


def rig_struct(rig) -> FsbRig:
    r = FsbRig()
    r.cam0 = camera_struct(rig.cam0)
    r.cam1 = camera_struct(rig.cam1)
    R = np.asarray(rig.pose.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(rig.pose.translation, dtype=np.float64).reshape(3)
    for i in range(9):
        r.rotation[i] = float(R[i])
    for i in range(3):
        r.translation[i] = float(t[i])
    return r


def params_struct(p) -> FsbParams:
    s = FsbParams()
    s.lam, s.alpha0, s.alpha1 = float(p.lam), float(p.alpha0), float(p.alpha1)
    s.beta, s.eta = float(p.beta), float(p.eta)
    s.warp_iters, s.pd_iters = int(p.warp_iters), int(p.pd_iters)
    s.du_max = float(p.du_max)
    s.pyramid_levels, s.min_width = int(p.pyramid_levels), int(p.min_width)
    s.pyramid_scale = float(p.pyramid_scale)
    s.epsilon_scale = float(p.epsilon_scale)
    s.tensor_sigma = float(p.tensor_sigma)
    s.theta = float(p.theta)
    s.regularizer = {"tgv": 0, "tv": 1, "huber": 2}[getattr(p, "regularizer", "tgv")]
    s.huber_eps = float(getattr(p, "huber_eps", 0.05))
    return s
