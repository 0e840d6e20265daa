"""Calibration and trajectory fields on the GPU (reference fields.py:34-182).

Both fields are computed in fp64 by libfsb200 (K1/K2); the trajectory
directions are stored as fp32 on the device and returned here as float64.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _dev, _ext
from .camera import RelativePose, StereoRig


def translation_only_rig(rig) -> StereoRig:
    """Residual rig after the calibration warp: (cam0, cam0, (I, R^T t)) (fields.py:159-167)."""
    t_res = rig.pose.rotation.T @ rig.pose.translation
    return StereoRig(rig.cam0, rig.cam0, RelativePose(np.eye(3), t_res))


def generate_calibration_field(rig):
    """Rotation + intrinsics flow x1 = x + field[x] and its validity (fields.py:34-45)."""
    L = _ext.lib()
    rs = _ext.rig_struct(rig)
    h, w = rs.cam0.height, rs.cam0.width
    field = _dev.empty((h, w, 2), torch.float64)
    ok = _dev.empty((h, w), torch.uint8)
    s = _dev.scratch(256)
    _ext.check(L.fsb_calibration_field(C.byref(rs), _dev.ptr(field), _dev.ptr(ok), _dev.ptr(s),
                                       s.numel(), _dev.stream_ptr()), "calibration_field")
    return _dev.download(field), _dev.download(ok, bool)


def trajectory_field_device(cam, t, epsilon_scale: float = 0.1, depth: float = 1.0,
                            dtype=torch.float32):
    """Device tensors (dirs (H,W,2) `dtype`, ok (H,W) u8) for the rig (cam, cam, (I, t)).
    Computed in fp64 either way; float32 storage is the fp32 path's field."""
    L = _ext.lib()
    cs = _ext.camera_struct(cam)
    tt = (C.c_double * 3)(*[float(v) for v in np.asarray(t, dtype=np.float64).reshape(3)])
    dirs = _dev.empty((cs.height, cs.width, 2), dtype)
    ok = _dev.empty((cs.height, cs.width), torch.uint8)
    s = _dev.scratch(L.fsb_trajectory_scratch_bytes(C.byref(cs)))
    fn = L.fsb_trajectory_field if dtype == torch.float32 else L.fsb_trajectory_field_f64
    _ext.check(fn(C.byref(cs), tt, float(epsilon_scale), float(depth), _dev.ptr(dirs),
                  _dev.ptr(ok), _dev.ptr(s), s.numel(), _dev.stream_ptr()),
               "generate_trajectory_field")
    return dirs, ok


def generate_trajectory_field(rig, epsilon_scale: float = 0.1, depth: float = 1.0):
    """Unit epipolar-curve tangents per pixel (fields.py:48-108).

    Requires a translation-only rig; raises ValueError for a rotated rig or a
    zero baseline like the reference.
    """
    R = np.asarray(rig.pose.rotation, dtype=np.float64)
    if np.max(np.abs(R - np.eye(3))) > 1e-9:
        raise ValueError("trajectory field needs a rotation-free rig; "
                         "apply the calibration field first")
    dirs, ok = trajectory_field_device(rig.cam0, rig.pose.translation, epsilon_scale, depth,
                                       torch.float64)
    return _dev.download(dirs), _dev.download(ok, bool)


def calibrate_second_image(i1, rig, mask1=None):
    """Warp image 1 by the calibration field once (solver.py:389-398).

    Returns (i1c, ok, cal, cal_ok) like the reference.
    """
    L = _ext.lib()
    rs = _ext.rig_struct(rig)
    i1a = np.asarray(i1, dtype=np.float64)
    if i1a.shape != (rs.cam1.height, rs.cam1.width):
        raise ValueError("image 1 does not match camera 1 dimensions")
    d1 = _dev.upload(i1a)
    dm1 = _dev.upload(np.asarray(mask1, dtype=bool), torch.uint8) if mask1 is not None else None
    h, w = rs.cam0.height, rs.cam0.width
    i1c = _dev.empty((h, w))
    ok = _dev.empty((h, w), torch.uint8)
    s = _dev.scratch(L.fsb_calibrate_scratch_bytes(C.byref(rs)))
    _ext.check(L.fsb_calibrate_second_image(C.byref(rs), _dev.ptr(d1), _dev.ptr(dm1),
                                            _dev.ptr(i1c), _dev.ptr(ok), _dev.ptr(s), s.numel(),
                                            _dev.stream_ptr()), "calibrate_second_image")
    cal, cal_ok = generate_calibration_field(rig)
    return _dev.download(i1c), _dev.download(ok, bool), cal, cal_ok


def compose_with_calibration(w, cal_field, cal_valid):
    """Solver warp (calibrated frame) -> full camera-1 correspondence
    (fields.py:170-182): (x + w) + calibration(x + w), f64 bicubic of the
    calibration field under `cal_valid`; 0 where that sample is invalid."""
    L = _ext.lib()
    ok_in = np.asarray(cal_valid, dtype=bool)
    h, wd = ok_in.shape
    wv = np.asarray(w, dtype=np.float64)
    cal = np.asarray(cal_field, dtype=np.float64)
    if wv.shape != (h, wd, 2) or cal.shape != (h, wd, 2):
        raise ValueError("w and cal_field must be (H, W, 2) on the cal_valid grid")
    dw, dc = _dev.upload(wv, torch.float64), _dev.upload(cal, torch.float64)
    dm = _dev.upload(ok_in, torch.uint8)
    full = _dev.empty((h, wd, 2), torch.float64)
    ok = _dev.empty((h, wd), torch.uint8)
    _ext.check(L.fsb_compose_calibration(_dev.ptr(dw), _dev.ptr(dc), _dev.ptr(dm), h, wd,
                                         _dev.ptr(full), _dev.ptr(ok), _dev.stream_ptr()),
               "compose_with_calibration")
    return _dev.download(full), _dev.download(ok, bool)


def trace_epipolar_curves(dirs, valid, starts, length: float, step: float):
    """Euler-integrate the direction field from several start pixels at once
    (fields.py:111-139), one GPU thread per start. Returns (vertices, alive):
    vertices (n_starts, n_steps + 1, 2) (NaN once a trace left the valid
    region), alive flags."""
    import math
    if step <= 0:
        raise ValueError("step must be positive")
    L = _ext.lib()
    d = np.asarray(dirs, dtype=np.float64)
    v = np.asarray(valid, dtype=bool)
    h, w = v.shape
    st = np.atleast_2d(np.asarray(starts, dtype=np.float64))
    n = st.shape[0]
    n_steps = max(int(math.ceil(length / step)), 0)
    dd = _dev.upload(d, torch.float64)
    dv = _dev.upload(v, torch.uint8)
    ds = _dev.upload(st.reshape(n, 2), torch.float64)
    verts = _dev.empty((max(n, 1), n_steps + 1, 2), torch.float64)
    alive = _dev.empty((max(n, 1), n_steps + 1), torch.uint8)
    _ext.check(L.fsb_trace_epipolar_curves(_dev.ptr(dd), _dev.ptr(dv), h, w, _dev.ptr(ds), n,
                                           n_steps, float(length), float(step), _dev.ptr(verts),
                                           _dev.ptr(alive), _dev.stream_ptr()),
               "trace_epipolar_curves")
    return _dev.download(verts)[:n], _dev.download(alive, bool)[:n]


def trace_epipolar_curve(dirs, valid, start, length: float, step: float):
    """Polyline (k, 2) traced from one pixel, truncated at the mask edge
    (fields.py:142-146)."""
    verts, alive = trace_epipolar_curves(dirs, valid, [start], length, step)
    return verts[0][alive[0]]


def depth_swept_curve(rig, x0, depths):
    """Exact epipolar curve of a pixel: its ray projected at each depth
    (fields.py:149-156), on the GPU lens models."""
    from .camera import project, unproject
    ray, ok0 = unproject(rig.cam0, np.asarray(x0, dtype=np.float64))
    if not bool(np.all(ok0)):
        raise ValueError(f"pixel {x0} is outside the camera-0 field of view")
    depths = np.asarray(depths, dtype=np.float64)
    pts = rig.pose.transform(ray[None, :] * depths[:, None])
    return project(rig.cam1, pts)
