"""Post-solve depth (reference evaluate.py:101-114), computed on the GPU.

SURVEY §8(f) row 1: turns the solver's correspondence into metric depth along
camera-0 rays. NumPy in, NumPy out, like the reference function.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _dev, _ext


def depth_from_correspondence(rig, corr, valid, depth_cap: float = 1e6):
    """Triangulate a correspondence field into depth along camera-0 rays
    (evaluate.py:101-114): x1 = x + corr, midpoint triangulation (min_angle
    1e-6), ok &= valid, depth capped at `depth_cap`, 0 where not ok."""
    L = _ext.lib()
    v = np.asarray(valid, dtype=bool)
    h, w = v.shape
    c = np.asarray(corr, dtype=np.float64)
    if c.shape != (h, w, 2):
        raise ValueError("corr must be (H, W, 2) on the valid grid")
    rs = _ext.rig_struct(rig)
    dc = _dev.upload(c, torch.float64)
    dv = _dev.upload(v, torch.uint8)
    depth = _dev.empty((h, w), torch.float64)
    ok = _dev.empty((h, w), torch.uint8)
    s = _dev.scratch(L.fsb_triangulate_scratch_bytes())
    _ext.check(L.fsb_depth_from_correspondence(C.byref(rs), _dev.ptr(dc), _dev.ptr(dv), h, w,
                                               float(depth_cap), _dev.ptr(depth), _dev.ptr(ok),
                                               _dev.ptr(s), s.numel(), _dev.stream_ptr()),
               "depth_from_correspondence")
    return _dev.download(depth), _dev.download(ok, bool)


def depth_error_map(depth_est, depth_gt, valid):
    """|depth_est - depth_gt| in meters, 0 outside `valid` (evaluate.py:117-120)."""
    return np.where(valid, np.abs(np.asarray(depth_est) - np.asarray(depth_gt)), 0.0)
