"""Post-solve depth and error reports (reference evaluate.py), on the GPU.

SURVEY §8(f) rows 1 and 4: metric depth along camera-0 rays from the solver's
correspondence, and the make_report reductions (error map, bad-pixel
percentages, mean / median error, depth error). NumPy in, NumPy out, like the
reference functions.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _ext

DEFAULT_TAUS = (1.0, 3.0, 5.0)


@dataclass
class ErrorReport:
    """Summary statistics over covisible, in-mask pixels (evaluate.py:40-58)."""

    pct_bad: dict
    mean_error_px: float
    median_error_px: float
    mean_abs_depth_error_m: float | None
    valid_count: int

    def to_dict(self) -> dict:
        return {"pct_bad": {f"tau>{t:g}": v for t, v in self.pct_bad.items()},
                "mean_error_px": self.mean_error_px,
                "median_error_px": self.median_error_px,
                "mean_abs_depth_error_m": self.mean_abs_depth_error_m,
                "valid_count": self.valid_count}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)


def _report(w_est, w_gt, valid, taus=(), depth_est=None, depth_gt=None):
    L = _ext.lib()
    we = np.asarray(w_est, dtype=np.float64)
    wg = np.asarray(w_gt, dtype=np.float64)
    if we.shape != wg.shape:
        raise ValueError("estimate and ground truth dimensions differ")
    v = np.asarray(valid, dtype=bool)
    n = int(v.size)
    taus = tuple(float(t) for t in taus)
    if any(t <= 0 for t in taus):
        raise ValueError("tau must be positive")
    dwe, dwg = _dev.upload(we, torch.float64), _dev.upload(wg, torch.float64)
    dv = _dev.upload(v, torch.uint8)
    dt = _dev.upload(np.asarray(taus or (1.0,), dtype=np.float64), torch.float64)
    dde = ddg = None
    if depth_est is not None and depth_gt is not None:
        dde = _dev.upload(np.asarray(depth_est, dtype=np.float64), torch.float64)
        ddg = _dev.upload(np.asarray(depth_gt, dtype=np.float64), torch.float64)
    err = _dev.empty(v.shape, torch.float64)
    out = _dev.empty((5 + max(len(taus), 1),), torch.float64)
    s = _dev.scratch(L.fsb_error_report_scratch_bytes(n))
    _ext.check(L.fsb_error_report(_dev.ptr(dwe), _dev.ptr(dwg), _dev.ptr(dv), n, _dev.ptr(dt),
                                  len(taus), _dev.ptr(dde) if dde is not None else None,
                                  _dev.ptr(ddg) if ddg is not None else None, _dev.ptr(err),
                                  _dev.ptr(out), _dev.ptr(s), s.numel(), _dev.stream_ptr()),
               "make_report")
    return _dev.download(err), _dev.download(out)


def correspondence_error(w_est, w_gt, valid) -> np.ndarray:
    """|(x + w_est) - (x + w_gt)| per pixel, 0 outside `valid` (evaluate.py:62-68)."""
    return _report(w_est, w_gt, valid)[0]


def erroneous_percentage(err, valid, tau: float) -> float:
    """Percentage of valid pixels with error above tau; NaN on an empty set
    (evaluate.py:71-78). `err` is an error map as from correspondence_error."""
    e = np.asarray(err, dtype=np.float64)
    z = np.zeros(e.shape + (2,))
    z[..., 0] = e
    return float(_report(z, np.zeros_like(z), valid, (tau,))[1][5])


def make_report(w_est, w_gt, valid, taus=DEFAULT_TAUS, depth_est=None,
                depth_gt=None) -> ErrorReport:
    """evaluate.make_report (evaluate.py:81-98), reductions on the GPU."""
    taus = tuple(taus)
    _, out = _report(w_est, w_gt, valid, taus, depth_est, depth_gt)
    n = int(out[0])
    depth_err = None
    if depth_est is not None and depth_gt is not None and out[4] > 0:
        depth_err = float(out[3])
    return ErrorReport(pct_bad={float(t): float(out[5 + k]) for k, t in enumerate(taus)},
                       mean_error_px=float(out[1]) if n else float("nan"),
                       median_error_px=float(out[2]) if n else float("nan"),
                       mean_abs_depth_error_m=depth_err, valid_count=n)


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
