"""Masked raster primitives on the GPU (reference rasters.py).

Host-array wrappers around libfsb200: NumPy in, NumPy (float64 / bool) out, so
they read like the reference functions they replace. Device-resident callers
use the solver's internal buffers directly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _ext


def pixel_grid(height: int, width: int) -> np.ndarray:
    """(H, W, 2) pixel-centre positions (x, y) (rasters.py:31-35)."""
    xs, ys = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64))
    return np.stack([xs, ys], axis=-1)


def sample_bicubic(field, pos, mask, acc64: bool = True):
    """Masked bicubic sampling with the reference fallback chain (rasters.py:57-141).

    Returns (values, valid): values NaN where invalid. Field values are fp32 on
    the device; `acc64` selects f64 weights/accumulation (the per-warp hot path
    inside the solver uses f32).
    """
    L = _ext.lib()
    data = np.asarray(field, dtype=np.float64)
    squeeze = data.ndim == 2
    if squeeze:
        data = data[:, :, None]
    h, w, c = data.shape
    if c not in (1, 2):
        raise ValueError("sample_bicubic supports 1 or 2 channels")
    p = np.asarray(pos, dtype=np.float64)
    shape = p.shape[:-1]
    n = int(np.prod(shape))
    df = _dev.upload(data)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    dp = _dev.upload(p.reshape(n, 2), torch.float64)
    out = _dev.empty((max(n, 1), c))
    ok = _dev.empty((max(n, 1),), torch.uint8)
    _ext.check(L.fsb_sample_bicubic(_dev.ptr(df), h, w, c, _dev.ptr(dm), _dev.ptr(dp), n,
                                    _dev.ptr(out), _dev.ptr(ok), int(acc64), _dev.stream_ptr()),
               "sample_bicubic")
    vals = _dev.download(out)[:n].reshape(shape + (c,))
    valid = _dev.download(ok, bool)[:n].reshape(shape)
    if squeeze:
        vals = vals[..., 0]
    return vals, valid


def gradient(field, mask) -> np.ndarray:
    """Forward-difference gradient, Neumann at mask/image borders (rasters.py:144-155)."""
    L = _ext.lib()
    f = np.asarray(field, dtype=np.float64)
    h, w = f.shape
    du = _dev.upload(f)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    g = _dev.empty((h, w, 2))
    _ext.check(L.fsb_gradient(_dev.ptr(du), _dev.ptr(dm), h, w, _dev.ptr(g), _dev.stream_ptr()),
               "gradient")
    return _dev.download(g)


def divergence(field, mask) -> np.ndarray:
    """Backward-difference divergence, negative adjoint of `gradient` (rasters.py:158-172)."""
    L = _ext.lib()
    p = np.asarray(field, dtype=np.float64)
    h, w, _ = p.shape
    dp = _dev.upload(p)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    d = _dev.empty((h, w))
    _ext.check(L.fsb_divergence(_dev.ptr(dp), _dev.ptr(dm), h, w, _dev.ptr(d),
                                _dev.stream_ptr()), "divergence")
    return _dev.download(d)


def smooth_masked(field, mask, sigma: float) -> np.ndarray:
    """Normalised Gaussian smoothing over in-mask pixels (rasters.py:185-191)."""
    L = _ext.lib()
    f = np.asarray(field, dtype=np.float64)
    h, w = f.shape
    df = _dev.upload(f)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    out = _dev.empty((h, w))
    s = _dev.scratch(L.fsb_smooth_scratch_bytes(h, w))
    _ext.check(L.fsb_smooth_masked(_dev.ptr(df), _dev.ptr(dm), h, w, float(sigma), _dev.ptr(out),
                                   _dev.ptr(s), s.numel(), _dev.stream_ptr()), "smooth_masked")
    return _dev.download(out)


def pyramid_shapes(height: int, width: int, levels: int, scale: float,
                   min_width: int) -> list[tuple[int, int]]:
    """Level shapes finest-first (rasters.py:207-221); ValueError on bad parameters."""
    L = _ext.lib()
    buf = (C.c_int32 * 64)()
    n = L.fsb_pyramid_shapes(int(height), int(width), int(levels), float(scale), int(min_width),
                             buf, 32)
    if n < 1:
        raise ValueError("levels must be >= 1 and scale > 1")
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n)]


@dataclass
class Pyramid:
    """Levels ordered coarsest to finest (rasters.py:194-204)."""

    fields: list
    masks: list
    scale: float

    @property
    def num_levels(self) -> int:
        return len(self.fields)


def downsample_area(field, mask, shape):
    """Masked area average + nearest-neighbour mask (rasters.py:228-260)."""
    L = _ext.lib()
    f = np.asarray(field, dtype=np.float64)
    fh, fw = f.shape
    ch, cw = shape
    df = _dev.upload(f)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    out = _dev.empty((ch, cw))
    om = _dev.empty((ch, cw), torch.uint8)
    _ext.check(L.fsb_downsample_area(_dev.ptr(df), _dev.ptr(dm), fh, fw, _dev.ptr(out),
                                     _dev.ptr(om), ch, cw, _dev.stream_ptr()), "downsample_area")
    return _dev.download(out), _dev.download(om, bool)


def build_pyramid(field, mask, levels: int, scale: float, min_width: int = 50) -> Pyramid:
    """Coarse-to-fine masked pyramid (rasters.py:263-273)."""
    shapes = pyramid_shapes(np.shape(mask)[0], np.shape(mask)[1], levels, scale, min_width)
    fields = [np.asarray(field, dtype=np.float64)]
    masks = [np.asarray(mask, dtype=bool)]
    for shape in shapes[1:]:
        f, m = downsample_area(fields[-1], masks[-1], shape)
        fields.append(f)
        masks.append(m)
    return Pyramid(fields=fields[::-1], masks=masks[::-1], scale=scale)


def upsample_state(u, w, mask, dst_shape, dst_mask):
    """Carry (u, w) to the next finer level (rasters.py:276-297)."""
    L = _ext.lib()
    uu = np.asarray(u, dtype=np.float64)
    sh, sw = uu.shape
    dh, dw = dst_shape
    du = _dev.upload(uu)
    dwv = _dev.upload(np.asarray(w, dtype=np.float64))
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    ddm = _dev.upload(np.asarray(dst_mask, dtype=bool), torch.uint8)
    uo = _dev.empty((dh, dw))
    wo = _dev.empty((dh, dw, 2))
    _ext.check(L.fsb_upsample_state(_dev.ptr(du), _dev.ptr(dwv), _dev.ptr(dm), sh, sw,
                                    _dev.ptr(ddm), dh, dw, _dev.ptr(uo), _dev.ptr(wo),
                                    _dev.stream_ptr()), "upsample_state")
    return _dev.download(uo), _dev.download(wo)
