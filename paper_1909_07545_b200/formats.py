"""PFM raster I/O (reference formats.py:17-66): float fields as little-endian
Portable Float Maps, rows bottom-up; vector fields as 3-channel PFM with the
third channel holding a validity flag or zero. Host-side file I/O only."""

from __future__ import annotations

from pathlib import Path

import numpy as np


def write_pfm(path, data) -> None:
    """(H, W) -> 'Pf', (H, W, 3) -> 'PF'; scale -1.0 marks little-endian."""
    a = np.asarray(data, dtype=np.float32)
    if a.ndim == 2:
        tag = b"Pf"
    elif a.ndim == 3 and a.shape[2] == 3:
        tag = b"PF"
    else:
        raise ValueError(f"PFM supports (H,W) or (H,W,3) arrays, got {a.shape}")
    h, w = a.shape[:2]
    header = tag + b"\n" + f"{w} {h}\n".encode() + b"-1.0\n"
    Path(path).write_bytes(header + np.ascontiguousarray(a[::-1]).astype("<f4").tobytes())


def read_pfm(path) -> np.ndarray:
    """PFM file -> float32 (H, W) or (H, W, 3), honouring the endianness sign."""
    raw = Path(path).read_bytes()
    lines = raw.split(b"\n", 3)
    if len(lines) < 4 or lines[0].strip() not in (b"Pf", b"PF"):
        raise ValueError(f"{path}: not a PFM file (header {lines[0][:8]!r})")
    c = 1 if lines[0].strip() == b"Pf" else 3
    w, h = (int(x) for x in lines[1].split())
    order = "<" if float(lines[2]) < 0 else ">"
    a = np.frombuffer(lines[3][: w * h * c * 4], dtype=f"{order}f4").reshape(h, w, c)
    a = a[::-1].astype(np.float32)
    return a[:, :, 0] if c == 1 else a


def write_vector_pfm(path, field, third=None) -> None:
    """(H, W, 2) field (+ optional (H, W) third channel) as a 3-channel PFM."""
    f = np.asarray(field)
    h, w = f.shape[:2]
    out = np.zeros((h, w, 3), dtype=np.float32)
    out[:, :, :2] = f
    if third is not None:
        out[:, :, 2] = np.asarray(third, dtype=np.float32)
    write_pfm(path, out)


def read_vector_pfm(path):
    """3-channel PFM -> ((H, W, 2) field, (H, W) third channel), float64."""
    a = read_pfm(path)
    if a.ndim != 3:
        raise ValueError(f"{path}: expected 3-channel PFM")
    return a[:, :, :2].astype(np.float64), a[:, :, 2].astype(np.float64)
