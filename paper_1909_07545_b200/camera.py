"""Camera models, poses and rigs — the parameter objects of the solve API.

Mirrors the reference's `fisheyestereo.camera` types (camera.py:47-314) so a
caller can switch packages without touching its rig code: same class names,
fields, `scaled_to`, pose construction and JSON schema (docs/rig_schema.json).
The per-pixel lens math (`project`, `unproject`, `fov_mask`) runs on the GPU
through libfsb200 (fp64); reference objects are accepted everywhere too
(duck-typed on `model` and the CameraBase fields).
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from . import _dev, _ext


def _points(x, last=(2, 3)) -> np.ndarray:
    a = np.asarray(x, dtype=np.float64)
    if a.shape[-1] not in last:
        raise ValueError(f"expected trailing dimension in {last}, got {a.shape}")
    return a


@dataclass(frozen=True)
class CameraBase:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    fov: float  # full field-of-view angle, radians

    def scaled_to(self, shape: tuple[int, int]) -> "CameraBase":
        """Same lens on a (height, width) grid (camera.py:66-77)."""
        h, w = shape
        sx = w / self.width
        sy = h / self.height
        d = asdict(self)
        d.update(width=w, height=h, fx=self.fx * sx, fy=self.fy * sy,
                 cx=(self.cx + 0.5) * sx - 0.5, cy=(self.cy + 0.5) * sy - 0.5)
        return type(self)(**d)

    def fov_mask(self) -> np.ndarray:
        return fov_mask(self)

    def project(self, points):
        return project(self, points)

    def unproject(self, pix):
        return unproject(self, pix)


@dataclass(frozen=True)
class PinholeCamera(CameraBase):
    model = "pinhole"


@dataclass(frozen=True)
class UnifiedCamera(CameraBase):
    xi: float = 1.0
    model = "unified"


@dataclass(frozen=True)
class PolynomialFisheyeCamera(CameraBase):
    k: tuple[float, float, float, float] = (1.0, 0.0, 0.0, 0.0)
    model = "polynomial"


_CLASSES = {"pinhole": PinholeCamera, "unified": UnifiedCamera,
            "polynomial": PolynomialFisheyeCamera}


def rotation_from_rotvec(rotvec) -> np.ndarray:
    """Axis-angle -> rotation matrix (Rodrigues), as camera.py:234-242."""
    v = np.asarray(rotvec, dtype=np.float64)
    angle = float(np.linalg.norm(v))
    if angle < 1e-14:
        return np.eye(3)
    a = v / angle
    K = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * (K @ K)


@dataclass(frozen=True)
class RelativePose:
    """X1 = R X0 + t (camera.py:245-276)."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        R = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        t = np.asarray(self.translation, dtype=np.float64).reshape(3)
        if np.max(np.abs(R.T @ R - np.eye(3))) > 1e-12 or np.linalg.det(R) < 0:
            raise ValueError("rotation must be orthonormal with det +1")
        object.__setattr__(self, "rotation", R)
        object.__setattr__(self, "translation", t)

    def transform(self, points) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) @ self.rotation.T + self.translation

    def inverse(self) -> "RelativePose":
        return RelativePose(self.rotation.T, -self.rotation.T @ self.translation)

    @property
    def camera1_center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @staticmethod
    def from_displacement(center1, rotvec=(0.0, 0.0, 0.0)) -> "RelativePose":
        R = rotation_from_rotvec(rotvec)
        return RelativePose(R, -R @ np.asarray(center1, dtype=np.float64))


@dataclass(frozen=True)
class StereoRig:
    cam0: CameraBase
    cam1: CameraBase
    pose: RelativePose

    @property
    def baseline(self) -> float:
        return float(np.linalg.norm(self.pose.translation))


# ---------------------------------------------------------------- JSON (docs/rig_schema.json)

def camera_from_dict(d: dict) -> CameraBase:
    kind = d["type"]
    if kind not in _CLASSES:
        raise ValueError(f"unknown camera type {kind!r}")
    kw = dict(width=int(d["width"]), height=int(d["height"]), fx=float(d["fx"]),
              fy=float(d["fy"]), cx=float(d["cx"]), cy=float(d["cy"]),
              fov=float(np.deg2rad(d["fov_deg"])))
    if kind == "unified":
        kw["xi"] = float(d["xi"])
    elif kind == "polynomial":
        k = [float(v) for v in d["k"]]
        if len(k) != 4:
            raise ValueError("polynomial camera needs 4 coefficients")
        kw["k"] = tuple(k)
    return _CLASSES[kind](**kw)


def camera_to_dict(cam) -> dict:
    d = {"type": cam.model, "width": cam.width, "height": cam.height, "fx": cam.fx,
         "fy": cam.fy, "cx": cam.cx, "cy": cam.cy, "fov_deg": float(np.rad2deg(cam.fov))}
    if cam.model == "unified":
        d["xi"] = cam.xi
    elif cam.model == "polynomial":
        d["k"] = list(cam.k)
    return d


def rig_from_dict(d: dict) -> StereoRig:
    pose = RelativePose(np.asarray(d["pose"]["rotation"], dtype=np.float64).reshape(3, 3),
                        np.asarray(d["pose"]["translation"], dtype=np.float64))
    return StereoRig(camera_from_dict(d["cam0"]), camera_from_dict(d["cam1"]), pose)


def rig_to_dict(rig) -> dict:
    return {"cam0": camera_to_dict(rig.cam0), "cam1": camera_to_dict(rig.cam1),
            "pose": {"rotation": [float(v) for v in np.ravel(rig.pose.rotation)],
                     "translation": [float(v) for v in rig.pose.translation]}}


def load_rig(path) -> StereoRig:
    return rig_from_dict(json.loads(Path(path).read_text()))


def save_rig(path, rig) -> None:
    Path(path).write_text(json.dumps(rig_to_dict(rig), indent=2) + "\n")


# ---------------------------------------------------------------- GPU lens math

def fov_mask(cam) -> np.ndarray:
    """Boolean (H, W) FOV mask (camera.py:79-84), computed on the GPU."""
    L = _ext.lib()
    cs = _ext.camera_struct(cam)
    m = _dev.empty((cs.height, cs.width), dtype=_dev.torch.uint8)
    s = _dev.scratch(L.fsb_fov_mask_scratch_bytes(C.byref(cs)))
    _ext.check(L.fsb_fov_mask(C.byref(cs), _dev.ptr(m), _dev.ptr(s), s.numel(),
                              _dev.stream_ptr()), "fov_mask")
    return _dev.download(m, bool)


def unproject(cam, pix):
    """Unit rays (..., 3) and validity for pixels (..., 2); NaN where invalid."""
    L = _ext.lib()
    p = _points(pix, (2,))
    shape = p.shape[:-1]
    n = int(np.prod(shape))
    cs = _ext.camera_struct(cam)
    dp = _dev.upload(p.reshape(n, 2), _dev.torch.float64)
    rays = _dev.empty((n, 3), _dev.torch.float64)
    ok = _dev.empty((n,), _dev.torch.uint8)
    s = _dev.scratch(L.fsb_unproject_scratch_bytes())
    _ext.check(L.fsb_unproject(C.byref(cs), _dev.ptr(dp), n, _dev.ptr(rays), _dev.ptr(ok),
                               _dev.ptr(s), s.numel(), _dev.stream_ptr()), "unproject")
    return _dev.download(rays).reshape(shape + (3,)), _dev.download(ok, bool).reshape(shape)


def project(cam, points):
    """Pixels (..., 2) and validity for 3-D points (..., 3); NaN where invalid."""
    L = _ext.lib()
    X = _points(points, (3,))
    shape = X.shape[:-1]
    n = int(np.prod(shape))
    cs = _ext.camera_struct(cam)
    dX = _dev.upload(X.reshape(n, 3), _dev.torch.float64)
    pix = _dev.empty((n, 2), _dev.torch.float64)
    ok = _dev.empty((n,), _dev.torch.uint8)
    _ext.check(L.fsb_project(C.byref(cs), _dev.ptr(dX), n, _dev.ptr(pix), _dev.ptr(ok),
                             _dev.stream_ptr()), "project")
    return _dev.download(pix).reshape(shape + (2,)), _dev.download(ok, bool).reshape(shape)


def triangulate_midpoint(rig, x0, x1, min_angle: float = 1e-6):
    """Depth along the camera-0 ray from pixel correspondences (camera.py:317-343):
    the midpoint of the shortest segment between the two unprojection rays;
    NaN / invalid for invalid rays, near-parallel rays (< min_angle) or a
    midpoint behind camera 0. x0, x1: (..., 2)."""
    L = _ext.lib()
    a = np.asarray(x0, dtype=np.float64)
    b = np.asarray(x1, dtype=np.float64)
    if a.shape != b.shape or a.shape[-1:] != (2,):
        raise ValueError("x0 and x1 must both be (..., 2)")
    shape = a.shape[:-1]
    n = int(np.prod(shape))
    rs = _ext.rig_struct(rig)
    da = _dev.upload(a.reshape(n, 2), _dev.torch.float64)
    db = _dev.upload(b.reshape(n, 2), _dev.torch.float64)
    depth = _dev.empty((max(n, 1),), _dev.torch.float64)
    ok = _dev.empty((max(n, 1),), _dev.torch.uint8)
    s = _dev.scratch(L.fsb_triangulate_scratch_bytes())
    _ext.check(L.fsb_triangulate_midpoint(C.byref(rs), _dev.ptr(da), _dev.ptr(db), n,
                                          float(min_angle), _dev.ptr(depth), _dev.ptr(ok),
                                          _dev.ptr(s), s.numel(), _dev.stream_ptr()),
               "triangulate_midpoint")
    d = _dev.download(depth)[:n].reshape(shape)
    v = _dev.download(ok, bool)[:n].reshape(shape)
    return d, v
