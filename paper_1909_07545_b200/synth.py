"""Synthetic fisheye stereo inputs, rendered on the GPU (reference synth.py).

Same scene vocabulary as the reference (`ValueNoise`, `Checkerboard`,
`SineGrating`, `Plane`, `Sphere`, `Box`, `Scene`, `default_scene`,
`reseed_scene`, `default_rig`, `pinhole_rig`, `plane_scene`, `render`); the
per-pixel ray casting runs in libfsb200's `fsb_render` kernel (fp64). Sensor
noise (`noise_sigma > 0`) is not supported: it uses NumPy's PCG64 stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from typing import Union

import numpy as np
import torch

from . import _dev, _ext
from .camera import PinholeCamera, RelativePose, StereoRig, UnifiedCamera


@dataclass(frozen=True)
class ValueNoise:
    scale: float = 0.5
    octaves: int = 3
    seed: int = 0
    lo: float = 0.1
    hi: float = 0.9
    persistence: float = 0.5
    kind = "noise"


@dataclass(frozen=True)
class Checkerboard:
    period: float = 0.4
    lo: float = 0.15
    hi: float = 0.9
    kind = "checker"


@dataclass(frozen=True)
class SineGrating:
    wavelength: float = 0.3
    direction: tuple = (1.0, 0.0, 0.0)
    lo: float = 0.1
    hi: float = 0.9
    kind = "sine"


Texture = Union[ValueNoise, Checkerboard, SineGrating]


@dataclass(frozen=True)
class Plane:
    point: tuple
    normal: tuple
    texture: Texture
    kind = "plane"


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float
    texture: Texture
    kind = "sphere"


@dataclass(frozen=True)
class Box:
    lo: tuple
    hi: tuple
    texture: Texture
    kind = "box"


@dataclass(frozen=True)
class Scene:
    primitives: tuple


def _prim_struct(p) -> _ext.FsbPrim:
    s = _ext.FsbPrim()
    g = [0.0] * 7
    if p.kind == "plane":
        s.kind = 0
        n = np.asarray(p.normal, dtype=np.float64)
        n = n / np.linalg.norm(n)
        g[0:3] = [float(v) for v in p.point]
        g[3:6] = [float(v) for v in n]
    elif p.kind == "sphere":
        s.kind = 1
        g[0:3] = [float(v) for v in p.center]
        g[3] = float(p.radius)
    elif p.kind == "box":
        s.kind = 2
        g[0:3] = [float(v) for v in p.lo]
        g[3:6] = [float(v) for v in p.hi]
    else:
        raise ValueError(f"unknown primitive kind {p.kind!r}")
    t = p.texture
    tx = [0.0] * 8
    if t.kind == "noise":
        s.tex_kind, s.octaves, s.seed = 0, int(t.octaves), int(t.seed)
        tx[0:4] = [float(t.scale), float(t.lo), float(t.hi), float(t.persistence)]
    elif t.kind == "checker":
        s.tex_kind = 1
        tx[0:3] = [float(t.period), float(t.lo), float(t.hi)]
    elif t.kind == "sine":
        s.tex_kind = 2
        d = np.asarray(t.direction, dtype=np.float64)
        d = d / np.linalg.norm(d)
        tx[0:3] = [float(t.wavelength), float(t.lo), float(t.hi)]
        tx[3:6] = [float(v) for v in d]
    else:
        raise ValueError(f"unknown texture kind {t.kind!r}")
    for i in range(7):
        s.geom[i] = g[i]
    for i in range(8):
        s.tex[i] = tx[i]
    return s


def _scene_device(scene) -> torch.Tensor:
    prims = [_prim_struct(p) for p in scene.primitives]
    raw = b"".join(bytes(p) for p in prims) or b"\0"
    host = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
    return host.to(_dev.device())


def render_device(scene, cam, pose: RelativePose | None = None, supersample: int = 1):
    """Device tensors (image f32, depth f32, hit u8) of `scene` seen by `cam` at `pose`."""
    if supersample < 1:
        raise ValueError("supersample must be >= 1")
    L = _ext.lib()
    cs = _ext.camera_struct(cam)
    prims = _scene_device(scene)
    img = _dev.empty((cs.height, cs.width))
    depth = _dev.empty((cs.height, cs.width))
    hit = _dev.empty((cs.height, cs.width), torch.uint8)
    if pose is None:
        Rp, op = None, None
    else:
        R = np.asarray(pose.rotation, dtype=np.float64).reshape(9)
        o = np.asarray(pose.camera1_center, dtype=np.float64).reshape(3)
        Rp = (C.c_double * 9)(*R.tolist())
        op = (C.c_double * 3)(*o.tolist())
    _ext.check(L.fsb_render(C.byref(cs), Rp, op, _dev.ptr(prims), len(scene.primitives),
                            int(supersample), _dev.ptr(img), _dev.ptr(depth), _dev.ptr(hit),
                            _dev.stream_ptr()), "render")
    return img, depth, hit


def render(scene, cam, pose: RelativePose | None = None, noise_sigma: float = 0.0,
           noise_seed: int = 0, supersample: int = 1):
    """(image, depth, valid) host arrays like synth.render (synth.py:217-254).

    The ray casting runs on the GPU; sensor noise (noise_sigma > 0) is drawn on
    the host from numpy's default_rng(noise_seed), exactly as the reference
    draws it, so noisy renders use the reference's noise stream."""
    img, depth, hit = render_device(scene, cam, pose, supersample)
    image, dep, valid = _dev.download(img), _dev.download(depth), _dev.download(hit, bool)
    if noise_sigma > 0:
        rng = np.random.default_rng(noise_seed)
        image = image + rng.normal(0.0, noise_sigma, size=image.shape)
        image = np.where(valid, np.clip(image, 0.0, 1.0), 0.0)
    return image, dep, valid


@dataclass(frozen=True)
class GroundTruth:
    """Exact per-pixel geometry of a rendered stereo pair (camera-0 grid)."""

    depth0: np.ndarray          # meters along the camera-0 ray
    correspondence: np.ndarray  # exact x1 - x0, pixels, zero where invalid
    covisibility: np.ndarray    # boolean: unoccluded and inside both views


def make_ground_truth(scene, rig: StereoRig, occlusion_tol: float = 1e-6) -> GroundTruth:
    """Exact depth, correspondence and covisibility (synth.py:271-303), ray-cast
    on the GPU in fp64 (fsb_ground_truth)."""
    L = _ext.lib()
    rs = _ext.rig_struct(rig)
    h, w = rs.cam0.height, rs.cam0.width
    prims = _scene_device(scene)
    depth = _dev.empty((h, w), torch.float64)
    corr = _dev.empty((h, w, 2), torch.float64)
    covis = _dev.empty((h, w), torch.uint8)
    s = _dev.scratch(256)
    _ext.check(L.fsb_ground_truth(C.byref(rs), _dev.ptr(prims), len(scene.primitives),
                                  float(occlusion_tol), _dev.ptr(depth), _dev.ptr(corr),
                                  _dev.ptr(covis), _dev.ptr(s), s.numel(), _dev.stream_ptr()),
               "make_ground_truth")
    return GroundTruth(depth0=_dev.download(depth), correspondence=_dev.download(corr),
                       covisibility=_dev.download(covis, bool))


# ---------------------------------------------------------------- stock configurations

def default_rig() -> StereoRig:
    """synth.py:306-318."""
    cam0 = UnifiedCamera(width=400, height=400, fx=200.0, fy=200.0, cx=199.5, cy=199.5,
                         fov=np.pi, xi=0.9)
    cam1 = UnifiedCamera(width=400, height=400, fx=200.0, fy=200.0, cx=200.5, cy=200.0,
                         fov=np.pi, xi=0.9)
    return StereoRig(cam0, cam1, RelativePose.from_displacement((0.1, 0.0, 0.0),
                                                                rotvec=(0.0, 0.035, 0.009)))


def pinhole_rig(width: int = 400, height: int = 400, f: float = 300.0,
                baseline: float = 0.1) -> StereoRig:
    """synth.py:321-328."""
    cam = PinholeCamera(width=width, height=height, fx=f, fy=f, cx=(width - 1) / 2.0,
                        cy=(height - 1) / 2.0, fov=np.deg2rad(90.0))
    return StereoRig(cam, cam, RelativePose.from_displacement((baseline, 0.0, 0.0)))


def default_scene() -> Scene:
    """Room-scale box + spheres scene (synth.py:331-364), same seeded layout."""
    rng = np.random.default_rng(12)
    prims = [
        Box(lo=(-1.3, -1.1, -0.4), hi=(1.3, 1.1, 1.5),
            texture=ValueNoise(scale=0.3, octaves=4, seed=11, lo=0.1, hi=0.95,
                               persistence=0.65)),
        Sphere(center=(0.28, -0.2, 0.6), radius=0.2,
               texture=ValueNoise(scale=0.07, octaves=4, seed=23, lo=0.1, hi=0.9,
                                  persistence=0.65)),
    ]
    placed = 0
    for i in range(60):
        if placed >= 12:
            break
        ang = rng.uniform(0, 2 * np.pi)
        rad = np.sqrt(rng.uniform(0.05, 1.0)) * 0.5
        x, y = rad * np.cos(ang), rad * np.sin(ang)
        if np.hypot(x - 0.28, y + 0.2) < 0.32:
            continue
        z = rng.uniform(0.55, 0.95)
        r = rng.uniform(0.04, 0.09)
        prims.append(Sphere(center=(float(x), float(y), float(z)), radius=float(r),
                            texture=ValueNoise(scale=float(r) * 0.7, octaves=3, seed=40 + i,
                                               lo=0.1, hi=0.95, persistence=0.6)))
        placed += 1
    return Scene(primitives=tuple(prims))


def reseed_scene(scene: Scene, seed: int) -> Scene:
    """Shift every noise seed by 1009*seed (synth.py:367-377)."""
    if seed == 0:
        return scene
    out = []
    for p in scene.primitives:
        t = p.texture
        if isinstance(t, ValueNoise) or getattr(t, "kind", None) == "noise":
            t = replace(t, seed=t.seed + 1009 * seed)
        out.append(replace(p, texture=t))
    return Scene(primitives=tuple(out))


def plane_scene(depth: float = 2.0, texture=None) -> Scene:
    """synth.py:380-386."""
    tex = texture if texture is not None else ValueNoise(scale=0.4, octaves=3, seed=7, lo=0.1,
                                                         hi=0.95)
    return Scene(primitives=(Plane(point=(0.0, 0.0, depth), normal=(0.0, 0.0, -1.0),
                                   texture=tex),))
