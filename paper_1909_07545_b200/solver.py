"""Anisotropic TGV-L1 primal-dual disparity solver on B200 — the drop-in boundary.

Same public surface as the reference's `fisheyestereo.solver` for the dense
mapping path (solver.py:36-452): `SolverParams`, `StereoResult`, `WarpState`,
`SolverState`, `Diagnostics`, `solve_pyramid`, `solve_level`,
`primal_dual_iterate`, `compute_tensor`, `precondition_steps`,
`image_derivative_along`, `warp_image`, `thresholding_step`,
`calibrate_second_image`. Host arrays in (float64, any layout the reference
accepts), host arrays out (float64 / bool) — every pixel of the solve runs in
libfsb200's sm_100a kernels. `energy`, `apply_tensor` and `sqrt_tensor` are
host-side evaluation helpers kept for the reference's tests (solver.py:164-178,
455-473); they are not on the solve path.

`Solver` is the device-resident engine underneath `solve_pyramid`: it owns the
workspace for one (rig, params) pair, can capture the whole frame into a CUDA
graph, and exposes device-tensor entry points for throughput measurement.
"""

from __future__ import annotations

import ctypes as C
import sys
import threading
from collections import OrderedDict
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from . import _dev, _ext
from .fields import calibrate_second_image  # noqa: F401  (re-export, solver.py:389)
from .rasters import pixel_grid, pyramid_shapes, sample_bicubic


REGULARIZERS = {"tgv": 0, "tv": 1, "huber": 2}


@dataclass
class SolverParams:
    """Optimisation weights and schedule (solver.py:36-80), same defaults."""

    lam: float = 5.0
    alpha0: float = 17.0
    alpha1: float = 1.2
    beta: float = 9.0
    eta: float = 0.85
    warp_iters: int = 50
    pd_iters: int = 10
    du_max: float = 0.2
    pyramid_levels: int = 5
    pyramid_scale: float = 2.0
    min_width: int = 50
    epsilon_scale: float = 0.1
    tensor_sigma: float = 1.0
    theta: float = 1.0
    # Regulariser (extension; the reference is TGV only, so "tv" / "huber" are
    # parity-unpinned): "tgv" = alpha1|T grad u - v| + alpha0|grad v| (reference),
    # "tv" = alpha1|T grad u| (TV-L1: v and q held at 0), "huber" = alpha1 *
    # Huber_eps(T grad u) (Huber-TV, BASELINE config C5).
    regularizer: str = "tgv"
    huber_eps: float = 0.05

    def __post_init__(self):
        if min(self.lam, self.alpha0, self.alpha1, self.beta, self.eta) <= 0:
            raise ValueError("all weights must be positive")
        if self.regularizer not in REGULARIZERS:
            raise ValueError(f"regularizer must be one of {sorted(REGULARIZERS)}")
        if self.huber_eps <= 0:
            raise ValueError("huber_eps must be positive")
        if self.du_max <= 0:
            raise ValueError("du_max must be positive")
        if self.warp_iters < 1 or self.pd_iters < 1:
            raise ValueError("iteration counts must be >= 1")

    def to_dict(self) -> dict:
        return asdict(self)

    @staticmethod
    def from_dict(d: dict) -> "SolverParams":
        unknown = set(d) - set(SolverParams.__dataclass_fields__)
        if unknown:
            raise ValueError(f"unknown solver parameters: {sorted(unknown)}")
        return SolverParams(**d)


@dataclass
class WarpState:
    u: np.ndarray
    w: np.ndarray
    omega: int = 0


@dataclass
class SolverState:
    u: np.ndarray
    v: np.ndarray
    p: np.ndarray
    q: np.ndarray
    u_bar: np.ndarray
    v_bar: np.ndarray


@dataclass
class Diagnostics:
    max_p_norm: list = field(default_factory=list)
    max_q_norm: list = field(default_factory=list)
    max_du: list = field(default_factory=list)
    mean_abs_du: list = field(default_factory=list)
    du_max_limit: float = 0.0
    record_increments: bool = False
    increments: list = field(default_factory=list)


@dataclass
class StereoResult:
    u: np.ndarray
    w: np.ndarray
    v: np.ndarray
    mask: np.ndarray
    i1_calibrated: np.ndarray
    diagnostics: Diagnostics | None = None


# ---------------------------------------------------------------- level buffers

def _planes(a, c: int) -> torch.Tensor:
    """(H, W, C) host array -> (C, H, W) contiguous device planes."""
    arr = np.asarray(a, dtype=np.float64)
    return _dev.upload(np.moveaxis(arr, -1, 0))


def _from_planes(t: torch.Tensor) -> np.ndarray:
    return np.moveaxis(_dev.download(t), 0, -1)


class _Level:
    """Device buffers of one pyramid level, viewable as the C `fsb_level`."""

    def __init__(self, h: int, w: int, blocked: bool = True):
        self.h, self.w = h, w
        E = _dev.empty
        U8 = torch.uint8
        self.i0 = E((h, w)); self.i1 = E((h, w)); self.mask = E((h, w), U8)
        self.traj = E((h, w, 2)); self.traj_ok = E((h, w), U8)
        # state planes as one (12, h, w) block and the per-warp constants as one
        # (10, h, w) block: the layout the TMA-fed PD kernel loads as 3-D boxes
        self.state_a = E((12, h, w))
        self.u, self.u_bar = self.state_a[0], self.state_a[1]
        self.v, self.v_bar = self.state_a[2:4], self.state_a[4:6]
        self.p, self.q = self.state_a[6:8], self.state_a[8:12]
        self.consts = E((10, h, w))
        self.tensor, self.steps = self.consts[0:3], self.consts[3:6]
        self.iu, self.rho0, self.u_omega = self.consts[6], self.consts[7], self.consts[8]
        self.maskf = self.consts[9] if blocked else None
        self.wv = E((h, w, 2))
        self.i1w = E((h, w))
        self.i1w_ok = E((h, w), U8); self.dirs = E((h, w, 2)); self.dir_ok = E((h, w), U8)
        self.partials = E((int(_ext.lib().fsb_level_partials(h, w)),), torch.float64)
        # second state set (ping-pong) -> temporally blocked PD kernel (K6)
        self.state_b = E((12, h, w)) if blocked else None
        self.packed = E((h, w, 4)) if blocked else None
        self.full16 = E((h, w), U8) if blocked else None
        ntl = int(_ext.lib().fsb_level_tiles(h, w))
        self.tiles = E((ntl,), torch.int32) if blocked else None

    def struct(self) -> _ext.FsbLevel:
        s = _ext.FsbLevel()
        s.h, s.w = self.h, self.w
        for name, _ in _ext.FsbLevel._fields_[2:]:
            setattr(s, name, _dev.ptr(getattr(self, name)))
        return s


def _setup_level(lv: _Level, i0, mask, prm: _ext.FsbParams) -> None:
    L = _ext.lib()
    lv.i0.copy_(_dev.upload(i0))
    lv.mask.copy_(_dev.upload(np.asarray(mask, dtype=bool), torch.uint8))
    s = _dev.scratch(L.fsb_smooth_scratch_bytes(lv.h, lv.w))
    st = lv.struct()
    _ext.check(L.fsb_level_setup(C.byref(st), C.byref(prm), _dev.ptr(s), s.numel(),
                                 _dev.stream_ptr()), "level_setup")


# ---------------------------------------------------------------- per-stage API

@dataclass
class _StepSizes:
    sigma_p: np.ndarray
    sigma_q: float
    tau_u: np.ndarray
    tau_v: np.ndarray


def compute_tensor(i0, beta: float, eta: float, mask) -> np.ndarray:
    """Edge tensor (a, b, c) per pixel from an already-smoothed image (solver.py:122-141)."""
    L = _ext.lib()
    f = np.asarray(i0, dtype=np.float64)
    h, w = f.shape
    df = _dev.upload(f)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    t = _dev.empty((3, h, w))
    s = _dev.scratch(L.fsb_smooth_scratch_bytes(h, w))
    _ext.check(L.fsb_compute_tensor(_dev.ptr(df), _dev.ptr(dm), h, w, float(beta), float(eta),
                                    _dev.ptr(t), _dev.ptr(s), s.numel(), _dev.stream_ptr()),
               "compute_tensor")
    return _from_planes(t)


def precondition_steps(t, mask, params: SolverParams) -> _StepSizes:
    """Diagonal preconditioner step sizes (solver.py:246-276)."""
    L = _ext.lib()
    tt = np.asarray(t, dtype=np.float64)
    h, w, _ = tt.shape
    dt = _planes(tt, 3)
    dm = _dev.upload(np.asarray(mask, dtype=bool), torch.uint8)
    steps = _dev.empty((3, h, w))
    s = _dev.scratch(h * w * 24 + 256)
    prm = _ext.params_struct(params)
    _ext.check(L.fsb_precondition_steps(_dev.ptr(dt), _dev.ptr(dm), h, w, C.byref(prm),
                                        _dev.ptr(steps), _dev.ptr(s), s.numel(),
                                        _dev.stream_ptr()), "precondition_steps")
    st = _dev.download(steps)
    sq = 1.0 / (2.0 * params.alpha0) if getattr(params, "regularizer", "tgv") == "tgv" else 0.0
    return _StepSizes(sigma_p=st[0], sigma_q=sq, tau_u=st[1],
                      tau_v=st[2])


def thresholding_step(u_hat, rho_hat, iu, tau_u, lam: float):
    """Closed-form prox of the linearised L1 data term (solver.py:205-218).

    Evaluated by the same device function the primal kernel inlines (here in
    f64, elementwise over broadcast host arrays).
    """
    L = _ext.lib()
    arrs = np.broadcast_arrays(*(np.asarray(a, dtype=np.float64)
                                 for a in (u_hat, rho_hat, iu, tau_u)))
    shape = arrs[0].shape
    n = int(np.prod(shape))
    dev = [_dev.upload(a.reshape(-1), torch.float64) for a in arrs]
    out = _dev.empty((max(n, 1),), torch.float64)
    _ext.check(L.fsb_thresholding_step(*[_dev.ptr(d) for d in dev], float(lam), n,
                                       _dev.ptr(out), _dev.stream_ptr()), "thresholding_step")
    return _dev.download(out)[:n].reshape(shape)


def primal_dual_iterate(state: SolverState, t, iu, rho0, u_omega, params: SolverParams, mask,
                        steps: _StepSizes | None = None, *, blocked: bool = False,
                        iters: int = 1) -> SolverState:
    """`iters` primal-dual cycles on the GPU (solver.py:279-303); one by default.

    blocked=True runs them in the temporally blocked tile kernel (K6) instead of
    the one-iteration-per-launch kernels.
    """
    L = _ext.lib()
    u = np.asarray(state.u, dtype=np.float64)
    h, w = u.shape
    lv = _Level(h, w, blocked=blocked)
    lv.mask.copy_(_dev.upload(np.asarray(mask, dtype=bool), torch.uint8))
    lv.tensor.copy_(_planes(t, 3))
    if steps is None:
        steps = precondition_steps(t, mask, params)
    lv.steps.copy_(_dev.upload(np.stack([steps.sigma_p, steps.tau_u, steps.tau_v])))
    lv.u.copy_(_dev.upload(u)); lv.u_bar.copy_(_dev.upload(state.u_bar))
    lv.v.copy_(_planes(state.v, 2)); lv.v_bar.copy_(_planes(state.v_bar, 2))
    lv.p.copy_(_planes(state.p, 2)); lv.q.copy_(_planes(state.q, 4))
    lv.iu.copy_(_dev.upload(iu)); lv.rho0.copy_(_dev.upload(rho0))
    lv.u_omega.copy_(_dev.upload(u_omega))
    prm = _ext.params_struct(params)
    st = lv.struct()
    _ext.check(L.fsb_pd_iterate(C.byref(st), C.byref(prm), int(iters), None, None,
                                _dev.stream_ptr()), "primal_dual_iterate")
    return SolverState(u=_dev.download(lv.u), v=_from_planes(lv.v), p=_from_planes(lv.p),
                       q=_from_planes(lv.q), u_bar=_dev.download(lv.u_bar),
                       v_bar=_from_planes(lv.v_bar))


def apply_tensor(t, vec) -> np.ndarray:
    """Packed symmetric tensors (a, b, c) times 2-vectors (solver.py:164-168)."""
    t = np.asarray(t)
    vec = np.asarray(vec)
    a, b, c = t[..., 0], t[..., 1], t[..., 2]
    return np.stack([a * vec[..., 0] + b * vec[..., 1], b * vec[..., 0] + c * vec[..., 1]],
                    axis=-1)


def sqrt_tensor(t) -> np.ndarray:
    """Symmetric PSD square root of packed tensors (solver.py:171-178)."""
    t = np.asarray(t, dtype=np.float64)
    a, b, c = t[..., 0], t[..., 1], t[..., 2]
    s = np.sqrt(np.maximum(a * c - b * b, 0.0))
    tau = np.sqrt(np.maximum((a + c) + 2.0 * s, 1e-300))
    return np.stack([(a + s) / tau, b / tau, (c + s) / tau], axis=-1)


def energy(i0, i1c, mask, u, v, w, params: SolverParams) -> float:
    """Variational energy of a candidate (u, v, w) on the calibrated pair
    (solver.py:455-473): lam |rho| + alpha1 |T^1/2 grad u - v| + alpha0 |grad v|
    over the pixels where the warp resolves. For the TV / Huber-TV extension
    v is zero and the first-order term is alpha1 |T^1/2 grad u| (TV) or
    alpha1 Huber_eps(|T^1/2 grad u|) (quadratic below eps)."""
    from .rasters import gradient, smooth_masked
    mask = np.asarray(mask, dtype=bool)
    i0 = np.asarray(i0, dtype=np.float64)
    i1w, ok = warp_image(i1c, w, mask)
    sel = mask & ok
    t_half = sqrt_tensor(compute_tensor(smooth_masked(i0, mask, params.tensor_sigma),
                                        params.beta, params.eta, mask))
    rho = np.where(sel, i1w - i0, 0.0)
    reg = getattr(params, "regularizer", "tgv")
    v = np.asarray(v, dtype=np.float64) if reg == "tgv" else np.zeros(i0.shape + (2,))
    gu = apply_tensor(t_half, gradient(u, mask)) - v
    gv = np.concatenate([gradient(v[..., 0], mask), gradient(v[..., 1], mask)], axis=-1)
    e_data = params.lam * float(np.sum(np.abs(rho[sel])))
    ng = np.linalg.norm(gu, axis=-1)[sel]
    if reg == "huber":
        eps = params.huber_eps
        ng = np.where(ng <= eps, ng * ng / (2.0 * eps), ng - 0.5 * eps)
    e_g1 = params.alpha1 * float(np.sum(ng))
    e_g0 = params.alpha0 * float(np.sum(np.linalg.norm(gv, axis=-1)[sel]))
    return e_data + e_g1 + e_g0


def warp_image(image, w, mask):
    """Masked bicubic resample of `image` at x + w(x), zero where invalid (solver.py:181-189)."""
    img = np.asarray(image, dtype=np.float64)
    vals, ok = sample_bicubic(img, pixel_grid(*img.shape) + np.asarray(w), mask, acc64=False)
    return np.where(ok, vals, 0.0), ok


def image_derivative_along(dirs, i1w, i1w_valid, mask):
    """I_u = i1w(x + dir) - i1w(x) on valid taps (solver.py:192-202)."""
    a = np.asarray(i1w, dtype=np.float64)
    valid = np.asarray(i1w_valid, dtype=bool)
    ahead, ok = sample_bicubic(a, pixel_grid(*a.shape) + np.asarray(dirs),
                               np.asarray(mask, dtype=bool) & valid, acc64=False)
    iu = np.where(ok & valid, ahead - a, 0.0)
    return iu, ok & valid


def warp_linearize64(i0, i1, mask, traj_dirs, traj_valid, w, kind: int = 0):
    """The float64 path's warp prologue on one level (solver.py:332-346 with
    image_derivative_along 192-202): returns (i1w, i1w_ok, dirs, dir_ok, I_u, rho0)
    as host arrays. kind 0 = masked-gather kernels (large levels), 1 = NaN-encoded
    texel kernels (levels up to 256^2). i1w / dirs / I_u / rho0 are 0 where invalid
    and off the mask."""
    L = _ext.lib()
    m = np.asarray(mask, dtype=bool)
    h, wd = m.shape
    up = lambda a, dt=torch.float64: _dev.upload(np.asarray(a), dt)  # noqa: E731
    d_i0, d_i1 = up(i0), up(i1)
    d_m, d_t = up(m, torch.uint8), up(traj_dirs)
    d_tok, d_w = up(np.asarray(traj_valid, dtype=bool), torch.uint8), up(w)
    i1w = _dev.empty((h, wd), torch.float64); dirs = _dev.empty((h, wd, 2), torch.float64)
    iu = _dev.empty((h, wd), torch.float64); rho0 = _dev.empty((h, wd), torch.float64)
    wok = _dev.empty((h, wd), torch.uint8); dok = _dev.empty((h, wd), torch.uint8)
    s = _dev.scratch(L.fsb_warp_linearize_f64_scratch_bytes(h, wd))
    _ext.check(L.fsb_warp_linearize_f64(h, wd, *[_dev.ptr(t) for t in (
        d_i0, d_i1, d_m, d_t, d_tok, d_w, i1w, wok, dirs, dok, iu, rho0, s)], s.numel(),
        int(kind), _dev.stream_ptr()), "warp_linearize64")
    return (_dev.download(i1w), _dev.download(wok, bool), _dev.download(dirs),
            _dev.download(dok, bool), _dev.download(iu), _dev.download(rho0))


def solve_level(i0, i1, traj_dirs, traj_valid, params: SolverParams, mask, init: WarpState,
                diagnostics: Diagnostics | None = None, *,
                blocked: bool = True) -> tuple[WarpState, SolverState]:
    """Warping loop on one pyramid level, all on the GPU (solver.py:306-367).

    `blocked=False` selects the one-iteration-per-launch kernels (the v1 path,
    kept as an on-device cross-check of the temporally blocked kernel).
    """
    L = _ext.lib()
    m = np.asarray(mask, dtype=bool)
    h, w = m.shape
    record = diagnostics is not None and diagnostics.record_increments
    lv = _Level(h, w, blocked=blocked and not record)
    lv.i1.copy_(_dev.upload(i1))
    lv.traj.copy_(_dev.upload(traj_dirs))
    lv.traj_ok.copy_(_dev.upload(np.asarray(traj_valid, dtype=bool), torch.uint8))
    lv.u.copy_(_dev.upload(init.u))
    lv.wv.copy_(_dev.upload(init.w))
    prm = _ext.params_struct(params)
    N, K = params.warp_iters, params.pd_iters
    if diagnostics is not None:
        diagnostics.du_max_limit = params.du_max
    dp = _dev.zeros((N * K,)); dq = _dev.zeros((N * K,))
    dmx = _dev.zeros((N,)); dmean = _dev.zeros((N,), torch.float64)
    if not record:
        s = _dev.scratch(L.fsb_smooth_scratch_bytes(h, w))
        lv.i0.copy_(_dev.upload(i0))
        lv.mask.copy_(_dev.upload(m, torch.uint8))
        st = lv.struct()
        diag = _ext.FsbDiag(_dev.ptr(dp), _dev.ptr(dq), _dev.ptr(dmx), _dev.ptr(dmean))
        _ext.check(L.fsb_solve_level(C.byref(st), C.byref(prm),
                                     C.byref(diag) if diagnostics is not None else None, 0, 0,
                                     _dev.ptr(s), s.numel(), _dev.stream_ptr()), "solve_level")
    else:
        # Per-warp enqueue so each (du, dirs) increment can be recorded (solver.py:364-365).
        _setup_level(lv, i0, m, prm)
        for t in (lv.v, lv.v_bar, lv.p, lv.q):
            t.zero_()
        lv.u_bar.copy_(lv.u)
        st = lv.struct()
        for wi in range(N):
            _ext.check(L.fsb_warp_linearize(C.byref(st), _dev.stream_ptr()), "warp_linearize")
            _ext.check(L.fsb_pd_iterate(C.byref(st), C.byref(prm), K,
                                        _dev.ptr(dp[wi * K:]), _dev.ptr(dq[wi * K:]),
                                        _dev.stream_ptr()), "pd_iterate")
            _ext.check(L.fsb_warp_finish(C.byref(st), C.byref(prm), _dev.ptr(dmx[wi:]),
                                         _dev.ptr(dmean[wi:]), _dev.stream_ptr()), "warp_finish")
            du = _dev.download(lv.u) - _dev.download(lv.u_omega)
            diagnostics.increments.append((du, _dev.download(lv.dirs)))
    if diagnostics is not None:
        diagnostics.max_p_norm.extend(float(x) for x in _dev.download(dp))
        diagnostics.max_q_norm.extend(float(x) for x in _dev.download(dq))
        diagnostics.max_du.extend(float(x) for x in _dev.download(dmx))
        diagnostics.mean_abs_du.extend(float(x) for x in _dev.download(dmean))
    ws = WarpState(u=_dev.download(lv.u), w=_dev.download(lv.wv), omega=init.omega + N)
    ss = SolverState(u=ws.u, v=_from_planes(lv.v), p=_from_planes(lv.p), q=_from_planes(lv.q),
                     u_bar=_dev.download(lv.u_bar), v_bar=_from_planes(lv.v_bar))
    return ws, ss


# ---------------------------------------------------------------- pyramid engine

class Solver:
    """Device-resident solve_pyramid engine for one (rig, params) pair.

    Owns the workspace, fixed input/output buffers (so the frame can be
    captured into a CUDA graph) and optional diagnostics slots.
    """

    def __init__(self, rig, params: SolverParams, collect_diagnostics: bool = False,
                 precision: str = "fp64"):
        if precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")
        L = _ext.lib()
        # the engine's workspace, buffers, graph and streams live on the device
        # current at construction; every later call runs there (solve() enters it)
        self.device = torch.cuda.current_device() if torch.cuda.is_available() else None
        self.rig = rig
        self.params = params
        self.precision = precision
        self.rs = _ext.rig_struct(rig)
        self.ps = _ext.params_struct(params)
        self.H, self.W = self.rs.cam0.height, self.rs.cam0.width
        self.H1, self.W1 = self.rs.cam1.height, self.rs.cam1.width
        sizer = (L.fsb_solve_pyramid_workspace_bytes if precision == "fp32"
                 else L.fsb_solve_pyramid_f64_workspace_bytes)
        nbytes = sizer(C.byref(self.rs), C.byref(self.ps))
        if nbytes == 0:
            raise ValueError("invalid rig or solver parameters")
        self.shapes = pyramid_shapes(self.H, self.W, params.pyramid_levels,
                                     params.pyramid_scale, params.min_width)
        self.workspace = _dev.scratch(nbytes)
        self.dtype = torch.float32 if precision == "fp32" else torch.float64
        E = lambda shape, dt=None: _dev.empty(shape, dt or self.dtype)  # noqa: E731
        self.i0 = E((self.H, self.W)); self.i1 = E((self.H1, self.W1))
        self.u = E((self.H, self.W)); self.w = E((self.H, self.W, 2))
        self.v = E((self.H, self.W, 2)); self.mask = E((self.H, self.W), torch.uint8)
        self.i1c = E((self.H, self.W))
        self.diag = None
        if collect_diagnostics:
            npd, nw = C.c_int64(), C.c_int64()
            L.fsb_diag_counts(self.H, self.W, C.byref(self.ps), C.byref(npd), C.byref(nw))
            self.d_p = E((npd.value,), torch.float32); self.d_q = E((npd.value,), torch.float32)
            # max |du| per warp: float64 on the float64 path (the reference's
            # du_max + 1e-15 bound holds exactly), float32 on the float32 path
            self.d_du = E((nw.value,), torch.float64 if precision == "fp64" else torch.float32)
            self.d_mean = E((nw.value,), torch.float64)
            f64 = precision == "fp64"
            self.diag = _ext.FsbDiag(_dev.ptr(self.d_p), _dev.ptr(self.d_q),
                                     None if f64 else _dev.ptr(self.d_du), _dev.ptr(self.d_mean),
                                     _dev.ptr(self.d_du) if f64 else None)
        self._traj = None
        self._host = None
        self._out_pool: list = []  # pinned output sets (see _out_set)
        self._early_stream = None   # D2H of mask / i1c during the frame (_solve)
        self.graph = None
        self.kernels_per_frame = None

    # -- trajectory override (solver.py:437-438)
    def set_traj_override(self, traj_override) -> None:
        from .camera import StereoRig
        from .fields import translation_only_rig
        if traj_override is None:
            self._traj = None
            return
        rig_t = translation_only_rig(self.rig)
        dirs_t, ok_t = [], []
        for (h, w) in self.shapes[::-1]:
            cam_l = self.rig.cam0.scaled_to((h, w))
            d, ok = traj_override(StereoRig(cam_l, cam_l, rig_t.pose))
            dirs_t.append(_dev.upload(np.asarray(d, dtype=np.float64), self.dtype))
            ok_t.append(_dev.upload(np.asarray(ok, dtype=bool), torch.uint8))
        n = len(dirs_t)
        self._traj = (dirs_t, ok_t, (C.c_void_p * n)(*[_dev.ptr(t) for t in dirs_t]),
                      (C.c_void_p * n)(*[_dev.ptr(t) for t in ok_t]))
        self.release()

    def _args(self, i0, i1):
        td, tk = (self._traj[2], self._traj[3]) if self._traj else (None, None)
        return (C.byref(self.rs), C.byref(self.ps), _dev.ptr(i0), _dev.ptr(i1),
                C.cast(td, C.c_void_p) if td else None, C.cast(tk, C.c_void_p) if tk else None,
                _dev.ptr(self.workspace), self.workspace.numel(), _dev.ptr(self.u),
                _dev.ptr(self.w), _dev.ptr(self.v), _dev.ptr(self.mask), _dev.ptr(self.i1c),
                C.byref(self.diag) if self.diag is not None else None)

    def run(self, i0: torch.Tensor | None = None, i1: torch.Tensor | None = None) -> None:
        """Enqueue one frame on the current stream (device inputs, device outputs)."""
        i0 = self.i0 if i0 is None else i0
        i1 = self.i1 if i1 is None else i1
        L = _ext.lib()
        fn = L.fsb_solve_pyramid if self.precision == "fp32" else L.fsb_solve_pyramid_f64
        _ext.check(fn(*self._args(i0, i1), _dev.stream_ptr()), "solve_pyramid")

    def time_phases(self, level: int = 0) -> dict:
        """One frame (direct enqueue, fp64 engines) with the native phase timer
        (fsb_solve_pyramid_f64_timed) at `level` (0 = finest): CUDA events on
        the solve stream around every warp's sampling kernels and its
        primal-dual launches. Returns summed milliseconds and launch counts."""
        if self.precision != "fp64":
            raise ValueError("phase timing is wired into the fp64 path")
        L = _ext.lib()
        tm = C.c_void_p()
        _ext.check(L.fsb_phase_timer_create(level, self.params.warp_iters, C.byref(tm)),
                   "phase_timer_create")
        try:
            _ext.check(L.fsb_solve_pyramid_f64_timed(
                C.byref(self.rs), C.byref(self.ps), _dev.ptr(self.i0), _dev.ptr(self.i1),
                _dev.ptr(self.workspace), self.workspace.numel(), _dev.ptr(self.u),
                _dev.ptr(self.w), _dev.ptr(self.v), _dev.ptr(self.mask), _dev.ptr(self.i1c),
                tm, _dev.stream_ptr()), "solve_pyramid_f64_timed")
            torch.cuda.current_stream().synchronize()
            a, b = C.c_double(), C.c_double()
            nw, npd, h, w = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            _ext.check(L.fsb_phase_timer_read(tm, C.byref(a), C.byref(b), C.byref(nw),
                                              C.byref(npd), C.byref(h), C.byref(w)),
                       "phase_timer_read")
        finally:
            L.fsb_phase_timer_destroy(tm)
        return {"sample_ms": a.value, "pd_ms": b.value, "warps": nw.value,
                "pd_launches_per_warp": npd.value, "h": h.value, "w": w.value}

    def capture(self) -> int:
        """Capture one frame on the fixed input buffers into a CUDA graph (native,
        fsb_graph_create); returns the number of kernel launches per frame."""
        L = _ext.lib()
        self.release()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = C.c_void_p()
        nk = C.c_int64()
        fn = L.fsb_graph_create if self.precision == "fp32" else L.fsb_graph_create_f64
        _ext.check(fn(*self._args(self.i0, self.i1), side.cuda_stream, C.byref(g), C.byref(nk)),
                   "graph_create")
        self.graph = g
        self.kernels_per_frame = int(nk.value)
        return self.kernels_per_frame

    def release(self) -> None:
        if getattr(self, "graph", None):
            _ext.lib().fsb_graph_destroy(self.graph)
        self.graph = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def replay(self) -> None:
        """Launch the captured frame on the current stream."""
        if not self.graph:
            self.capture()
        _ext.check(_ext.lib().fsb_graph_launch(self.graph, _dev.stream_ptr()), "graph_launch")

    def _staging(self):
        """Pinned fp32 input staging (the fp32 path's inputs; fp64 engines stage fp64)."""
        if self._host is None:
            P = dict(dtype=self.i0.dtype, pin_memory=True)
            self._host = {"i0": torch.empty((self.H, self.W), **P),
                          "i1": torch.empty((self.H1, self.W1), **P)}
        return self._host

    _OUT = (("u", torch.float64), ("w", torch.float64), ("v", torch.float64),
            ("mask", torch.bool), ("i1c", torch.float64))
    _POOL = 3  # output sets kept pinned per engine

    def _out_set(self) -> dict:
        """Pinned host buffers for one result, as (tensor, owner ndarray) pairs.

        The arrays handed to the caller are views of the owner ndarray, so a
        set is free again exactly when no caller-held view remains (its
        refcount is back to the pool's own). Reusing a free set avoids a
        cudaHostAlloc of ~50 MB per call; a set still referenced is never
        written, so every StereoResult stays fresh as in the reference.
        """
        for st in self._out_pool:
            if all(sys.getrefcount(st[k][1]) <= st["_free"] for k, _ in self._OUT):
                return st
        st = {}
        for k, dt in self._OUT:
            t = torch.empty(tuple(getattr(self, k).shape), dtype=dt, pin_memory=True)
            st[k] = (t, t.numpy())
        st["_free"] = sys.getrefcount(st["u"][1])
        if len(self._out_pool) < self._POOL:
            self._out_pool.append(st)
        return st

    def solve(self, i0, i1) -> StereoResult:
        """Host images in, StereoResult (float64 host arrays) out, on the
        engine's own device (copies, graph launch and sync on one stream)."""
        if self.device is None:
            return self._solve(i0, i1)
        with torch.cuda.device(self.device):
            return self._solve(i0, i1)

    def _solve(self, i0, i1) -> StereoResult:
        """Host images in, StereoResult (float64 host arrays) out.

        Inputs go host -> pinned staging in the engine's dtype (one
        multi-threaded copy per image) -> device; the frame runs as a replayed
        CUDA graph; outputs (widened to float64 on the device by fp32 engines)
        are copied straight into fresh pinned host buffers whose NumPy views
        are returned (no host-side conversion pass).
        """
        i0a = np.asarray(i0)
        i1a = np.asarray(i1)
        if i0a.shape != (self.H, self.W):
            raise ValueError("image 0 does not match camera 0 dimensions")
        if i1a.shape != (self.H1, self.W1):
            raise ValueError("image 1 does not match camera 1 dimensions")
        h = self._staging()
        # The caller's float64 images are rounded to the engine's dtype by the
        # host copy into pinned staging (IEEE round-to-nearest, as a device cast
        # would; torch spreads one whole-image copy over its host threads, which
        # measured faster than row chunks overlapped with their DMA), then one
        # H2D per image.
        for key, src in (("i0", i0a), ("i1", i1a)):
            src_t = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64))
            h[key].copy_(src_t)
            getattr(self, key).copy_(h[key], non_blocking=True)
        if self._traj is None:
            self.replay()
        else:
            self.run()
        st = self._out_set()
        outs = {}
        # float64 graphs record an event once mask and i1c are final: those two
        # go out on a side stream while the frame is still solving
        early = (_ext.lib().fsb_graph_early_event(self.graph)
                 if self._traj is None and self.graph else None)
        side = None
        if early:
            if self._early_stream is None:
                self._early_stream = torch.cuda.Stream()
            side = self._early_stream
            _ext.check(_ext.lib().fsb_stream_wait_event(C.c_void_p(side.cuda_stream),
                                                        C.c_void_p(early)), "stream_wait_event")
        for k, dt in self._OUT:
            src = getattr(self, k)
            # fp64 engines: every output is already float64 on the device and the
            # uint8 0/1 mask is viewed as bool, so no conversion kernel runs;
            # fp32 engines widen u / w / v / i1c on the device first.
            src = src.view(torch.bool) if dt == torch.bool else src.to(dt)
            if side is not None and k in ("mask", "i1c"):
                with torch.cuda.stream(side):
                    st[k][0].copy_(src, non_blocking=True)
            else:
                st[k][0].copy_(src, non_blocking=True)
            outs[k] = st[k][1].view()
        torch.cuda.current_stream().synchronize()
        if side is not None:
            side.synchronize()
        diag = None
        if self.diag is not None:
            diag = Diagnostics(du_max_limit=self.params.du_max)
            diag.max_p_norm = [float(x) for x in _dev.download(self.d_p)]
            diag.max_q_norm = [float(x) for x in _dev.download(self.d_q)]
            diag.max_du = [float(x) for x in _dev.download(self.d_du)]
            diag.mean_abs_du = [float(x) for x in _dev.download(self.d_mean)]
        return StereoResult(u=outs["u"], w=outs["w"], v=outs["v"], mask=outs["mask"],
                            i1_calibrated=outs["i1c"], diagnostics=diag)


_CACHE: "OrderedDict[tuple, list[Solver]]" = OrderedDict()
_CACHE_KEYS = 4      # distinct (rig, params, device, precision) keys kept
_CACHE_IDLE = 4      # idle engines kept per key (concurrent callers of one rig)
_CACHE_LOCK = threading.Lock()


def _rig_key(rig) -> tuple:
    def cam(c):
        return (c.model, c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.fov,
                getattr(c, "xi", None), tuple(getattr(c, "k", ())))
    return (cam(rig.cam0), cam(rig.cam1),
            tuple(np.asarray(rig.pose.rotation, dtype=np.float64).ravel()),
            tuple(np.asarray(rig.pose.translation, dtype=np.float64).ravel()))


def _checkout(key: tuple):
    """Pop an idle engine for `key` (None if there is none)."""
    with _CACHE_LOCK:
        idle = _CACHE.get(key)
        if idle:
            _CACHE.move_to_end(key)
            return idle.pop()
    return None


def _checkin(key: tuple, eng: "Solver") -> None:
    """Return an engine after a successful call; bounded per key and overall."""
    evicted = []
    with _CACHE_LOCK:
        idle = _CACHE.setdefault(key, [])
        _CACHE.move_to_end(key)
        if len(idle) < _CACHE_IDLE:
            idle.append(eng)
        else:
            evicted.append(eng)
        while len(_CACHE) > _CACHE_KEYS:
            evicted.extend(_CACHE.popitem(last=False)[1])
    for e in evicted:
        e.release()


def solve_pyramid(i0, i1, rig, params: SolverParams, collect_diagnostics: bool = False,
                  traj_override=None, *, precision: str = "fp64") -> StereoResult:
    """Full coarse-to-fine solve of a calibrated stereo pair (solver.py:401-452).

    Drop-in for `fisheyestereo.solve_pyramid`: same arguments, same
    `StereoResult` fields, ValueError on shape mismatch / invalid params /
    zero baseline. Engines are cached per (rig, params, device, precision) so
    repeated frames reuse the workspace and CUDA graph.

    precision="fp64" (default) is the reference's float64 arithmetic: it holds
    the north-star disparity gate (median 1e-3 / p99 1e-2 px) at every
    configuration, including C3 at N=50 (tests/test_gpu_c3_parity.py).
    precision="fp32" is the faster float32 path; it holds the median gate but
    not the p99 gate at N=50 warps (p99 ~3e-2 px at C3), so it
    must be requested explicitly.
    """
    i0a, i1a = np.asarray(i0), np.asarray(i1)
    if i0a.shape != (rig.cam0.height, rig.cam0.width):
        raise ValueError("image 0 does not match camera 0 dimensions")
    if i1a.shape != (rig.cam1.height, rig.cam1.width):
        raise ValueError("image 1 does not match camera 1 dimensions")
    if traj_override is None and not np.any(rig.pose.rotation.T @ rig.pose.translation):
        raise ValueError("trajectory field undefined for zero baseline")
    if precision not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    if traj_override is not None:
        eng = Solver(rig, params, collect_diagnostics, precision)
        eng.set_traj_override(traj_override)
        return eng.solve(i0a, i1a)
    # An engine is exclusive-use (workspace, graph, staging) and lives on one
    # device: it is checked OUT of the cache for the call, so concurrent
    # callers with the same rig each get their own engine and the function
    # stays re-entrant like the reference's. It goes back only
    # after a successful call; an engine whose call raised is released.
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    key = (_rig_key(rig), tuple(asdict(params).items()), bool(collect_diagnostics), precision,
           dev)
    eng = _checkout(key)
    if eng is None:
        eng = Solver(rig, params, collect_diagnostics, precision)
    try:
        res = eng.solve(i0a, i1a)
    except BaseException:
        eng.release()
        raise
    _checkin(key, eng)
    return res
