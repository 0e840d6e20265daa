"""Float64 NumPy restatement of the reference dense-mapping path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the checker the GPU path is
compared against, never the thing measured or shipped.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/fisheyestereo/). Operation order follows the
reference wherever rounding could differ, so on identical float64 inputs the
oracle reproduces the reference to the last bit on the pinned golden vectors
(tests/test_oracle_golden.py).

Cameras / rigs / params are duck-typed: any object with the reference
attribute names works (the product's own classes or the reference's).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

POLY_TOL = 1e-10      # camera.py:30
POLY_MAX_ITER = 50    # camera.py:31
DEGENERATE = 1e-12    # fields.py:25


# =============================================================== lens models

def _angle_from_axis(x, y, z):
    """Polar angle of a ray from +z (camera.py:41-44)."""
    return np.arctan2(np.hypot(x, y), z)


def _norm3(x, y, z):
    return np.sqrt((x * x + y * y) + z * z)


def _poly_r(k, t):
    """r/f for the odd polynomial model (camera.py:145-148)."""
    t2 = t * t
    return t * (k[0] + t2 * (k[1] + t2 * (k[2] + t2 * k[3])))


def _poly_dr(k, t):
    """d(r/f)/dtheta (camera.py:150-153)."""
    t2 = t * t
    return k[0] + t2 * (3 * k[1] + t2 * (5 * k[2] + t2 * 7 * k[3]))


def unproject(cam, px, py):
    """Unit rays (rx, ry, rz) and validity for pixel coordinates.

    pinhole camera.py:101-106, unified 126-136, polynomial 171-190 (Newton run
    until every pixel of the call has converged, at most 50 steps).
    """
    px = np.asarray(px, dtype=np.float64)
    py = np.asarray(py, dtype=np.float64)
    lim = 0.5 * cam.fov + 1e-12
    mx = (px - cam.cx) / cam.fx
    my = (py - cam.cy) / cam.fy
    kind = cam.model
    if kind == "pinhole":
        n = _norm3(mx, my, np.ones_like(mx))
        rx, ry, rz = mx / n, my / n, 1.0 / n
        ok = _angle_from_axis(rx, ry, rz) <= lim
    elif kind == "unified":
        xi = cam.xi
        r2 = mx * mx + my * my
        disc = 1.0 + (1.0 - xi * xi) * r2
        ok = disc >= 0.0
        eta = (xi + np.sqrt(np.maximum(disc, 0.0))) / (1.0 + r2)
        x, y, z = eta * mx, eta * my, eta - xi
        n = np.maximum(_norm3(x, y, z), 1e-300)
        rx, ry, rz = x / n, y / n, z / n
        ok = ok & (_angle_from_axis(rx, ry, rz) <= lim)
    elif kind == "polynomial":
        k = tuple(cam.k)
        rd = np.hypot(mx, my)
        phi = np.arctan2(my, mx)
        theta = rd / max(abs(k[0]), 1e-6)
        conv = np.zeros(rd.shape, dtype=bool)
        for _ in range(POLY_MAX_ITER):
            f = _poly_r(k, theta) - rd
            df = _poly_dr(k, theta)
            step = np.clip(f / np.where(np.abs(df) > 1e-12, df, 1e-12), -0.5, 0.5)
            theta = np.clip(theta - step, 0.0, np.pi)
            conv = np.abs(step) < POLY_TOL
            if conv.all():
                break
        st = np.sin(theta)
        rx, ry, rz = st * np.cos(phi), st * np.sin(phi), np.cos(theta)
        ok = conv & (theta <= lim)
    else:
        raise ValueError(f"unknown camera model {kind!r}")
    nan = np.nan
    return (np.where(ok, rx, nan), np.where(ok, ry, nan), np.where(ok, rz, nan), ok)


def project(cam, X, Y, Z):
    """Pixel coordinates and validity of 3-D points (camera.py:91-99, 115-124, 155-169)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    lim = 0.5 * cam.fov + 1e-12
    kind = cam.model
    if kind == "pinhole":
        ok = Z > 1e-12
        d = np.where(ok, Z, 1.0)
        px = cam.fx * X / d + cam.cx
        py = cam.fy * Y / d + cam.cy
        ok = ok & (_angle_from_axis(X, Y, Z) <= lim)
    elif kind == "unified":
        rho = _norm3(X, Y, Z)
        den = Z + cam.xi * rho
        ok = (den > 1e-12) & (rho > 0)
        d = np.where(ok, den, 1.0)
        px = cam.fx * X / d + cam.cx
        py = cam.fy * Y / d + cam.cy
        ok = ok & (_angle_from_axis(X, Y, Z) <= lim)
    elif kind == "polynomial":
        theta = _angle_from_axis(X, Y, Z)
        rxy = np.hypot(X, Y)
        r = _poly_r(tuple(cam.k), theta)
        safe = np.maximum(rxy, 1e-300)
        px = cam.fx * r * X / safe + cam.cx
        py = cam.fy * r * Y / safe + cam.cy
        axis = rxy == 0
        px = np.where(axis, cam.cx, px)
        py = np.where(axis, cam.cy, py)
        ok = (theta <= lim) & (_norm3(X, Y, Z) > 0)
    else:
        raise ValueError(f"unknown camera model {kind!r}")
    return np.where(ok, px, np.nan), np.where(ok, py, np.nan), ok


def grid_xy(h, w):
    ys, xs = np.mgrid[0:h, 0:w]
    return xs.astype(np.float64), ys.astype(np.float64)


def fov_mask(cam):
    """camera.py:79-84."""
    gx, gy = grid_xy(cam.height, cam.width)
    return unproject(cam, gx, gy)[3]


@dataclass(frozen=True)
class Lens:
    """Minimal camera record for rescaled levels (fields copied from any camera)."""

    model: str
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    fov: float
    xi: float = 0.0
    k: tuple = (1.0, 0.0, 0.0, 0.0)


def as_lens(cam) -> Lens:
    return Lens(cam.model, int(cam.width), int(cam.height), float(cam.fx), float(cam.fy),
                float(cam.cx), float(cam.cy), float(cam.fov),
                float(getattr(cam, "xi", 0.0)), tuple(getattr(cam, "k", (1.0, 0.0, 0.0, 0.0))))


def rescale(cam, h, w) -> Lens:
    """CameraBase.scaled_to (camera.py:66-77)."""
    sx = w / cam.width
    sy = h / cam.height
    c = as_lens(cam)
    return Lens(c.model, w, h, c.fx * sx, c.fy * sy, (c.cx + 0.5) * sx - 0.5,
                (c.cy + 0.5) * sy - 0.5, c.fov, c.xi, c.k)


# =============================================================== fields

def _rays_on_grid(cam):
    """fields.py:28-31: unit rays of every pixel, zero where invalid."""
    gx, gy = grid_xy(cam.height, cam.width)
    rx, ry, rz, ok = unproject(cam, gx, gy)
    return gx, gy, np.where(ok, rx, 0.0), np.where(ok, ry, 0.0), np.where(ok, rz, 0.0), ok


def calibration_field(rig):
    """Rotation+intrinsics flow on the cam0 grid (fields.py:34-45)."""
    gx, gy, rx, ry, rz, ok0 = _rays_on_grid(rig.cam0)
    R = np.asarray(rig.pose.rotation, dtype=np.float64)
    rays = np.stack([rx, ry, rz], axis=-1)
    rot = rays @ R.T
    px, py, ok1 = project(rig.cam1, rot[..., 0], rot[..., 1], rot[..., 2])
    ok = ok0 & ok1
    fld = np.stack([np.where(ok, px - gx, 0.0), np.where(ok, py - gy, 0.0)], axis=-1)
    return fld, ok


def residual_translation(rig):
    """translation_only_rig (fields.py:159-167): t_res = R^T t."""
    return np.asarray(rig.pose.rotation).T @ np.asarray(rig.pose.translation)


def trajectory_field(cam, t, epsilon_scale=0.1, depth=1.0):
    """Unit epipolar tangents of the rig (cam, cam, (I, t)) (fields.py:48-108)."""
    t = np.asarray(t, dtype=np.float64)
    tn = np.linalg.norm(t)
    if tn == 0:
        raise ValueError("trajectory field undefined for zero baseline")
    that = t / tn
    gx, gy, rx, ry, rz, ok0 = _rays_on_grid(cam)
    X, Y, Z = rx * depth, ry * depth, rz * depth

    def displaced_flow(eps):
        px, py, ok1 = project(cam, X + eps * that[0], Y + eps * that[1], Z + eps * that[2])
        ok = ok0 & ok1
        return np.where(ok, px - gx, 0.0), np.where(ok, py - gy, 0.0), ok

    fx, fy, ok = displaced_flow(1e-4 * depth)
    mags = np.sqrt(fx * fx + fy * fy)
    peak = float(np.max(mags[ok], initial=0.0))
    if peak > 0:
        fx, fy, ok = displaced_flow(1e-4 * depth * epsilon_scale / peak)
    mag = np.sqrt(fx * fx + fy * fy)
    degen = ok & (mag < DEGENERATE)
    good = ok & (mag >= DEGENERATE)
    safe = np.where(good, mag, 1.0)
    dx = np.where(good, fx / safe, 0.0)
    dy = np.where(good, fy / safe, 0.0)
    tiny = lambda a: (np.abs(a) < 1e-9) & (a != 0.0)  # noqa: E731
    if tiny(dx).any() or tiny(dy).any():  # fields.py:91-96 (global renormalisation)
        dx = np.where(tiny(dx), 0.0, dx)
        dy = np.where(tiny(dy), 0.0, dy)
        n = np.sqrt(dx * dx + dy * dy)
        big = n > 0.5
        n1 = np.where(big, n, 1.0)
        dx = np.where(big, dx / n1, 0.0)
        dy = np.where(big, dy / n1, 0.0)
    if degen.any():  # fields.py:100-107: 4-neighbour cross around the epipole
        blk = degen.copy()
        blk[1:, :] |= degen[:-1, :]
        blk[:-1, :] |= degen[1:, :]
        blk[:, 1:] |= degen[:, :-1]
        blk[:, :-1] |= degen[:, 1:]
        good = good & ~blk
        dx = np.where(good, dx, 0.0)
        dy = np.where(good, dy, 0.0)
    return np.stack([dx, dy], axis=-1), good


# =============================================================== rasters

def _cr_weights(f):
    """Catmull-Rom weights at offsets -1..2 (rasters.py:45-54)."""
    f2 = f * f
    f3 = f2 * f
    return (-0.5 * f + f2 - 0.5 * f3, 1.0 - 2.5 * f2 + 1.5 * f3,
            0.5 * f + 2.0 * f2 - 1.5 * f3, -0.5 * f2 + 0.5 * f3)


def bicubic(field, pos, mask):
    """Mask-aware bicubic with the bilinear / nearest fallback (rasters.py:57-141)."""
    data = np.asarray(field, dtype=np.float64)
    one = data.ndim == 2
    if one:
        data = data[..., None]
    H, W, nc = data.shape
    mask = np.asarray(mask, dtype=bool)
    pos = np.asarray(pos, dtype=np.float64)
    lead = pos.shape[:-1]
    x = pos[..., 0].reshape(-1)
    y = pos[..., 1].reshape(-1)
    finite = np.isfinite(x) & np.isfinite(y)
    x = np.where(finite, x, 0.0)
    y = np.where(finite, y, 0.0)
    bx = np.floor(x)
    by = np.floor(y)
    fx = x - bx
    fy = y - by
    ix = bx.astype(np.int64)
    iy = by.astype(np.int64)
    wx = _cr_weights(fx)
    wy = _cr_weights(fy)
    lin_x = (1.0 - fx, fx)
    lin_y = (1.0 - fy, fy)
    npos = x.size
    acc = np.zeros((npos, nc))
    lin = np.zeros((npos, nc))
    lin_w = np.zeros(npos)
    best = np.zeros((npos, nc))
    best_d2 = np.full(npos, np.inf)
    every = np.ones(npos, dtype=bool)
    some = np.zeros(npos, dtype=bool)
    for a in range(4):
        r = iy + (a - 1)
        r_ok = (r >= 0) & (r < H)
        rc = np.clip(r, 0, H - 1)
        for b in range(4):
            c = ix + (b - 1)
            tap = r_ok & (c >= 0) & (c < W)
            cc = np.clip(c, 0, W - 1)
            tap &= mask[rc, cc]
            v = np.where(tap[:, None], data[rc, cc], 0.0)
            every &= tap
            some |= tap
            acc += (wy[a] * wx[b])[:, None] * v
            if 1 <= a <= 2 and 1 <= b <= 2:
                wgt = np.where(tap, lin_y[a - 1] * lin_x[b - 1], 0.0)
                lin += wgt[:, None] * v
                lin_w += wgt
            d2 = ((b - 1) - fx) ** 2 + ((a - 1) - fy) ** 2
            nearer = tap & (d2 < best_d2)
            best_d2 = np.where(nearer, d2, best_d2)
            best = np.where(nearer[:, None], v, best)
    use_lin = lin_w > 1e-12
    out = np.where(use_lin[:, None], lin / np.maximum(lin_w, 1e-300)[:, None], best)
    out = np.where(every[:, None], acc, out)
    ok = some & finite
    out = np.where(ok[:, None], out, np.nan).reshape(lead + (nc,))
    if one:
        out = out[..., 0]
    return out, ok.reshape(lead)


def edges(mask):
    """Forward edges inside the mask (rasters.py:175-182)."""
    m = np.asarray(mask, dtype=bool)
    ex = np.zeros_like(m)
    ey = np.zeros_like(m)
    ex[:, :-1] = m[:, :-1] & m[:, 1:]
    ey[:-1, :] = m[:-1, :] & m[1:, :]
    return ex, ey


def grad_fwd(f, mask):
    """Forward-difference gradient with Neumann edges (rasters.py:144-155)."""
    f = np.asarray(f, dtype=np.float64)
    ex, ey = edges(mask)
    g = np.zeros(f.shape + (2,))
    g[:, :-1, 0] = (f[:, 1:] - f[:, :-1]) * ex[:, :-1]
    g[:-1, :, 1] = (f[1:, :] - f[:-1, :]) * ey[:-1, :]
    return g


def div_bwd(p, mask):
    """Backward-difference divergence, -adjoint of grad_fwd (rasters.py:158-172)."""
    p = np.asarray(p, dtype=np.float64)
    ex, ey = edges(mask)
    px = p[..., 0] * ex
    py = p[..., 1] * ey
    d = px.copy()
    d[:, 1:] -= px[:, :-1]
    d += py
    d[1:, :] -= py[:-1, :]
    return d


# -- scipy.ndimage.gaussian_filter restated (SciPy >= 1.10; 1.18.1 here):
#    kernel exp(-x^2/(2 s^2)) normalised, radius int(4 s + 0.5); correlate along
#    axis 0 then axis 1 with 'reflect' (half-sample symmetric) borders; symmetric
#    accumulation centre*w0 + sum_{j=r..1} (a[-j] + a[+j]) * w[j] (ni_filters.c).

def gauss_weights(sigma):
    radius = int(4.0 * sigma + 0.5)
    xs = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * xs ** 2)
    return radius, phi / phi.sum()


def _reflect(idx, n):
    if n == 1:
        return np.zeros_like(idx)
    period = 2 * n
    i = np.mod(idx, period)
    return np.where(i < n, i, period - 1 - i)


def _gauss_axis(a, radius, wts, axis):
    n = a.shape[axis]
    base = np.arange(n)
    centre = wts[radius]
    take = lambda off: np.take(a, _reflect(base + off, n), axis=axis)  # noqa: E731
    out = a * centre
    for j in range(radius, 0, -1):
        out = out + (take(-j) + take(j)) * wts[radius + j]
    return out


def gauss_filter(a, sigma):
    radius, wts = gauss_weights(sigma)
    out = np.asarray(a, dtype=np.float64)
    for axis in range(out.ndim):
        out = _gauss_axis(out, radius, wts, axis)
    return out


def smooth_in_mask(f, mask, sigma):
    """Normalised convolution over in-mask pixels (rasters.py:185-191)."""
    m = np.asarray(mask, dtype=bool)
    mf = m.astype(np.float64)
    num = gauss_filter(np.asarray(f, dtype=np.float64) * mf, sigma)
    den = gauss_filter(mf, sigma)
    return np.where(m, num / np.maximum(den, 1e-12), 0.0)


def level_shapes(h, w, levels, scale, min_width):
    """Finest-first level shapes (rasters.py:207-221)."""
    if levels < 1:
        raise ValueError("levels must be >= 1")
    if scale <= 1.0:
        raise ValueError("scale must be > 1")
    out = [(h, w)]
    while len(out) < levels:
        ph, pw = out[-1]
        nh, nw = int(np.ceil(ph / scale)), int(np.ceil(pw / scale))
        if nw < min_width:
            break
        out.append((nh, nw))
    return out


def area_down(f, mask, shape):
    """Masked area average onto `shape`, nearest-sample mask (rasters.py:224-260)."""
    f = np.asarray(f, dtype=np.float64)
    m = np.asarray(mask, dtype=bool)
    fh, fw = m.shape
    ch, cw = shape
    rows = (np.arange(fh, dtype=np.int64) * ch) // fh
    cols = (np.arange(fw, dtype=np.int64) * cw) // fw
    bins = (rows[:, None] * cw + cols[None, :]).ravel()
    count = np.bincount(bins, weights=m.astype(np.float64).ravel(), minlength=ch * cw)
    total = np.bincount(bins, weights=(f * m).ravel(), minlength=ch * cw)
    mean = (total / np.maximum(count, 1.0)).reshape(ch, cw)
    rr = np.clip(np.rint((np.arange(ch) + 0.5) * fh / ch - 0.5).astype(np.int64), 0, fh - 1)
    cc = np.clip(np.rint((np.arange(cw) + 0.5) * fw / cw - 0.5).astype(np.int64), 0, fw - 1)
    cm = m[rr[:, None], cc[None, :]] & (count.reshape(ch, cw) > 0)
    return np.where(cm, mean, 0.0), cm


def build_levels(f, mask, levels, scale, min_width):
    """Coarsest-first (images, masks) (rasters.py:263-273)."""
    shapes = level_shapes(mask.shape[0], mask.shape[1], levels, scale, min_width)
    fs = [np.asarray(f, dtype=np.float64)]
    ms = [np.asarray(mask, dtype=bool)]
    for shp in shapes[1:]:
        a, b = area_down(fs[-1], ms[-1], shp)
        fs.append(a)
        ms.append(b)
    return fs[::-1], ms[::-1]


def lift_state(u, w, mask, dst_shape, dst_mask):
    """upsample_state (rasters.py:276-297)."""
    sh, sw = mask.shape
    dh, dw = dst_shape
    sx, sy = dw / sw, dh / sh
    gx, gy = grid_xy(dh, dw)
    src = np.stack([(gx + 0.5) / sx - 0.5, (gy + 0.5) / sy - 0.5], axis=-1)
    uu, ok_u = bicubic(u, src, mask)
    ww, ok_w = bicubic(w, src, mask)
    uu = np.where(ok_u & dst_mask, uu, 0.0) * (0.5 * (sx + sy))
    ww = np.where((ok_w & dst_mask)[..., None], ww, 0.0)
    ww[..., 0] *= sx
    ww[..., 1] *= sy
    return uu, ww


# =============================================================== solver

def edge_tensor(sm, mask, beta, eta):
    """compute_tensor on a smoothed image (solver.py:122-161) -> (H, W, 3)."""
    f = np.asarray(sm, dtype=np.float64)
    ex, ey = edges(mask)
    dx = np.zeros_like(f)
    dy = np.zeros_like(f)
    dx[:, :-1] = (f[:, 1:] - f[:, :-1]) * ex[:, :-1]
    dy[:-1, :] = (f[1:, :] - f[:-1, :]) * ey[:-1, :]
    gx, nx = dx.copy(), ex.astype(np.float64)
    gx[:, 1:] += dx[:, :-1]
    nx[:, 1:] += ex[:, :-1]
    gy, ny = dy.copy(), ey.astype(np.float64)
    gy[1:, :] += dy[:-1, :]
    ny[1:, :] += ey[:-1, :]
    gx = gx / np.maximum(nx, 1.0)
    gy = gy / np.maximum(ny, 1.0)
    mag = np.hypot(gx, gy)
    flat = mag <= 1e-12
    safe = np.maximum(mag, 1e-300)
    ux = np.where(flat, 1.0, gx / safe)
    uy = np.where(flat, 0.0, gy / safe)
    lam = np.exp(-beta * mag ** eta)
    T = np.stack([lam * ux * ux + uy * uy, (lam - 1.0) * ux * uy, lam * uy * uy + ux * ux],
                 axis=-1)
    T[~np.asarray(mask, dtype=bool)] = (1.0, 0.0, 1.0)
    return T


@dataclass
class Steps:
    sigma_p: np.ndarray
    sigma_q: float
    tau_u: np.ndarray
    tau_v: np.ndarray


def step_sizes(T, mask, alpha0, alpha1, regularizer="tgv"):
    """Diagonal preconditioning (solver.py:246-276). For the TV / Huber-TV
    extension (no reference; parity unpinned) v and q are held at zero by
    tau_v = sigma_q = 0."""
    a, b, c = np.abs(T[..., 0]), np.abs(T[..., 1]), np.abs(T[..., 2])
    ex, ey = edges(mask)
    exf, eyf = ex.astype(np.float64), ey.astype(np.float64)
    sp = 1.0 / (alpha1 * np.maximum(2.0 * a * exf + 2.0 * b * eyf + 1.0,
                                    2.0 * b * exf + 2.0 * c * eyf + 1.0))
    hx = (a + b) * exf
    hy = (b + c) * eyf
    col = hx + hy
    col[:, 1:] += hx[:, :-1]
    col[1:, :] += hy[:-1, :]
    cnt = exf + eyf
    cnt[:, 1:] += exf[:, :-1]
    cnt[1:, :] += eyf[:-1, :]
    tgv = regularizer == "tgv"
    return Steps(sigma_p=sp, sigma_q=1.0 / (2.0 * alpha0) if tgv else 0.0,
                 tau_u=1.0 / np.maximum(alpha1 * col, 1e-12),
                 tau_v=1.0 / (alpha1 + alpha0 * cnt) if tgv else np.zeros_like(cnt))


def apply_T(T, v):
    return np.stack([T[..., 0] * v[..., 0] + T[..., 1] * v[..., 1],
                     T[..., 1] * v[..., 0] + T[..., 2] * v[..., 1]], axis=-1)


def shrink(u_hat, rho_hat, iu, tau, lam):
    """thresholding_step (solver.py:205-218)."""
    th = tau * lam * iu * iu
    nz = iu != 0
    q = np.zeros_like(u_hat)
    np.divide(rho_hat, np.where(nz, iu, 1.0), out=q, where=nz)
    delta = np.where(rho_hat < -th, tau * lam * iu,
                     np.where(rho_hat > th, -tau * lam * iu, -q))
    return u_hat + np.where(nz, delta, 0.0)


def _unit_ball(a):
    return a / np.maximum(1.0, np.linalg.norm(a, axis=-1, keepdims=True))


@dataclass
class PDState:
    u: np.ndarray
    v: np.ndarray
    p: np.ndarray
    q: np.ndarray
    u_bar: np.ndarray
    v_bar: np.ndarray


def pd_cycle(s: PDState, T, iu, rho0, u_omega, prm, mask, st: Steps) -> PDState:
    """primal_dual_iterate (solver.py:279-303)."""
    p = s.p + st.sigma_p[..., None] * prm.alpha1 * (apply_T(T, grad_fwd(s.u_bar, mask)) - s.v_bar)
    if getattr(prm, "regularizer", "tgv") == "huber":  # prox of the Huber conjugate
        p = p / (1.0 + st.sigma_p[..., None] * prm.alpha1 * prm.huber_eps)
    p = _unit_ball(p)
    jac = np.concatenate([grad_fwd(s.v_bar[..., 0], mask), grad_fwd(s.v_bar[..., 1], mask)],
                         axis=-1)
    q = _unit_ball(s.q + st.sigma_q * prm.alpha0 * jac)
    u_hat = s.u + st.tau_u * prm.alpha1 * div_bwd(apply_T(T, p), mask)
    rho_hat = rho0 + (u_hat - u_omega) * iu
    u = shrink(u_hat, rho_hat, iu, st.tau_u, prm.lam)
    divq = np.stack([div_bwd(q[..., 0:2], mask), div_bwd(q[..., 2:4], mask)], axis=-1)
    v = s.v + st.tau_v[..., None] * (prm.alpha0 * divq + prm.alpha1 * p)
    return PDState(u=u, v=v, p=p, q=q, u_bar=u + prm.theta * (u - s.u),
                   v_bar=v + prm.theta * (v - s.v))


def _masked_sample(f, pos, mask):
    vals, ok = bicubic(f, pos, mask)
    if vals.ndim == ok.ndim:
        return np.where(ok, vals, 0.0), ok
    return np.where(ok[..., None], vals, 0.0), ok


def linearize(i0, i1, traj, traj_ok, mask, w):
    """Warp-loop prologue (solver.py:332-343, image_derivative_along 192-202).

    Returns (i1w, warp_ok, dirs, dir_ok, iu, rho0).
    """
    h, wd = mask.shape
    gx, gy = grid_xy(h, wd)
    grid = np.stack([gx, gy], axis=-1)
    pos = grid + w
    i1w, warp_ok = _masked_sample(i1, pos, mask)
    raw, d_ok = _masked_sample(traj, pos, traj_ok)
    nrm = np.linalg.norm(raw, axis=-1)
    d_ok = d_ok & (nrm > 0.5) & mask
    dirs = np.where(d_ok[..., None], raw / np.maximum(nrm, 1e-300)[..., None], 0.0)
    valid = warp_ok & mask
    ahead, a_ok = bicubic(i1w, grid + dirs, mask & valid)
    iu_ok = a_ok & valid
    data_ok = iu_ok & d_ok
    iu = np.where(data_ok, np.where(iu_ok, ahead - i1w, 0.0), 0.0)
    rho0 = np.where(data_ok, i1w - i0, 0.0)
    return i1w, warp_ok, dirs, d_ok, iu, rho0


@dataclass
class Trace:
    max_p_norm: list = field(default_factory=list)
    max_q_norm: list = field(default_factory=list)
    max_du: list = field(default_factory=list)
    mean_abs_du: list = field(default_factory=list)


def level_solve(i0, i1, traj, traj_ok, prm, mask, u0, w0, trace: Trace | None = None):
    """solve_level (solver.py:306-367). Returns (u, w, PDState)."""
    mask = np.asarray(mask, dtype=bool)
    h, wd = mask.shape
    T = edge_tensor(smooth_in_mask(i0, mask, prm.tensor_sigma), mask, prm.beta, prm.eta)
    st = step_sizes(T, mask, prm.alpha0, prm.alpha1, getattr(prm, "regularizer", "tgv"))
    z2 = np.zeros((h, wd, 2))
    s = PDState(u=np.array(u0, dtype=np.float64), v=z2.copy(), p=z2.copy(),
                q=np.zeros((h, wd, 4)), u_bar=np.array(u0, dtype=np.float64), v_bar=z2.copy())
    w = np.array(w0, dtype=np.float64)
    for _ in range(prm.warp_iters):
        _, _, dirs, _, iu, rho0 = linearize(i0, i1, traj, traj_ok, mask, w)
        u_om = s.u.copy()
        s.u_bar = s.u.copy()
        s.v_bar = s.v.copy()
        for _k in range(prm.pd_iters):
            s = pd_cycle(s, T, iu, rho0, u_om, prm, mask, st)
            if trace is not None:
                trace.max_p_norm.append(float(np.max(np.linalg.norm(s.p, axis=-1), initial=0.0)))
                trace.max_q_norm.append(float(np.max(np.linalg.norm(s.q, axis=-1), initial=0.0)))
        du = np.where(mask, np.clip(s.u - u_om, -prm.du_max, prm.du_max), 0.0)
        s.u = u_om + du
        s.u_bar = s.u.copy()
        w = w + du[..., None] * dirs
        if trace is not None:
            trace.max_du.append(float(np.max(np.abs(du), initial=0.0)))
            trace.mean_abs_du.append(float(np.mean(np.abs(du[mask]))) if mask.any() else 0.0)
    return s.u, w, s


def calibrate(i1, rig):
    """calibrate_second_image (solver.py:389-398) -> (i1c, ok)."""
    fld, fok = calibration_field(rig)
    gx, gy = grid_xy(rig.cam0.height, rig.cam0.width)
    vals, ok = bicubic(i1, np.stack([gx, gy], axis=-1) + fld, fov_mask(rig.cam1))
    ok = ok & fok
    return np.where(ok, vals, 0.0), ok


@dataclass
class Solution:
    u: np.ndarray
    w: np.ndarray
    v: np.ndarray
    mask: np.ndarray
    i1c: np.ndarray
    trace: Trace | None = None


def pyramid_solve(i0, i1, rig, prm, traj_override=None, trace: bool = False) -> Solution:
    """solve_pyramid (solver.py:401-452)."""
    i0 = np.asarray(i0, dtype=np.float64)
    i1 = np.asarray(i1, dtype=np.float64)
    if i0.shape != (rig.cam0.height, rig.cam0.width):
        raise ValueError("image 0 does not match camera 0 dimensions")
    if i1.shape != (rig.cam1.height, rig.cam1.width):
        raise ValueError("image 1 does not match camera 1 dimensions")
    m0 = fov_mask(rig.cam0)
    i1c, cok = calibrate(i1, rig)
    smask = m0 & cok
    t_res = residual_translation(rig)
    f0, masks = build_levels(i0, smask, prm.pyramid_levels, prm.pyramid_scale, prm.min_width)
    f1, _ = build_levels(i1c, smask, prm.pyramid_levels, prm.pyramid_scale, prm.min_width)
    tr = Trace() if trace else None
    u = w = s = prev = None
    for lvl in range(len(f0)):
        lm = masks[lvl]
        h, wd = lm.shape
        cam_l = rescale(rig.cam0, h, wd)
        if traj_override is not None:
            dirs, tok = traj_override(cam_l, t_res)
        else:
            dirs, tok = trajectory_field(cam_l, t_res, prm.epsilon_scale)
        if u is None:
            u0, w0 = np.zeros((h, wd)), np.zeros((h, wd, 2))
        else:
            u0, w0 = lift_state(u, w, prev, (h, wd), lm)
        u, w, s = level_solve(f0[lvl], f1[lvl], dirs, tok, prm, lm, u0, w0, tr)
        prev = lm
    return Solution(u=u, w=w, v=s.v, mask=prev, i1c=i1c, trace=tr)


# ---------------------------------------------------------------- post-solve depth
# the solver's warp -> camera-1 correspondence -> depth.

def compose_calibration(w, cal, cal_ok):
    """compose_with_calibration (fields.py:170-182): the camera-1 pixel of x is
    (x + w) + cal(x + w); cal is sampled bicubically under cal_ok."""
    h, wd = cal_ok.shape
    gx, gy = grid_xy(h, wd)
    probe = np.stack([gx, gy], axis=-1) + w
    cal_at, ok = bicubic(cal, probe, cal_ok)
    full = np.where(ok[..., None], w + np.where(ok[..., None], cal_at, 0.0), 0.0)
    return full, ok


def camera1_center(pose):
    """RelativePose.camera1_center (camera.py:267-270): -R^T t."""
    return -np.asarray(pose.rotation).T @ np.asarray(pose.translation)


def triangulate(rig, x0, x1, min_angle=1e-6):
    """triangulate_midpoint (camera.py:317-343): distance along the camera-0 ray
    of the midpoint of the shortest segment between the two rays."""
    x0 = np.asarray(x0, dtype=np.float64)
    x1 = np.asarray(x1, dtype=np.float64)
    r0x, r0y, r0z, v0 = unproject(rig.cam0, x0[..., 0], x0[..., 1])
    r1x, r1y, r1z, v1 = unproject(rig.cam1, x1[..., 0], x1[..., 1])
    R = np.asarray(rig.pose.rotation, dtype=np.float64)
    c1 = camera1_center(rig.pose)
    r0 = np.stack([r0x, r0y, r0z], axis=-1)
    d1 = np.stack([r1x, r1y, r1z], axis=-1) @ R  # R^T r1
    r0 = np.where(v0[..., None], r0, 0.0)
    d1 = np.where(v1[..., None], d1, 0.0)
    b = np.sum(r0 * d1, axis=-1)
    sin_angle = np.linalg.norm(np.cross(r0, d1), axis=-1)
    p = r0 @ c1
    q = d1 @ c1
    ok = v0 & v1 & (sin_angle >= min_angle)
    denom = np.where(ok, 1.0 - b * b, 1.0)
    s0 = (p - b * q) / denom
    ok = ok & (s0 > 0)
    return np.where(ok, s0, np.nan), ok


def depth_from_corr(rig, corr, valid, depth_cap=1e6):
    """depth_from_correspondence (evaluate.py:101-114)."""
    h, wd = valid.shape
    gx, gy = grid_xy(h, wd)
    grid = np.stack([gx, gy], axis=-1)
    depth, ok = triangulate(rig, grid, grid + corr)
    ok = ok & valid
    return np.where(ok, np.minimum(depth, depth_cap), 0.0), ok
