// Per-pixel arithmetic of one primal-dual cycle, shared by every PD kernel
// (the one-iteration-per-launch kernels in pd.cu and the temporally blocked
// tile kernel in pd_block.cu) so all paths round identically.
//
// Reference: solver.py:279-303 (primal_dual_iterate), solver.py:205-218
// (thresholding_step), solver.py:164-168 (apply_tensor), solver.py:221-223
// (_project_unit), rasters.py:144-172 (masked gradient / divergence).
#pragma once

#include "fsb_common.cuh"

namespace fsb {

// thresholding_step (solver.py:205-218): closed-form prox of
// lam*|rho_hat + (u - u_hat) iu| + (u - u_hat)^2 / (2 tau_u); iu == 0 passes through.
template <typename T>
FSB_INLINE T shrink_step(T u_hat, T rho_hat, T g, T tau_u, T lam) {
  const T tl = tau_u * lam;
  const T th = (tl * g) * g;
  T step;
  if (rho_hat < -th) step = tl * g;
  else if (rho_hat > th) step = -(tl * g);
  else step = g != T(0) ? -(rho_hat / g) : T(0);
  return g != T(0) ? u_hat + step : u_hat;
}

// Dual ascent + unit-ball projection (solver.py:290-293). Forward differences
// of u_bar / v_bar are passed in already masked by the edge indicators.
//   sp = sigma_p * alpha1, sq = sigma_q * alpha0.
FSB_INLINE void dual_update(float a, float b, float c, float sp, float sq, float gx, float gy,
                            float g00, float g01, float g10, float g11, float vb0, float vb1,
                            float& p0, float& p1, float& q0, float& q1, float& q2, float& q3,
                            float heps = 0.f) {
  p0 = p0 + sp * ((a * gx + b * gy) - vb0);
  p1 = p1 + sp * ((b * gx + c * gy) - vb1);
  if (heps > 0.f) {  // Huber-TV: prox of the conjugate, p / (1 + sp eps)
    const float k = __frcp_rn(1.f + sp * heps);
    p0 = p0 * k;
    p1 = p1 * k;
  }
  // x / max(1, |x|) (solver.py:221-223): identity inside the unit ball (exactly
  // as the reference, divisor 1), x * rsqrt(|x|^2) outside (<= 2 ulp, fp32 path).
  const float pn2 = p0 * p0 + p1 * p1;
  const float rp = pn2 > 1.f ? rsqrtf(pn2) : 1.f;
  p0 = p0 * rp;
  p1 = p1 * rp;
  q0 = q0 + sq * g00;
  q1 = q1 + sq * g01;
  q2 = q2 + sq * g10;
  q3 = q3 + sq * g11;
  const float qn2 = (q0 * q0 + q1 * q1) + (q2 * q2 + q3 * q3);
  const float rq = qn2 > 1.f ? rsqrtf(qn2) : 1.f;
  q0 = q0 * rq;
  q1 = q1 * rq;
  q2 = q2 * rq;
  q3 = q3 * rq;
}

// Edge-masked fluxes of one pixel: the x / y components of T p and of the two
// q blocks, zero where the forward edge leaves the mask (Dirichlet, rasters.py:166-167).
struct Flux {
  float px, py, q0x, q0y, q1x, q1y;
};

FSB_INLINE Flux make_flux(float a, float b, float c, bool ex, bool ey, float p0, float p1,
                          float q0, float q1, float q2, float q3) {
  Flux f;
  f.px = ex ? a * p0 + b * p1 : 0.f;
  f.py = ey ? b * p0 + c * p1 : 0.f;
  f.q0x = ex ? q0 : 0.f;
  f.q0y = ey ? q1 : 0.f;
  f.q1x = ex ? q2 : 0.f;
  f.q1y = ey ? q3 : 0.f;
  return f;
}

// Primal descent with data-term shrinkage and over-relaxation
// (solver.py:295-302). div* are backward-difference divergences of the fluxes.
FSB_INLINE void primal_update(float div_tp, float div_q0, float div_q1, float tau_u, float tau_v,
                              float iu, float rho0, float u_omega, float p0, float p1,
                              float lam, float alpha0, float alpha1, float theta, float& u,
                              float& v0, float& v1, float& u_bar, float& v_bar0, float& v_bar1) {
  const float u_hat = u + (tau_u * alpha1) * div_tp;
  const float rho_hat = rho0 + (u_hat - u_omega) * iu;
  const float u_new = shrink_step<float>(u_hat, rho_hat, iu, tau_u, lam);
  const float v0n = v0 + tau_v * (alpha0 * div_q0 + alpha1 * p0);
  const float v1n = v1 + tau_v * (alpha0 * div_q1 + alpha1 * p1);
  u_bar = u_new + theta * (u_new - u);
  v_bar0 = v0n + theta * (v0n - v0);
  v_bar1 = v1n + theta * (v1n - v1);
  u = u_new;
  v0 = v0n;
  v1 = v1n;
}

}  // namespace fsb

namespace fsb {

// ---------------------------------------------------------------- exact variants
// The same cycle with IEEE division / square root throughout, for the fp64
// parity path (the reference's own operation order, solver.py:290-302).

template <typename T>
FSB_INLINE void dual_update_exact(T a, T b, T c, T sp, T sq, T gx, T gy, T g00, T g01, T g10,
                                  T g11, T vb0, T vb1, T& p0, T& p1, T& q0, T& q1, T& q2,
                                  T& q3, T heps = T(0)) {
  p0 = p0 + sp * ((a * gx + b * gy) - vb0);
  p1 = p1 + sp * ((b * gx + c * gy) - vb1);
  if (heps > T(0)) {
    const T dd = T(1) + sp * heps;
    p0 = p0 / dd;
    p1 = p1 / dd;
  }
  // x / max(1, |x|): inside the unit ball the reference divides by exactly 1.0
  // (an identity), so only |x|^2 > 1 takes the sqrt and the divisions; there
  // sqrt(|x|^2) >= 1 is max(1, |x|) itself. Bit-identical, far fewer fp64 ops.
  const T pn2 = p0 * p0 + p1 * p1;
  if (pn2 > T(1)) {
    const T pd = sqrt(pn2);
    p0 = p0 / pd;
    p1 = p1 / pd;
  }
  q0 = q0 + sq * g00;
  q1 = q1 + sq * g01;
  q2 = q2 + sq * g10;
  q3 = q3 + sq * g11;
  const T qn2 = ((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3;
  if (qn2 > T(1)) {
    const T qd = sqrt(qn2);
    q0 = q0 / qd;
    q1 = q1 / qd;
    q2 = q2 / qd;
    q3 = q3 / qd;
  }
}

template <typename T>
struct FluxT {
  T px, py, q0x, q0y, q1x, q1y;
};

template <typename T>
FSB_INLINE FluxT<T> make_flux_exact(T a, T b, T c, bool ex, bool ey, T p0, T p1, T q0, T q1,
                                    T q2, T q3) {
  FluxT<T> f;
  f.px = ex ? a * p0 + b * p1 : T(0);
  f.py = ey ? b * p0 + c * p1 : T(0);
  f.q0x = ex ? q0 : T(0);
  f.q0y = ey ? q1 : T(0);
  f.q1x = ex ? q2 : T(0);
  f.q1y = ey ? q3 : T(0);
  return f;
}

template <typename T>
FSB_INLINE void primal_update_exact(T div_tp, T div_q0, T div_q1, T tau_u, T tau_v, T iu, T rho0,
                                    T u_omega, T p0, T p1, T lam, T alpha0, T alpha1, T theta,
                                    T& u, T& v0, T& v1, T& u_bar, T& v_bar0, T& v_bar1) {
  const T u_hat = u + (tau_u * alpha1) * div_tp;
  const T rho_hat = rho0 + (u_hat - u_omega) * iu;
  const T u_new = shrink_step<T>(u_hat, rho_hat, iu, tau_u, lam);
  const T v0n = v0 + tau_v * (alpha0 * div_q0 + alpha1 * p0);
  const T v1n = v1 + tau_v * (alpha0 * div_q1 + alpha1 * p1);
  u_bar = u_new + theta * (u_new - u);
  v_bar0 = v0n + theta * (v0n - v0);
  v_bar1 = v1n + theta * (v1n - v1);
  u = u_new;
  v0 = v0n;
  v1 = v1n;
}

}  // namespace fsb
