// K5 / K6 / K8: per-warp linearisation, the primal-dual iteration, and the
// warp epilogue. fp32 compute and storage.
//
// Reference: solver.py:279-303 (primal_dual_iterate), solver.py:331-365 (warp
// loop body), solver.py:192-218 (image_derivative_along, thresholding_step),
// rasters.py:144-182 (gradient, divergence, edge indicators).
//
// Layout: every per-pixel quantity is a row-major fp32 plane of h*w (pitch w);
// multi-channel state (v, v_bar, p, q, tensor, steps) is stored as consecutive
// planes so every load of a warp is a coalesced 128-byte line.

#include <stdlib.h>

#include "pd_math.cuh"
#include "warp_math.cuh"

namespace fsb {

constexpr int kBX = 32, kBY = 8;
constexpr bool kNanSampler = true;  // warp_sample_nan (tools/sampler_check.cu: bit-identical to warp_sample_px)
constexpr bool kSplitDefault = true;  // measured faster at 1024^2, 512^2 and 256^2 (C3)

struct PD {
  int h, w;
  size_t n;
  const uint8_t* __restrict__ m;
  const float* __restrict__ T;   // a,b,c planes
  const float* __restrict__ S;   // sigma_p, tau_u, tau_v planes
  const float* __restrict__ iu;
  const float* __restrict__ rho0;
  const float* __restrict__ u_omega;
  float* u; float* u_bar; float* v; float* v_bar; float* p; float* q;
  float lam, alpha0, alpha1, theta, sigma_q, heps;
};

__device__ __forceinline__ bool ex_at(const uint8_t* __restrict__ m, int w, int x, size_t i) {
  return x + 1 < w && m[i] && m[i + 1];
}
__device__ __forceinline__ bool ey_at(const uint8_t* __restrict__ m, int h, int w, int y, size_t i) {
  return y + 1 < h && m[i] && m[i + w];
}

__global__ void k_threshold(const double* __restrict__ u_hat, const double* __restrict__ rho_hat,
                            const double* __restrict__ iu, const double* __restrict__ tau_u,
                            double lam, int64_t n, double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = shrink_step<double>(u_hat[i], rho_hat[i], iu[i], tau_u[i], lam);
}

// Dual ascent with unit-ball projection (solver.py:290-293), one pixel per thread.
template <bool kDiag>
__global__ void __launch_bounds__(256) k_pd_dual(PD s, float* __restrict__ dp, float* __restrict__ dq) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  float pn = 0.f, qn = 0.f;
  if (x < s.w && y < s.h) {
    const size_t i = (size_t)y * s.w + x, n = s.n;
    const bool ex = ex_at(s.m, s.w, x, i), ey = ey_at(s.m, s.h, s.w, y, i);
    const float ub = s.u_bar[i];
    const float vb0 = s.v_bar[i], vb1 = s.v_bar[n + i];
    float gx = 0.f, gy = 0.f, g00 = 0.f, g01 = 0.f, g10 = 0.f, g11 = 0.f;
    if (ex) { gx = s.u_bar[i + 1] - ub; g00 = s.v_bar[i + 1] - vb0; g10 = s.v_bar[n + i + 1] - vb1; }
    if (ey) { gy = s.u_bar[i + s.w] - ub; g01 = s.v_bar[i + s.w] - vb0; g11 = s.v_bar[n + i + s.w] - vb1; }
    float p0 = s.p[i], p1 = s.p[n + i];
    float q0 = s.q[i], q1 = s.q[n + i], q2 = s.q[2 * n + i], q3 = s.q[3 * n + i];
    dual_update(s.T[i], s.T[n + i], s.T[2 * n + i], s.S[i] * s.alpha1, s.sigma_q * s.alpha0, gx,
                gy, g00, g01, g10, g11, vb0, vb1, p0, p1, q0, q1, q2, q3, s.heps);
    s.p[i] = p0; s.p[n + i] = p1;
    s.q[i] = q0; s.q[n + i] = q1; s.q[2 * n + i] = q2; s.q[3 * n + i] = q3;
    if (kDiag) {
      pn = sqrtf(p0 * p0 + p1 * p1);
      qn = sqrtf((q0 * q0 + q1 * q1) + (q2 * q2 + q3 * q3));
    }
  }
  if (kDiag) {
    pn = warp_max(pn); qn = warp_max(qn);
    if ((threadIdx.x & 31) == 0) { atomic_max_nonneg(dp, pn); atomic_max_nonneg(dq, qn); }
  }
}

__device__ __forceinline__ Flux flux_at(const PD& s, size_t i, int x, int y) {
  const size_t n = s.n;
  const bool ex = ex_at(s.m, s.w, x, i), ey = ey_at(s.m, s.h, s.w, y, i);
  return make_flux(s.T[i], s.T[n + i], s.T[2 * n + i], ex, ey, s.p[i], s.p[n + i], s.q[i],
                   s.q[n + i], s.q[2 * n + i], s.q[3 * n + i]);
}

// Primal descent, data-term shrinkage and over-relaxation (solver.py:295-303).
__global__ void __launch_bounds__(256) k_pd_primal(PD s) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= s.w || y >= s.h) return;
  const size_t i = (size_t)y * s.w + x, n = s.n;
  const Flux f = flux_at(s, i, x, y);
  const Flux fl = x > 0 ? flux_at(s, i - 1, x - 1, y) : Flux{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const Flux fu = y > 0 ? flux_at(s, i - s.w, x, y - 1) : Flux{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  // backward differences in the reference's order: ((f - f_left) + f_y) - f_up
  const float dv = ((f.px - fl.px) + f.py) - fu.py;
  const float d0 = ((f.q0x - fl.q0x) + f.q0y) - fu.q0y;
  const float d1 = ((f.q1x - fl.q1x) + f.q1y) - fu.q1y;
  float u = s.u[i], v0 = s.v[i], v1 = s.v[n + i], ub, vb0, vb1;
  primal_update(dv, d0, d1, s.S[n + i], s.S[2 * n + i], s.iu[i], s.rho0[i], s.u_omega[i], s.p[i],
                s.p[n + i], s.lam, s.alpha0, s.alpha1, s.theta, u, v0, v1, ub, vb0, vb1);
  s.u[i] = u;
  s.v[i] = v0; s.v[n + i] = v1;
  s.u_bar[i] = ub;
  s.v_bar[i] = vb0; s.v_bar[n + i] = vb1;
}

// Warp prologue part 1 (solver.py:332-337): i1w at x+w, trajectory direction
// at x+w (renormalised, valid if norm > 0.5 and in mask).
__global__ void __launch_bounds__(256) k_warp_sample(fsb_level L) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  const SampleSrc S{L.i1, L.mask, L.traj, L.traj_ok, reinterpret_cast<const float4*>(L.packed),
                    L.full16, L.h, L.w};
  float iw;
  bool iok, dok;
  float2 d;
  warp_sample_px(S, x, y, reinterpret_cast<const float2*>(L.wv)[i], L.mask[i] != 0, iw, iok, d,
                 dok);
  L.i1w[i] = iw;
  L.i1w_ok[i] = iok;
  reinterpret_cast<float2*>(L.dirs)[i] = d;
  L.dir_ok[i] = dok;
}

// Fused warp prologue (solver.py:332-346 with image_derivative_along 192-202):
// i1w / directions at x + w for the output tile plus a 3-px halo into shared
// memory, then I_u = i1w(x + dir) - i1w(x) from that tile, and rho0. One
// kernel, no global round trip of i1w between the two gathers. Pixels outside
// the level mask are skipped: their i1w_ok / dir_ok are false by definition
// (solver.py:336, 339), so nothing downstream reads their samples.
template <int TX, int TY>
__global__ void __launch_bounds__(256) k_warp_prologue(fsb_level L) {
  constexpr int H = 3;  // |dir| <= 1 (+1 ulp) puts the stencil base within 2 px
  constexpr int SW = TX + 2 * H, SH = TY + 2 * H;
  static_assert(SW <= 64, "row validity words are 64-bit");
  __shared__ float s_iw[SH * SW];
  __shared__ uint8_t s_okb[SH * SW];
  __shared__ unsigned long long s_okrow[SH];  // bit c of row r: i1w_ok of tile pixel (r, c)
  __shared__ float2 s_dir[TY * TX];
  __shared__ uint8_t s_dok[TY * TX];
  const int ox = blockIdx.x * TX, oy = blockIdx.y * TY;
  const SampleSrc S{L.i1, L.mask, L.traj, L.traj_ok, reinterpret_cast<const float4*>(L.packed),
                    L.full16, L.h, L.w};
  // flat loop over the halo tile; (r, c) advanced incrementally (no division)
  constexpr int kStep = 256;  // == blockDim.x (launch_bounds)
  int r = threadIdx.x / SW, c = threadIdx.x - (threadIdx.x / SW) * SW;
  for (int k = threadIdx.x; k < SH * SW; k += kStep) {
    const int gx = ox - H + c, gy = oy - H + r;
    float iw = 0.f;
    bool iok = false, dok = false;
    float2 d = make_float2(0.f, 0.f);
    if ((unsigned)gx < (unsigned)L.w && (unsigned)gy < (unsigned)L.h) {
      const size_t gi = (size_t)gy * L.w + gx;
      if (L.mask[gi])
        warp_sample_px(S, gx, gy, reinterpret_cast<const float2*>(L.wv)[gi], true, iw, iok, d,
                       dok);
      const int tr = r - H, tc = c - H;
      if (tr >= 0 && tr < TY && tc >= 0 && tc < TX) {
        s_dir[tr * TX + tc] = d;
        s_dok[tr * TX + tc] = dok;
        L.i1w[gi] = iw;
        L.i1w_ok[gi] = iok;
        reinterpret_cast<float2*>(L.dirs)[gi] = d;
        L.dir_ok[gi] = dok;
      }
    }
    s_iw[k] = iw;
    s_okb[k] = iok;
    r += kStep / SW;
    c += kStep % SW;
    if (c >= SW) { c -= SW; ++r; }
  }
  __syncthreads();
  {  // pack the validity bytes into one 64-bit word per tile row (warp ballots)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int r = warp; r < SH; r += nwarps) {
      const unsigned lo = __ballot_sync(0xffffffffu, lane < SW && s_okb[r * SW + lane]);
      const unsigned hi =
          __ballot_sync(0xffffffffu, lane + 32 < SW && s_okb[r * SW + lane + 32]);
      if (lane == 0) s_okrow[r] = (unsigned long long)lo | ((unsigned long long)hi << 32);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < TY * TX; k += blockDim.x) {
    const int tr = k / TX, tc = k - tr * TX;
    const int gx = ox + tc, gy = oy + tr;
    if (gx >= L.w || gy >= L.h) continue;
    const size_t gi = (size_t)gy * L.w + gx;
    const int si = (tr + H) * SW + (tc + H);
    const bool own_ok = (s_okrow[tr + H] >> (tc + H)) & 1ull;
    float iu = 0.f, rho0 = 0.f;
    if (own_ok && s_dok[k]) {
      const float2 d = s_dir[k];
      int ix, iy;
      float fx, fy;
      if (split_off(gx, gy, d.x, d.y, L.h, L.w, ix, iy, fx, fy)) {
        const int lx = ix - (ox - H), ly = iy - (oy - H);  // tile-local stencil base
        unsigned okb = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
          okb |= (unsigned)((s_okrow[ly + a - 1] >> (lx - 1)) & 0xFull) << (4 * a);
        float ahead;
        if (okb && bicubic_bits<1, float, false>(s_iw, okb, SW, lx, ly, fx, fy, &ahead)) {
          const float iw = s_iw[si];
          iu = ahead - iw;
          rho0 = iw - L.i0[gi];
        }
      }
    }
    L.iu[gi] = iu;
    L.rho0[gi] = rho0;
  }
}

// Per-level gather tables: packed {i1, traj} texels and the all-16-taps-valid
// flags of the mask and of traj_ok.
__global__ void k_pack_level(fsb_level L) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  // NaN marks an invalid tap (mask / traj_ok false): warp_sample_nan reads the
  // validity from the texel itself; warp_sample_px only reads all-valid texels
  const float2 t = reinterpret_cast<const float2*>(L.traj)[i];
  const float qnan = __int_as_float(0x7fc00000);
  const bool tok = L.traj_ok[i] != 0;
  reinterpret_cast<float4*>(L.packed)[i] =
      make_float4(L.mask[i] ? L.i1[i] : qnan, tok ? t.x : qnan, tok ? t.y : qnan, 0.f);
  uint8_t fl = 0;
  if (x >= 1 && x + 2 < L.w && y >= 1 && y + 2 < L.h) {
    bool am = true, at = true;
#pragma unroll
    for (int a = -1; a <= 2; ++a)
#pragma unroll
      for (int b = -1; b <= 2; ++b) {
        const size_t k = (size_t)(y + a) * L.w + (x + b);
        am = am && L.mask[k];
        at = at && L.traj_ok[k];
      }
    fl = (am ? 1 : 0) | (at ? 2 : 0);
  }
  L.full16[i] = fl;
  if (L.maskf) L.maskf[i] = L.mask[i] ? 1.f : 0.f;
}

// Warp prologue part 2 (solver.py:339-346 with image_derivative_along 192-202):
// I_u = i1w(x+dir) - i1w(x) on taps valid in mask & warp_ok; rho0; resets.
__global__ void __launch_bounds__(256) k_warp_linearize(fsb_level L) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x, n = (size_t)L.h * L.w;
  const float2 d = reinterpret_cast<const float2*>(L.dirs)[i];
  float ahead[1];
  bool ok = bicubic_sample<1, float>(L.i1w, L.i1w_ok, L.h, L.w, (double)x + (double)d.x,
                                     (double)y + (double)d.y, ahead);
  const float i1w = L.i1w[i];
  const bool data_ok = ok && L.i1w_ok[i] && L.dir_ok[i];
  L.iu[i] = data_ok ? ahead[0] - i1w : 0.f;
  L.rho0[i] = data_ok ? i1w - L.i0[i] : 0.f;
  const float u = L.u[i];
  L.u_omega[i] = u;
  L.u_bar[i] = u;
  L.v_bar[i] = L.v[i];
  L.v_bar[n + i] = L.v[n + i];
}

// Warp epilogue (solver.py:356-360): clip the increment, accumulate u and w.
template <bool kDiag>
__global__ void __launch_bounds__(256) k_warp_finish(fsb_level L, float du_max, float* dmax,
                                                     double* partials) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  float adu = 0.f;
  if (x < L.w && y < L.h) {
    const size_t i = (size_t)y * L.w + x;
    const float uo = L.u_omega[i];
    float du = fminf(fmaxf(L.u[i] - uo, -du_max), du_max);
    if (!L.mask[i]) du = 0.f;
    const float u = uo + du;
    L.u[i] = u;
    L.u_bar[i] = u;
    const float2 d = reinterpret_cast<const float2*>(L.dirs)[i];
    float2 wv = reinterpret_cast<float2*>(L.wv)[i];
    wv.x = wv.x + du * d.x;
    wv.y = wv.y + du * d.y;
    reinterpret_cast<float2*>(L.wv)[i] = wv;
    adu = fabsf(du);
  }
  if (kDiag) {
    // max is order-free; the sum goes to fixed per-block slots (deterministic)
    __shared__ double ssum[8];
    __shared__ float smax[8];
    float mx = warp_max(adu);
    double sm = warp_sum((double)adu);
    int lane = threadIdx.x & 31, wid = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0) { ssum[wid] = sm; smax[wid] = mx; }
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      double t = 0.0; float mm = 0.f;
      int nw = (blockDim.x * blockDim.y) >> 5;
      for (int k = 0; k < nw; ++k) { t += ssum[k]; mm = fmaxf(mm, smax[k]); }
      partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
      atomic_max_nonneg(dmax, mm);
    }
  }
}

// mean |du| over the mask: ordered sum of the block partials / mask count.
__global__ void k_mean_finish(const double* __restrict__ partials, int nparts,
                              const uint8_t* __restrict__ m, size_t n, double* out) {
  __shared__ double sh[256];
  __shared__ unsigned long long cnt[256];
  double t = 0.0;
  unsigned long long c = 0;
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) t += partials[k];
  for (size_t k = threadIdx.x; k < n; k += blockDim.x) c += m[k] ? 1 : 0;
  sh[threadIdx.x] = t; cnt[threadIdx.x] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) { sh[threadIdx.x] += sh[threadIdx.x + s]; cnt[threadIdx.x] += cnt[threadIdx.x + s]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = cnt[0] ? sh[0] / (double)cnt[0] : 0.0;
}

PD make_pd(const fsb_level* L, const fsb_params* prm) {
  PD s;
  s.h = L->h; s.w = L->w; s.n = (size_t)L->h * L->w;
  s.m = L->mask; s.T = L->tensor; s.S = L->steps; s.iu = L->iu; s.rho0 = L->rho0;
  s.u_omega = L->u_omega; s.u = L->u; s.u_bar = L->u_bar; s.v = L->v; s.v_bar = L->v_bar;
  s.p = L->p; s.q = L->q;
  s.lam = (float)prm->lam; s.alpha0 = (float)prm->alpha0; s.alpha1 = (float)prm->alpha1;
  s.theta = (float)prm->theta;
  s.sigma_q = (float)sigma_q_of(prm);  // solver.py:265
  s.heps = (float)huber_eps_of(prm);
  return s;
}

int pd_iterate_internal(const fsb_level* L, const fsb_params* prm, int iters, float* diag_p,
                        float* diag_q, cudaStream_t st) {
  PD s = make_pd(L, prm);
  dim3 blk(kBX, kBY), grd = grid2d(L->w, L->h, blk);
  for (int k = 0; k < iters; ++k) {
    if (diag_p && diag_q)
      k_pd_dual<true><<<grd, blk, 0, st>>>(s, diag_p + k, diag_q + k);
    else
      k_pd_dual<false><<<grd, blk, 0, st>>>(s, nullptr, nullptr);
    k_pd_primal<<<grd, blk, 0, st>>>(s);
  }
  return launch_status();
}

int warp_linearize_internal(const fsb_level* L, cudaStream_t st) {
  dim3 blk(kBX, kBY), grd = grid2d(L->w, L->h, blk);
  k_warp_sample<<<grd, blk, 0, st>>>(*L);
  k_warp_linearize<<<grd, blk, 0, st>>>(*L);
  return launch_status();
}

int warp_sample_internal(const fsb_level* L, cudaStream_t st) {
  dim3 blk(kBX, kBY), grd = grid2d(L->w, L->h, blk);
  k_warp_sample<<<grd, blk, 0, st>>>(*L);
  return launch_status();
}

// Split prologue for large levels: the samples at x + w once per pixel (no
// halo re-sampling), then I_u from the sampled image in global memory (L1/L2
// resident) in a second kernel. Same arithmetic as k_warp_prologue.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_sample_px(fsb_level L) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  float iw = 0.f;
  bool iok = false, dok = false;
  float2 d = make_float2(0.f, 0.f);
  // the warp is loaded with the mask byte, not after it (one round trip less)
  const uint8_t mk = L.mask[i];
  const float2 wv = reinterpret_cast<const float2*>(L.wv)[i];
  if (mk) {
    if (kNanSampler)
      warp_sample_nan(reinterpret_cast<const float4*>(L.packed), L.h, L.w, x, y, wv, iw, iok, d,
                      dok);
    else {
      const SampleSrc S{L.i1, L.mask, L.traj, L.traj_ok,
                        reinterpret_cast<const float4*>(L.packed), L.full16, L.h, L.w};
      warp_sample_px(S, x, y, wv, true, iw, iok, d, dok);
    }
  }
  // i1w is stored NaN where invalid (warp_ok & mask false): k_iu_px reads the
  // tap validity from the values themselves, one load per tap
  L.i1w[i] = iok ? iw : __int_as_float(0x7fc00000);
  L.i1w_ok[i] = iok;
  reinterpret_cast<float2*>(L.dirs)[i] = d;
  L.dir_ok[i] = dok;
}

__global__ void __launch_bounds__(256) k_iu_px(fsb_level L) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  float iu = 0.f, rho0 = 0.f;
  // loaded together, ahead of their conditions (one round trip less)
  const float iw = L.i1w[i];
  const bool dk = L.dir_ok[i];
  const float2 d = reinterpret_cast<const float2*>(L.dirs)[i];
  const float i0 = L.i0[i];
  if (!isnan(iw) && dk) {
    int ix, iy;
    float fx, fy;
    if (split_off(x, y, d.x, d.y, L.h, L.w, ix, iy, fx, fy)) {
      // 16 taps (out-of-image taps invalid), validity = not NaN; the validity
      // bits are only formed when the Catmull-Rom sum says a tap is invalid
      float t[16];
      const bool inner = ix >= 1 && ix + 2 < L.w && iy >= 1 && iy + 2 < L.h;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int r = iy + a - 1, c = ix + b - 1;
          const bool in = inner || ((unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w);
          t[4 * a + b] = in ? __ldg(L.i1w + (size_t)r * L.w + c) : __int_as_float(0x7fc00000);
        }
      float wx[4], wy[4], cub = 0.f;
      cubic_weights(fx, wx);
      cubic_weights(fy, wy);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cub = tap_acc(cub, wy[a] * wx[b], t[4 * a + b]);
      unsigned okb = 0xFFFFu;
      if (isnan(cub)) {
        okb = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) okb |= (isnan(t[k]) ? 0u : 1u) << k;
      }
      float ahead = cub;
      if (okb == 0xFFFFu || bicubic_regs(t, okb, fx, fy, ahead)) {
        iu = ahead - iw;
        rho0 = iw - i0;
      }
    }
  }
  L.iu[i] = iu;
  L.rho0[i] = rho0;
}

int warp_prologue_internal(const fsb_level* L, cudaStream_t st) {
  // FSB_PROLOGUE=fused|split (tuning); default by level size. Read once
  // (function-local statics initialise thread-safely).
  static const int mode = [] {
    const char* e = getenv("FSB_PROLOGUE");
    return e ? (e[0] == 's' ? 1 : (e[0] == 'f' ? 2 : 0)) : 0;
  }();
  const bool big = (size_t)L->w * L->h >= (size_t)512 * 512;
  if (mode == 1 || (mode == 0 && kSplitDefault)) {
    dim3 blk(kBX, kBY), grd = grid2d(L->w, L->h, blk);
    // 6 CTAs / SM (42 registers; spills only on the masked fallback) hides the
    // gather latency on >= 512^2 levels: C3 1024^2 7.83 -> 7.49 ms, bench 69.5
    // -> 71.5 frames/s (A/B, 3 x 30 steps); at 256^2 the unconstrained build
    // is 0.05 ms faster (tools/level_times.py)
    if (big) k_sample_px<6><<<grd, blk, 0, st>>>(*L);
    else k_sample_px<1><<<grd, blk, 0, st>>>(*L);
    k_iu_px<<<grd, blk, 0, st>>>(*L);  // (8 CTAs / SM measured slower)
    return launch_status();
  }
  // small levels: 16 x 16 tiles so the grid still spreads over the SMs
  if (big) {
    dim3 grd((L->w + 31) / 32, (L->h + 31) / 32);
    k_warp_prologue<32, 32><<<grd, 256, 0, st>>>(*L);
  } else {
    dim3 grd((L->w + 15) / 16, (L->h + 15) / 16);
    k_warp_prologue<16, 16><<<grd, 256, 0, st>>>(*L);
  }
  return launch_status();
}

int pack_level_internal(const fsb_level* L, cudaStream_t st) {
  dim3 blk(kBX, kBY), grd = grid2d(L->w, L->h, blk);
  k_pack_level<<<grd, blk, 0, st>>>(*L);
  return launch_status();
}

__global__ void k_mask_to_float(const uint8_t* __restrict__ m, size_t n, float* __restrict__ f) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = m[i] ? 1.f : 0.f;
}

int mask_to_float_internal(const uint8_t* m, size_t n, float* f, cudaStream_t st) {
  k_mask_to_float<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(m, n, f);
  return launch_status();
}

int mean_finish_internal(const double* partials, int nparts, const uint8_t* mask, size_t n,
                         double* out, cudaStream_t st) {
  k_mean_finish<<<1, 256, 0, st>>>(partials, nparts, mask, n, out);
  return launch_status();
}

size_t level_partials_internal(int h, int w) {
  dim3 blk(kBX, kBY), grd = grid2d(w, h, blk);
  return (size_t)grd.x * grd.y;
}

int warp_finish_internal(const fsb_level* L, const fsb_params* prm, float* dmax, double* dmean,
                         cudaStream_t st) {
  dim3 blk(kBX, kBY), grd = grid2d(L->w, L->h, blk);
  if (dmax && dmean && L->partials) {
    k_warp_finish<true><<<grd, blk, 0, st>>>(*L, (float)prm->du_max, dmax, L->partials);
    k_mean_finish<<<1, 256, 0, st>>>(L->partials, (int)(grd.x * grd.y), L->mask,
                                     (size_t)L->h * L->w, dmean);
  } else {
    k_warp_finish<false><<<grd, blk, 0, st>>>(*L, (float)prm->du_max, nullptr, nullptr);
  }
  return launch_status();
}

}  // namespace fsb

extern "C" int fsb_thresholding_step(const double* u_hat, const double* rho_hat, const double* iu,
                                     const double* tau_u, double lam, int64_t n, double* out,
                                     void* stream) {
  if (n < 0 || (n > 0 && (!u_hat || !rho_hat || !iu || !tau_u || !out))) return FSB_EINVAL;
  if (n == 0) return FSB_OK;
  fsb::k_threshold<<<(unsigned)((n + 255) / 256), 256, 0, fsb::as_stream(stream)>>>(
      u_hat, rho_hat, iu, tau_u, lam, n, out);
  return fsb::launch_status();
}
