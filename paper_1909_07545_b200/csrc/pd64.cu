// The float64 path — the drop-in default and the credited path: the whole
// solve_pyramid frame in float64 storage and arithmetic. Geometry, setup and
// the samplers are compiled with -fmad=false (NumPy's rounding order); the
// primal-dual cycles run in k64_tile (pd64_tile.cu, FMA contraction, IEEE
// division / sqrt). The one-cycle-per-launch kernels below (k64_dual /
// k64_primal / k64_finish) remain as the FSB_PD64=plain cross-check.
//
// Why float64: at the reference defaults (N=50 warps) the problem is at its
// conditioning limit — ANY float32 rounding of the state or the constants moves
// the p99 disparity past 1e-2 px against the reference
// (profiles/r01_precision_study.txt). This path reproduces the
// reference to round-off at every N (C3: p99 3.3e-6 px).
//
// Reference: solver.py:306-452 (solve_level, solve_pyramid) with the stages of
// solver.py:279-303 and :332-365; rasters.py:57-141 (bicubic).

#include <stdlib.h>
#include <string.h>

#include <vector>

#include "pd_math.cuh"
#include "pd64_block.cuh"
#include "sample64.cuh"

namespace fsb {

// defined in the other translation units
int trajectory_field64_internal(const fsb_camera* cam, const double t[3], double eps_scale,
                                double depth, double* dirs, uint8_t* ok, void* scratch,
                                size_t scratch_bytes, cudaStream_t st);
size_t traj_scratch_bytes_internal(int w, int h);
int fov_mask_internal(const fsb_camera* cam, uint8_t* mask, int* iters, cudaStream_t st);
int calibrate64_internal(const fsb_rig* rig, const double* i1, const uint8_t* mask1, double* i1c,
                         uint8_t* ok, int* iters0, cudaStream_t st);
int pyramid_shapes_internal(int h, int w, int levels, double scale, int min_width, int* shapes,
                            int max_levels);
int downsample64_internal(const double* src, const uint8_t* mask, int fh, int fw, double* dst,
                          uint8_t* dmask, int ch, int cw, cudaStream_t st);
int upsample64_internal(const double* u, const double* wv, const uint8_t* mask, int sh, int sw,
                        const uint8_t* dmask, int dh, int dw, double* uo, double* wo,
                        cudaStream_t st);
size_t level_setup_scratch_internal(int h, int w);
int level_setup64_internal(const double* i0, const uint8_t* mask, int h, int w,
                           const fsb_params* prm, double* tensor, double* steps, void* scratch,
                           size_t scratch_bytes, cudaStream_t st);
int mean_finish_internal(const double* partials, int nparts, const uint8_t* mask, size_t n,
                         double* out, cudaStream_t st);
int pack64_internal(const double* i1, const uint8_t* mask, const double* traj,
                    const uint8_t* tok, int h, int w, double4* tex, cudaStream_t st);
int sample_nan64_internal(const P64& L, int bx, int by, cudaStream_t st);
int linearize_nan64_internal(const P64& L, int bx, int by, cudaStream_t st);
bool side_stream_for(cudaStream_t main, cudaStream_t* side, cudaEvent_t** ev);  // solver.cu
bool pd64_level_fits(int w, int h);  // pd64_level.cu
int pd64_level_ctas(int w, int h);
int pd64_level_launch(const P64& P, const double* T, const double* S, const uint32_t* ecode,
                      double* u, double* v, double* wv, double* scratch2, double lam,
                      double alpha0, double alpha1, double theta, double sigma_q, double heps,
                      double du_max, int N, int K, const LvlDiag* diag, cudaStream_t st);

}  // namespace fsb

// Live per-warp phase events at one pyramid level (fsb200.h fsb_phase_timer):
// three events per warp on the solve stream: before the sampling kernels,
// between sampling and the primal-dual launches, after the last PD launch.
struct fsb_phase_timer {
  int level;          // 0 = finest
  int cap;            // warps with events
  int used;           // warps recorded by the last solve
  int pd_launches;    // PD launches per warp at that level (last solve)
  int level_h, level_w;
  cudaEvent_t* ev;    // 3 * cap
};

namespace fsb {

namespace {

constexpr int kBX = 32, kBY = 8;
constexpr int kMaxLevels = 32;

struct L64 {
  int h, w;
  size_t n;
  const double* i0; const double* i1; const uint8_t* mask;
  const double* traj; const uint8_t* traj_ok;
  double* T; double* S;
  double* u; double* ub; double* v; double* vb; double* p; double* q;
  double* wv; double* uo; double* iu; double* rho0; double* i1w; uint8_t* i1w_ok;
  double* dirs; uint8_t* dir_ok;
  double* partials;
  // second state set for the blocked cycles (pd64_block.cu); nullptr = one-cycle kernels
  double *u2, *ub2, *v2, *vb2, *p2, *q2;
  // per-pixel flags: bit0 all 16 bicubic taps in mask, bit1 all in traj_ok (nullptr = off)
  uint8_t* full16;
  // k64_tile: per-pixel edge codes and the level's tile work list
  uint32_t* ecode;
  int* tiles;
  double4* tex;  // NaN-encoded packed texels of the level (sample64.cu)
  double* lvl_partials;     // k64_level's per-warp per-CTA |du| sums (diagnostics)
  size_t lvl_partials_cap;  // their count
};

__device__ __forceinline__ bool ex_at(const uint8_t* __restrict__ m, int w, int x, size_t i) {
  return x + 1 < w && m[i] && m[i + 1];
}
__device__ __forceinline__ bool ey_at(const uint8_t* __restrict__ m, int h, int w, int y, size_t i) {
  return y + 1 < h && m[i] && m[i + w];
}

// All-16-taps-valid flags of a level (mask -> bit0, traj_ok -> bit1) for the
// sampler's unmasked fast path.
__global__ void k64_full16(L64 L) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  uint8_t fl = 0;
  if (x >= 1 && x + 2 < L.w && y >= 1 && y + 2 < L.h) {
    bool am = true, at = true;
    for (int a = -1; a <= 2; ++a)
      for (int b = -1; b <= 2; ++b) {
        const size_t k = (size_t)(y + a) * L.w + (x + b);
        am = am && L.mask[k];
        at = at && L.traj_ok[k];
      }
    fl = (am ? 1 : 0) | (at ? 2 : 0);
  }
  L.full16[(size_t)y * L.w + x] = fl;
}

// solver.py:332-337
// The loads of the fast path are issued speculatively: the warp position
// does not wait for the mask byte, and the 16 taps do not wait for the
// full16 flag (inner stencils only; the flag decides which result is used),
// so the chain is wv -> taps instead of mask -> wv -> flag -> taps. The fast
// branch is the all-valid Catmull-Rom branch of bicubic_bits (same weights,
// same order); everything else takes the masked gathers.
__global__ void k64_sample(L64 L) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  const uint8_t mk = L.mask[i];
  const double2 wv = reinterpret_cast<const double2*>(L.wv)[i];
  const double px = (double)x + wv.x, py = (double)y + wv.y;
  double iv[1], dr[2];
  bool wok = false, dok = false, fast = false;
  int ix, iy;
  double fx, fy;
  if (L.full16 && split_pos<double>(px, py, L.h, L.w, ix, iy, fx, fy) && ix >= 1 &&
      ix + 2 < L.w && iy >= 1 && iy + 2 < L.h) {
    const size_t base = (size_t)(iy - 1) * L.w + (ix - 1);
    double ti[16];
    double2 tt[16];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        ti[4 * a + b] = __ldg(L.i1 + base + (size_t)a * L.w + b);
        tt[4 * a + b] = __ldg(reinterpret_cast<const double2*>(L.traj) + base + (size_t)a * L.w + b);
      }
    if (L.full16[(size_t)iy * L.w + ix] == 3) {
      double wx[4], wy[4];
      cubic_weights(fx, wx);
      cubic_weights(fy, wy);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double wt = wy[a] * wx[b];
          a0 = tap_acc(a0, wt, ti[4 * a + b]);
          a1 = tap_acc(a1, wt, tt[4 * a + b].x);
          a2 = tap_acc(a2, wt, tt[4 * a + b].y);
        }
      iv[0] = a0; dr[0] = a1; dr[1] = a2;
      wok = dok = fast = true;
    }
  }
  if (!mk) {  // i1w_ok = warp_ok & mask and dir_ok & mask are false: unused
    L.i1w[i] = 0.0;
    L.i1w_ok[i] = 0;
    L.dirs[2 * i] = 0.0; L.dirs[2 * i + 1] = 0.0;
    L.dir_ok[i] = 0;
    return;
  }
  if (!fast) {
    wok = bicubic_sample<1, double, double>(L.i1, L.mask, L.h, L.w, px, py, iv);
    dok = bicubic_sample<2, double, double>(L.traj, L.traj_ok, L.h, L.w, px, py, dr);
  }
  double d0 = 0.0, d1 = 0.0;
  if (dok) {
    const double nrm = sqrt(dr[0] * dr[0] + dr[1] * dr[1]);
    if (nrm > 0.5) { d0 = dr[0] / fmax(nrm, 1e-300); d1 = dr[1] / fmax(nrm, 1e-300); }
    else dok = false;
  }
  L.i1w[i] = wok ? iv[0] : 0.0;
  L.i1w_ok[i] = wok;
  L.dirs[2 * i] = d0; L.dirs[2 * i + 1] = d1;
  L.dir_ok[i] = dok;
}

// solver.py:339-346 with image_derivative_along 192-202
// Loads issued ahead of their conditions (flags, direction, the 16 taps and
// their validity bytes together): two dependent memory round trips instead of
// four. The all-valid case is bicubic_bits' Catmull-Rom branch on the
// preloaded taps (same weights, same order); partial stencils take
// bicubic_bits itself.
__global__ void k64_linearize(L64 L, bool reset) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x, n = L.n;
  const double i1w = L.i1w[i], i0 = L.i0[i];
  const bool ok0 = L.i1w_ok[i] && L.dir_ok[i];
  const double2 dv = reinterpret_cast<const double2*>(L.dirs)[i];
  // data_ok needs i1w_ok and dir_ok: only then is the gather needed
  bool data_ok = false;
  double ahead = 0.0;
  int ix, iy;
  double fx, fy;
  if (split_pos<double>((double)x + dv.x, (double)y + dv.y, L.h, L.w, ix, iy, fx, fy)) {
    const bool inner = ix >= 1 && ix + 2 < L.w && iy >= 1 && iy + 2 < L.h;
    if (inner) {
      const size_t base = (size_t)(iy - 1) * L.w + (ix - 1);
      double t[16];
      unsigned okb = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const size_t k = base + (size_t)a * L.w + b;
          t[4 * a + b] = L.i1w[k];
          okb |= (L.i1w_ok[k] ? 1u : 0u) << (4 * a + b);
        }
      if (ok0 && okb == 0xFFFFu) {
        double wx[4], wy[4];
        cubic_weights(fx, wx);
        cubic_weights(fy, wy);
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc = tap_acc(acc, wy[a] * wx[b], t[4 * a + b]);
        ahead = acc;
        data_ok = true;
      } else if (ok0) {
        double o[1];
        data_ok = bicubic_bits<1, double, true, double>(L.i1w, okb, L.w, ix, iy, fx, fy, o);
        ahead = o[0];
      }
    } else if (ok0) {
      double o[1];
      data_ok = bicubic_at<1, double, true, double>(L.i1w, L.i1w_ok, L.h, L.w, ix, iy, fx, fy, o);
      ahead = o[0];
    }
  }
  L.iu[i] = data_ok ? ahead - i1w : 0.0;
  L.rho0[i] = data_ok ? i1w - i0 : 0.0;
  if (!reset) return;  // the blocked path resets in its first launch (A.first)
  const double u = L.u[i];
  L.uo[i] = u;
  L.ub[i] = u;
  L.vb[i] = L.v[i];
  L.vb[n + i] = L.v[n + i];
}

// solver.py:290-293
template <bool kDiag>
__global__ void k64_dual(L64 L, double alpha0, double alpha1, double sigma_q, double heps,
                         float* dp, float* dq) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  double pn = 0.0, qn = 0.0;
  if (x < L.w && y < L.h) {
    const size_t i = (size_t)y * L.w + x, n = L.n;
    const bool ex = ex_at(L.mask, L.w, x, i), ey = ey_at(L.mask, L.h, L.w, y, i);
    const double ub = L.ub[i], vb0 = L.vb[i], vb1 = L.vb[n + i];
    double gx = 0.0, gy = 0.0, g00 = 0.0, g01 = 0.0, g10 = 0.0, g11 = 0.0;
    if (ex) { gx = L.ub[i + 1] - ub; g00 = L.vb[i + 1] - vb0; g10 = L.vb[n + i + 1] - vb1; }
    if (ey) { gy = L.ub[i + L.w] - ub; g01 = L.vb[i + L.w] - vb0; g11 = L.vb[n + i + L.w] - vb1; }
    double p0 = L.p[i], p1 = L.p[n + i];
    double q0 = L.q[i], q1 = L.q[n + i], q2 = L.q[2 * n + i], q3 = L.q[3 * n + i];
    dual_update_exact<double>(L.T[i], L.T[n + i], L.T[2 * n + i], L.S[i] * alpha1,
                              sigma_q * alpha0, gx, gy, g00, g01, g10, g11, vb0, vb1, p0, p1, q0,
                              q1, q2, q3, heps);
    L.p[i] = p0; L.p[n + i] = p1;
    L.q[i] = q0; L.q[n + i] = q1; L.q[2 * n + i] = q2; L.q[3 * n + i] = q3;
    if (kDiag) {
      pn = sqrt(p0 * p0 + p1 * p1);
      qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
    }
  }
  if (kDiag) {
    pn = warp_max(pn); qn = warp_max(qn);
    if ((threadIdx.x & 31) == 0) {
      atomic_max_nonneg(dp, (float)pn);
      atomic_max_nonneg(dq, (float)qn);
    }
  }
}

__device__ __forceinline__ FluxT<double> flux64(const L64& L, size_t i, int x, int y) {
  const size_t n = L.n;
  const bool ex = ex_at(L.mask, L.w, x, i), ey = ey_at(L.mask, L.h, L.w, y, i);
  return make_flux_exact<double>(L.T[i], L.T[n + i], L.T[2 * n + i], ex, ey, L.p[i], L.p[n + i],
                                 L.q[i], L.q[n + i], L.q[2 * n + i], L.q[3 * n + i]);
}

// solver.py:295-303
__global__ void k64_primal(L64 L, double lam, double alpha0, double alpha1, double theta) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x, n = L.n;
  const FluxT<double> z = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const FluxT<double> f = flux64(L, i, x, y);
  const FluxT<double> fl = x > 0 ? flux64(L, i - 1, x - 1, y) : z;
  const FluxT<double> fu = y > 0 ? flux64(L, i - L.w, x, y - 1) : z;
  const double dv = ((f.px - fl.px) + f.py) - fu.py;
  const double d0 = ((f.q0x - fl.q0x) + f.q0y) - fu.q0y;
  const double d1 = ((f.q1x - fl.q1x) + f.q1y) - fu.q1y;
  double u = L.u[i], v0 = L.v[i], v1 = L.v[n + i], ub, vb0, vb1;
  primal_update_exact<double>(dv, d0, d1, L.S[n + i], L.S[2 * n + i], L.iu[i], L.rho0[i], L.uo[i],
                              L.p[i], L.p[n + i], lam, alpha0, alpha1, theta, u, v0, v1, ub, vb0,
                              vb1);
  L.u[i] = u; L.v[i] = v0; L.v[n + i] = v1;
  L.ub[i] = ub; L.vb[i] = vb0; L.vb[n + i] = vb1;
}

// solver.py:356-365
template <bool kDiag>
__global__ void k64_finish(L64 L, double du_max, float* dmax, double* dmax64) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  double adu = 0.0;
  if (x < L.w && y < L.h) {
    const size_t i = (size_t)y * L.w + x;
    const double uo = L.uo[i];
    double du = fmin(fmax(L.u[i] - uo, -du_max), du_max);
    if (!L.mask[i]) du = 0.0;
    const double u = uo + du;
    L.u[i] = u;
    L.ub[i] = u;
    L.wv[2 * i] = L.wv[2 * i] + du * L.dirs[2 * i];
    L.wv[2 * i + 1] = L.wv[2 * i + 1] + du * L.dirs[2 * i + 1];
    adu = fabs(du);
  }
  if (kDiag) {
    __shared__ double ssum[8];
    __shared__ double smax[8];
    const double mx = warp_max(adu), sm = warp_sum(adu);
    const int lane = threadIdx.x & 31, wid = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0) { ssum[wid] = sm; smax[wid] = mx; }
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      double t = 0.0, m = 0.0;
      const int nw = (blockDim.x * blockDim.y) >> 5;
      for (int k = 0; k < nw; ++k) { t += ssum[k]; m = fmax(m, smax[k]); }
      L.partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
      if (dmax64) atomic_max_nonneg(dmax64, m);
      else atomic_max_nonneg(dmax, (float)m);
    }
  }
}

// NaN-encoded sampled image -> (value or 0, validity), the masked-gather convention.
__global__ void k64_nan_split(double* v, uint8_t* ok, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = v[i];
  const bool k = !isnan(x);
  ok[i] = k;
  v[i] = k ? x : 0.0;
}

__global__ void k64_and_mask(const uint8_t* a, const uint8_t* b, size_t n, uint8_t* o) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i] && b[i];
}

// interleave two planes of v into (H, W, 2)
__global__ void k64_interleave(const double* v, size_t n, double* out) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { out[2 * i] = v[i]; out[2 * i + 1] = v[n + i]; }
}

struct Carve {
  char* base;
  size_t off = 0;
  template <typename X>
  X* take(size_t count) {
    size_t bytes = align_up(count * sizeof(X));
    X* p = base ? reinterpret_cast<X*>(base + off) : nullptr;
    off += bytes;
    return p;
  }
};

struct Plan64 {
  int nlev, shapes[2 * kMaxLevels];
  size_t n0;
  uint8_t *mask0, *mask1, *i1c_ok, *solve_mask;
  int* iters;
  double *lvl_i0[kMaxLevels], *lvl_i1[kMaxLevels], *traj[kMaxLevels];
  uint8_t *lvl_mask[kMaxLevels], *traj_ok[kMaxLevels];
  void* traj_scratch; size_t traj_bytes;
  void* setup_scratch; size_t setup_bytes;
  // the two primal-dual state sets, each one block of 12 planes of the level's
  // size (u, v x2, p x2, q x4, u_bar, v_bar x2: the 3-D TMA box of k64_tma)
  double *setA, *setB;
  double* carry_u;  // the finished level's u, read by the next level's upsample
  double *wv[2], *i1w, *dirs, *partials;
  double* lvl_partials;  // k64_level diagnostics: N x CTAs partial sums
  size_t lvl_partials_n;
  uint8_t *i1w_ok, *dir_ok;
  // per-level setup products (filled ahead on the side stream); cst: one block
  // of 10 planes per level — tensor a, b, c, steps sigma_p, tau_u, tau_v, I_u,
  // rho0, u_omega, edge code (k64_tma's constant box)
  double* cst[kMaxLevels];
  uint8_t* f16l[kMaxLevels];
  uint32_t* ecl[kMaxLevels];
  int* tll[kMaxLevels];
  double4* texl[kMaxLevels];
  size_t bytes;
};

size_t partial_count(int h, int w) {  // k64_finish blocks or blocked-kernel tiles (halo <= 5)
  const size_t blocks = (size_t)((w + kBX - 1) / kBX) * ((h + kBY - 1) / kBY);
  size_t tiles = pd64_block_tiles(w, h, 5);
  if (pd64_ctile_partials(w, h) > tiles) tiles = pd64_ctile_partials(w, h);
  return (blocks > tiles ? blocks : tiles) + 64;
}

int plan64(const fsb_rig* rig, const fsb_params* prm, void* base, Plan64& P) {
  const int H = rig->cam0.height, W = rig->cam0.width;
  int n = pyramid_shapes_internal(H, W, prm->pyramid_levels, prm->pyramid_scale, prm->min_width,
                                  P.shapes, kMaxLevels);
  if (n < 1 || n > kMaxLevels) return FSB_EINVAL;
  P.nlev = n;
  P.n0 = (size_t)H * W;
  const size_t n0 = P.n0, n1 = (size_t)rig->cam1.height * rig->cam1.width;
  Carve c{static_cast<char*>(base)};
  P.mask0 = c.take<uint8_t>(n0); P.mask1 = c.take<uint8_t>(n1);
  P.i1c_ok = c.take<uint8_t>(n0); P.solve_mask = c.take<uint8_t>(n0);
  P.iters = c.take<int>(64);
  for (int l = 0; l < n; ++l) {
    size_t np = (size_t)P.shapes[2 * l] * P.shapes[2 * l + 1];
    P.lvl_i0[l] = l == 0 ? nullptr : c.take<double>(np);
    P.lvl_i1[l] = l == 0 ? nullptr : c.take<double>(np);
    P.lvl_mask[l] = l == 0 ? nullptr : c.take<uint8_t>(np);
    P.traj[l] = c.take<double>(2 * np);
    P.traj_ok[l] = c.take<uint8_t>(np);
  }
  P.traj_bytes = traj_scratch_bytes_internal(W, H);
  P.traj_scratch = c.take<char>(P.traj_bytes);
  P.setup_bytes = level_setup_scratch_internal(H, W);
  P.setup_scratch = c.take<char>(P.setup_bytes);
  for (int k = 0; k < 2; ++k) P.wv[k] = c.take<double>(2 * n0);
  P.setA = c.take<double>(12 * n0); P.setB = c.take<double>(12 * n0);
  P.carry_u = c.take<double>(n0);
  P.i1w = c.take<double>(n0); P.dirs = c.take<double>(2 * n0);
  P.i1w_ok = c.take<uint8_t>(n0); P.dir_ok = c.take<uint8_t>(n0);
  P.partials = c.take<double>(partial_count(H, W));
  P.lvl_partials_n = (size_t)prm->warp_iters * 16;
  P.lvl_partials = c.take<double>(P.lvl_partials_n);
  for (int l = 0; l < n; ++l) {
    const int lh = P.shapes[2 * l], lw = P.shapes[2 * l + 1];
    const size_t np = (size_t)lh * lw;
    P.cst[l] = c.take<double>(10 * np);
    P.f16l[l] = c.take<uint8_t>(np); P.ecl[l] = c.take<uint32_t>(np);
    P.tll[l] = c.take<int>(partial_count(lh, lw) + 1); P.texl[l] = c.take<double4>(np);
  }
  P.bytes = c.off;
  return FSB_OK;
}

fsb_camera scaled(const fsb_camera& c, int h, int w) {  // camera.py:66-77
  fsb_camera o = c;
  double sx = (double)w / (double)c.width, sy = (double)h / (double)c.height;
  o.width = w; o.height = h;
  o.fx = c.fx * sx; o.fy = c.fy * sy;
  o.cx = (c.cx + 0.5) * sx - 0.5;
  o.cy = (c.cy + 0.5) * sy - 0.5;
  return o;
}

// FSB_PD64=plain runs the one-cycle-per-launch kernels (reference for the
// blocked kernel in tests/tools); default: blocked, halo 2.
// Blocked PD kernel choice. Default: k64_tile over the level's work list of
// mask tiles (K64_TILEL), and on the halo-2 levels whose layout allows it the
// TMA-fed k64_tma (K64_TMA, pd64_tma.cu) over the same list. FSB_PD64K=tilel:
// k64_tile everywhere; =tile: k64_tile over every tile (masked gathers, no work
// list); =block: the round-1 k64_block (pd64_block.cu). The persistent
// cp.async-pipelined variants measured slower.
enum { K64_BLOCK = 0, K64_TILE = 1, K64_TILEL = 3, K64_TMA = 4, K64_CTILE = 5 };
int pd64_kernel_choice() {
  static const int v = [] {
    const char* e = getenv("FSB_PD64K");
    if (e && strcmp(e, "block") == 0) return (int)K64_BLOCK;
    if (e && strcmp(e, "tile") == 0) return (int)K64_TILE;
    if (e && strcmp(e, "tilel") == 0) return (int)K64_TILEL;
    if (e && strcmp(e, "tma") == 0) return (int)K64_TMA;
    return (int)K64_CTILE;
  }();
  return v;
}
int pd64_kernel_for(int) {
  const int k = pd64_kernel_choice();
  // k64_tma / k64_ctile are picked per level (level_cfg64)
  return k == K64_TMA || k == K64_CTILE ? (int)K64_TILEL : k;
}
// Persistent, phase-staggered k64_tile on the halo-2 (large) levels: 2 CTAs per
// SM stride over the work list and the second half starts 2 us late, so an SM's
// two CTAs keep opposite phases (C3 1024^2: 16.5 -> 15.9 ms). The small levels
// (halo 3 / 5, one wave) keep one tile per CTA. FSB_PD64_PERSIST=<ns> (0 = off).
int pd64_persist(int halo) {
  static const int v = [] {
    const char* e = getenv("FSB_PD64_PERSIST");
    return e ? atoi(e) : 2000;
  }();
  return halo == 2 ? v : 0;
}

int pd64_launch(const B64& A0, int halo, cudaStream_t st) {
  static const int zero = [] {  // FSB_PD64_ZERO=1: timing experiment, load/store only
    const char* e = getenv("FSB_PD64_ZERO");
    return e && e[0] == '1';
  }();
  B64 A = A0;
  if (zero && halo <= 3) {
    A.iters = 0;
    if (pd64_kernel_for(halo) == K64_TILEL || pd64_kernel_for(halo) == K64_TILE)
      return pd64_tile_launch_unchecked(A, halo, st);
  }
  switch (pd64_kernel_for(halo)) {
    case K64_TILE: case K64_TILEL: return pd64_tile_launch(A, halo, st);
    default: return pd64_block_launch(A, halo, st);
  }
}

size_t pd64_tiles(int w, int h, int halo) {
  switch (pd64_kernel_for(halo)) {
    case K64_TILE: case K64_TILEL: return pd64_tile_count(w, h, halo);
    default: return pd64_block_tiles(w, h, halo);
  }
}

int pd64_halo() {
  static const int h = [] {
    const char* e = getenv("FSB_PD64");
    return e && e[0] == 'p' ? 0 : (e && e[0] >= '1' && e[0] <= '3' ? e[0] - '0' : 2);
  }();
  return h;
}

L64 swapped(const L64& L) {
  L64 o = L;
  o.u = L.u2; o.ub = L.ub2; o.v = L.v2; o.vb = L.vb2; o.p = L.p2; o.q = L.q2;
  o.u2 = L.u; o.ub2 = L.ub; o.v2 = L.v; o.vb2 = L.vb; o.p2 = L.p; o.q2 = L.q;
  return o;
}

// Per-level kernel configuration (deterministic from the level size and the
// tuning environment, so the side-stream setup and the solve agree).
struct LevelCfg64 {
  int halo, kern;
  bool listed, pro_nan;
};

// k64_tma's layout: each state set and the constants one block of planes
// (pd64_block.cuh)
bool tma_layout64(const L64& L) {
  const size_t n = L.n;
  auto set_ok = [n](const double* u, const double* v, const double* p, const double* q,
                    const double* ub, const double* vb) {
    return u && v == u + n && p == u + 3 * n && q == u + 5 * n && ub == u + 9 * n &&
           vb == u + 10 * n;
  };
  return set_ok(L.u, L.v, L.p, L.q, L.ub, L.vb) && set_ok(L.u2, L.v2, L.p2, L.q2, L.ub2, L.vb2) &&
         L.T && L.S == L.T + 3 * n && L.iu == L.T + 6 * n && L.rho0 == L.T + 7 * n &&
         L.uo == L.T + 8 * n;
}

LevelCfg64 level_cfg64(const L64& L) {
  LevelCfg64 c;
  // latency-bound small levels: 5 cycles per launch when those tiles fit
  // two resident CTAs per SM (C3: 64^2, 128^2), else R = 2 (throughput)
  int halo = L.u2 ? pd64_halo() : 0;
  if (halo == 2 && getenv("FSB_PD64") == nullptr) {
    if (pd64_tile_count(L.w, L.h, 5) <= 2 * 148) halo = 5;
    else if (pd64_tile_count(L.w, L.h, 3) <= 2 * 148) halo = 3;
  }
  if (halo > 0) {  // FSB_PD64_HALO_L="w:R,w:R" overrides per level width (tuning)
    const char* e = getenv("FSB_PD64_HALO_L");
    for (const char* p = e; p && *p;) {
      const int lw = atoi(p);
      const char* colon = strchr(p, ':');
      if (!colon) break;
      const int r = atoi(colon + 1);
      if (lw == L.w && (r == 1 || r == 2 || r == 3 || r == 5)) halo = r;
      p = strchr(colon, ',');
      if (p) ++p;
    }
  }
  c.halo = halo;
  c.kern = halo > 0 ? pd64_kernel_for(halo) : -1;
  // k64_ctile on levels of 512^2 and more (C3 1024^2: 16.0 -> 13.5 ms per
  // frame, 512^2: 4.64 -> 4.57 ms); FSB_CTILE_MIN=<pixels> moves the cut.
  static const size_t ctile_min = [] {
    const char* e = getenv("FSB_CTILE_MIN");
    return e ? (size_t)atoll(e) : (size_t)512 * 512;
  }();
  const int choice = pd64_kernel_choice();
  if (c.kern == K64_TILEL && halo > 1 && choice == K64_CTILE && tma_layout64(L) &&
      (size_t)L.w * L.h >= ctile_min && pd64_ctile_usable(L.w, L.h)) {
    c.kern = K64_CTILE;
    c.halo = pd64_ctile_halo();
  } else if (c.kern == K64_TILEL && halo == 2 && choice == K64_TMA && tma_layout64(L) &&
             pd64_tma_usable(L.w, L.h) &&
             pd64_tma_tile_count(L.w, L.h) == pd64_tile_count(L.w, L.h, 2)) {
    c.kern = K64_TMA;
  }
  c.listed = c.kern == K64_TILEL || c.kern == K64_TMA || c.kern == K64_CTILE;
  // Warp prologue: the NaN-encoded texel kernels (sample64.cu) on levels up to
  // 256^2, where the masked-gather chains of k64_sample / k64_linearize are
  // latency floors (C3: 64^2 -0.18 ms, 128^2 -0.34 ms per frame); on larger
  // levels the 32-byte texels cost more DRAM traffic than they save
  // (1024^2 +0.8 ms). FSB_PRO64=old / new forces one kind everywhere.
  static const int pro_mode = [] {
    const char* e = getenv("FSB_PRO64");
    return e && strcmp(e, "old") == 0 ? 0 : (e && strcmp(e, "new") == 0 ? 2 : 1);
  }();
  c.pro_nan =
      halo > 0 && (pro_mode == 2 || (pro_mode == 1 && (size_t)L.w * L.h <= 256 * 256));
  return c;
}

// Level setup that depends only on the pyramid and the rig (solver.py:319-321
// and the gather / tile tables): runs ahead on the side stream.
int level_prepare64(const L64& L, const fsb_params* prm, const LevelCfg64& c, void* scratch,
                    size_t scratch_bytes, cudaStream_t st) {
  int rc = level_setup64_internal(L.i0, L.mask, L.h, L.w, prm, L.T, L.S, scratch, scratch_bytes,
                                  st);
  if (rc) return rc;
  if (c.listed) {  // per-level edge codes and tile work list
    // k64_tma / k64_ctile: edge codes also as the 10th constant plane
    const bool tma = c.kern == K64_TMA || c.kern == K64_CTILE;
    rc = pd64_edge_codes(L.mask, L.w, L.h, L.ecode, tma ? L.T + 9 * L.n : nullptr, st);
    if (rc) return rc;
    if (c.kern == K64_CTILE) rc = pd64_ctile_list(L.mask, L.w, L.h, L.tiles, st);
    else if (c.kern == K64_TMA) rc = pd64_tma_tile_list(L.mask, L.w, L.h, L.tiles, st);
    else rc = pd64_tile_tile_list(L.mask, L.w, L.h, c.halo, L.tiles, st);
    if (rc) return rc;
  }
  if (c.pro_nan) {
    rc = pack64_internal(L.i1, L.mask, L.traj, L.traj_ok, L.h, L.w, L.tex, st);
    if (rc) return rc;
  } else if (L.full16) {  // all-16-taps-valid flags of the masked-gather sampler
    dim3 b(kBX, kBY);
    k64_full16<<<grid2d(L.w, L.h, b), b, 0, st>>>(L);
  }
  return launch_status();
}

int solve_level64(const L64& L0, const fsb_params* prm, const fsb_diag* diag, int64_t pd_off,
                  int64_t warp_off, void* scratch, size_t scratch_bytes, cudaStream_t st,
                  fsb_phase_timer* tm = nullptr, bool prepared = false) {
  L64 L = L0;  // L's state pointers follow the ping-pong of the blocked cycles
  const size_t n = L.n;
  const LevelCfg64 cfg = level_cfg64(L);
  const int halo = cfg.halo, kern = cfg.kern;
  const bool listed = cfg.listed, pro_nan = cfg.pro_nan;
  int rc = FSB_OK;
  if (!prepared) {
    rc = level_prepare64(L, prm, cfg, scratch, scratch_bytes, st);
    if (rc) return rc;
  }
  cudaMemsetAsync(L.v, 0, 2 * n * sizeof(double), st);
  cudaMemsetAsync(L.vb, 0, 2 * n * sizeof(double), st);
  cudaMemsetAsync(L.p, 0, 2 * n * sizeof(double), st);
  cudaMemsetAsync(L.q, 0, 4 * n * sizeof(double), st);
  cudaMemcpyAsync(L.ub, L.u, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (L.u2) {  // the blocked kernel skips masked pixels: their state is 0 in both sets
    cudaMemsetAsync(L.u2, 0, n * sizeof(double), st);
    cudaMemsetAsync(L.ub2, 0, n * sizeof(double), st);
    cudaMemsetAsync(L.v2, 0, 2 * n * sizeof(double), st);
    cudaMemsetAsync(L.vb2, 0, 2 * n * sizeof(double), st);
    cudaMemsetAsync(L.p2, 0, 2 * n * sizeof(double), st);
    cudaMemsetAsync(L.q2, 0, 4 * n * sizeof(double), st);
  }
  const int N = prm->warp_iters, K = prm->pd_iters;
  dim3 blk(kBX, kBY), grd = grid2d(L.w, L.h, blk);
  const bool dpq = diag && diag->max_p_norm && diag->max_q_norm;
  const bool ddu = diag && (diag->max_du || diag->max_du_f64) && diag->mean_abs_du;
  Tma64Level tmaps;  // k64_tma's / k64_ctile's tensor maps: set 0 = L0's primary set
  Ctile64Maps cmaps;
  if (kern == K64_TMA && !pd64_tma_level_maps(&tmaps, L0.u, L0.u2, L0.T, L0.w, L0.h))
    return FSB_EINVAL;
  if (kern == K64_CTILE && !pd64_ctile_maps(&cmaps, L0.u, L0.u2, L0.T, L0.w, L0.h))
    return FSB_EINVAL;
  // per-tile partial sums of |du| (DIAG): count of the kernel's tile / CTA slots
  const size_t nparts =
      kern == K64_CTILE ? pd64_ctile_partials(L.w, L.h) : pd64_tiles(L.w, L.h, halo);
  P64 PL;
  PL.h = L.h; PL.w = L.w; PL.i0 = L.i0; PL.mask = L.mask; PL.tex = L.tex; PL.wv = L.wv;
  PL.i1wn = L.i1w; PL.dirs = L.dirs; PL.dir_ok = L.dir_ok; PL.iu = L.iu; PL.rho0 = L.rho0;
  // a small level: the whole warp loop in one cluster launch (k64_level,
  // pd64_level.cu); the sampled-image scratch is 2 level planes of the
  // finest-level i1w buffer. With diagnostics the kernel reduces them itself
  // (the same kernels run with and without: bit-identical results).
  if (pro_nan && listed && L.u2 && pd64_level_fits(L.w, L.h) &&
      (!ddu || (size_t)N * pd64_level_ctas(L.w, L.h) <= L.lvl_partials_cap)) {
    LvlDiag ld;
    memset(&ld, 0, sizeof(ld));
    if (dpq) { ld.p = diag->max_p_norm + pd_off; ld.q = diag->max_q_norm + pd_off; }
    if (ddu) {
      if (diag->max_du_f64) ld.du64 = diag->max_du_f64 + warp_off;
      else ld.du = diag->max_du + warp_off;
      ld.partials = L.lvl_partials;
    }
    rc = pd64_level_launch(PL, L.T, L.S, L.ecode, L.u, L.v, L.wv, L.i1w, prm->lam,
                           prm->alpha0, prm->alpha1, prm->theta, sigma_q_of(prm),
                           huber_eps_of(prm), prm->du_max, N, K, (dpq || ddu) ? &ld : nullptr,
                           st);
    if (rc) return rc;
    const int nc = pd64_level_ctas(L.w, L.h);
    for (int wi = 0; ddu && wi < N; ++wi) {
      rc = mean_finish_internal(L.lvl_partials + (size_t)wi * nc, nc, L.mask, n,
                                diag->mean_abs_du + warp_off + wi, st);
      if (rc) return rc;
    }
    if (tm) {  // phase timer: the level is one launch
      tm->used = 0;
      tm->level_h = L.h; tm->level_w = L.w;
    }
    return launch_status();
  }
  for (int wi = 0; wi < N; ++wi) {
    const bool timed = tm && wi < tm->cap;
    if (timed) cudaEventRecord(tm->ev[3 * wi], st);
    if (pro_nan) {
      rc = sample_nan64_internal(PL, kBX, kBY, st);
      if (rc) return rc;
      rc = linearize_nan64_internal(PL, kBX, kBY, st);
      if (rc) return rc;
    } else {
      k64_sample<<<grd, blk, 0, st>>>(L);
      k64_linearize<<<grd, blk, 0, st>>>(L, halo == 0);
    }
    if (timed) cudaEventRecord(tm->ev[3 * wi + 1], st);
    int pd_launches = 0;
    for (int k = 0; halo > 0 && k < K;) {  // blocked: `it` cycles per launch, src -> dst
      const int it = K - k < halo ? K - k : halo;
      B64 A;
      A.h = L.h; A.w = L.w; A.n = n; A.mask = L.mask; A.T = L.T; A.S = L.S;
      A.iu = L.iu; A.rho0 = L.rho0; A.uo = L.uo; A.first = k == 0;
      A.su = L.u; A.sub = L.ub; A.sv = L.v; A.svb = L.vb; A.sp = L.p; A.sq = L.q;
      A.du = L.u2; A.dub = L.ub2; A.dv = L.v2; A.dvb = L.vb2; A.dp = L.p2; A.dq = L.q2;
      A.lam = prm->lam; A.alpha0 = prm->alpha0; A.alpha1 = prm->alpha1; A.theta = prm->theta;
      A.sigma_q = sigma_q_of(prm); A.heps = huber_eps_of(prm);
      A.iters = it;
      const int64_t slot = pd_off + (int64_t)wi * K + k;
      A.diag_p = dpq ? diag->max_p_norm + slot : nullptr;
      A.diag_q = dpq ? diag->max_q_norm + slot : nullptr;
      A.fin = k + it == K;  // the warp's last cycles: fused clip / accumulate
      A.du_max = prm->du_max;
      A.dirs = L.dirs; A.wv = L.wv;
      A.diag_du = (A.fin && ddu && diag->max_du) ? diag->max_du + warp_off + wi : nullptr;
      A.diag_du64 = (A.fin && ddu && diag->max_du_f64) ? diag->max_du_f64 + warp_off + wi : nullptr;
      if (A.diag_du64) A.diag_du = nullptr;
      A.partials = L.partials;
      A.ecode = listed ? L.ecode : nullptr;
      A.tiles = listed ? L.tiles : nullptr;
      A.persist = pd64_persist(halo);
      if (listed && (A.diag_du || A.diag_du64))  // tiles off the work list keep a zero partial sum
        cudaMemsetAsync(L.partials, 0, nparts * sizeof(double), st);
      const int src = L.u == L0.u ? 0 : 1;
      rc = kern == K64_CTILE ? pd64_ctile_launch(A, cmaps, src, st)
           : kern == K64_TMA ? pd64_tma_launch(A, tmaps, src, st)
                             : pd64_launch(A, halo, st);
      if (rc) return rc;
      ++pd_launches;
      L = swapped(L);
      k += it;
      if (k == K && ddu) {
        rc = mean_finish_internal(L.partials, (int)nparts, L.mask, n,
                                  diag->mean_abs_du + warp_off + wi, st);
        if (rc) return rc;
      }
    }
    if (halo > 0) {  // the blocked launches fused k64_finish
      if (timed) {
        cudaEventRecord(tm->ev[3 * wi + 2], st);
        tm->used = wi + 1;
        tm->pd_launches = pd_launches;
        tm->level_h = L.h; tm->level_w = L.w;
      }
      continue;
    }
    for (int k = 0; halo == 0 && k < K; ++k) {
      if (dpq) {
        const int64_t slot = pd_off + (int64_t)wi * K + k;
        k64_dual<true><<<grd, blk, 0, st>>>(L, prm->alpha0, prm->alpha1, sigma_q_of(prm),
                                            huber_eps_of(prm), diag->max_p_norm + slot,
                                            diag->max_q_norm + slot);
      } else {
        k64_dual<false><<<grd, blk, 0, st>>>(L, prm->alpha0, prm->alpha1, sigma_q_of(prm),
                                             huber_eps_of(prm), nullptr, nullptr);
      }
      k64_primal<<<grd, blk, 0, st>>>(L, prm->lam, prm->alpha0, prm->alpha1, prm->theta);
    }
    if (ddu) {
      k64_finish<true><<<grd, blk, 0, st>>>(
          L, prm->du_max, diag->max_du ? diag->max_du + warp_off + wi : nullptr,
          diag->max_du_f64 ? diag->max_du_f64 + warp_off + wi : nullptr);
      rc = mean_finish_internal(L.partials, (int)(grd.x * grd.y), L.mask, n,
                                diag->mean_abs_du + warp_off + wi, st);
      if (rc) return rc;
    } else {
      k64_finish<false><<<grd, blk, 0, st>>>(L, prm->du_max, nullptr, nullptr);
    }
  }
  if (L.u != L0.u) {  // the level result back into the primary set (u carries on, v is output)
    cudaMemcpyAsync(L0.u, L.u, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(L0.v, L.v, 2 * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  return launch_status();
}

bool params_ok64(const fsb_params* p) {
  if (!p) return false;
  if (!(p->lam > 0 && p->alpha0 > 0 && p->alpha1 > 0 && p->beta > 0 && p->eta > 0)) return false;
  if (!(p->du_max > 0) || p->warp_iters < 1 || p->pd_iters < 1) return false;
  if (p->regularizer < FSB_REG_TGV || p->regularizer > FSB_REG_HUBER) return false;
  if (p->regularizer == FSB_REG_HUBER && !(p->huber_eps > 0)) return false;
  return p->pyramid_levels >= 1 && p->pyramid_scale > 1.0;
}

}  // namespace

// Event recorded inside a float64 graph capture once mask / i1c are final
// (fsb_graph_create_f64 sets it around the capture; thread-local like the
// capture mode).
thread_local cudaEvent_t g_early_event = nullptr;
void set_early_output_event64(cudaEvent_t ev) { g_early_event = ev; }

size_t solve_pyramid64_bytes(const fsb_rig* rig, const fsb_params* prm) {
  if (!rig || !params_ok64(prm)) return 0;
  Plan64 P;
  if (plan64(rig, prm, nullptr, P)) return 0;
  return P.bytes;
}

int solve_pyramid64(const fsb_rig* rig, const fsb_params* prm, const double* i0, const double* i1,
                    const double* const* traj_dirs, const uint8_t* const* traj_okv, void* ws,
                    size_t ws_bytes, double* u_out, double* w_out, double* v_out,
                    uint8_t* mask_out, double* i1c, const fsb_diag* diag, cudaStream_t st,
                    fsb_phase_timer* tm = nullptr) {
  if (!rig || !params_ok64(prm) || !i0 || !i1 || !ws || !u_out || !w_out || !v_out ||
      !mask_out || !i1c)
    return FSB_EINVAL;
  if ((traj_dirs == nullptr) != (traj_okv == nullptr)) return FSB_EINVAL;
  Plan64 P;
  int rc = plan64(rig, prm, nullptr, P);
  if (rc) return rc;
  if (ws_bytes < P.bytes) return FSB_ENOSPC;
  plan64(rig, prm, ws, P);
  const fsb_rig& r = *rig;
  double t_res[3];
  for (int k = 0; k < 3; ++k)  // translation_only_rig (fields.py:159-167)
    t_res[k] = (r.rotation[0 * 3 + k] * r.translation[0] + r.rotation[1 * 3 + k] * r.translation[1]) +
               r.rotation[2 * 3 + k] * r.translation[2];
  if (!traj_dirs && t_res[0] == 0.0 && t_res[1] == 0.0 && t_res[2] == 0.0) return FSB_EDOMAIN;
  const size_t n0 = P.n0;
  const int N = prm->warp_iters, K = prm->pd_iters;
  if (diag) {
    const int64_t npd = (int64_t)P.nlev * N * K, nw = (int64_t)P.nlev * N;
    if (diag->max_p_norm) cudaMemsetAsync(diag->max_p_norm, 0, npd * sizeof(float), st);
    if (diag->max_q_norm) cudaMemsetAsync(diag->max_q_norm, 0, npd * sizeof(float), st);
    if (diag->max_du) cudaMemsetAsync(diag->max_du, 0, nw * sizeof(float), st);
    if (diag->max_du_f64) cudaMemsetAsync(diag->max_du_f64, 0, nw * sizeof(double), st);
  }
  // Side stream (shared with the float32 driver, solver.cu side_ctx): the
  // trajectory fields of every level (rig only) start there at once; after the
  // pyramids, every level's setup runs there coarse to fine with one event per
  // level, which the level's solve on the caller's stream waits for. The small
  // levels leave most SMs idle, so the finer levels' setup fills them.
  // FSB_OVERLAP=0 keeps everything on the caller's stream.
  cudaStream_t ss = st;
  cudaEvent_t* ev = nullptr;
  const bool side = !tm && side_stream_for(st, &ss, &ev);
  if (!side) ss = st;
  if (side) {
    cudaEventRecord(ev[0], st);
    cudaStreamWaitEvent(ss, ev[0], 0);
  }
  if (!traj_dirs) {
    for (int l = P.nlev - 1; l >= 0; --l) {
      const int h = P.shapes[2 * l], w = P.shapes[2 * l + 1];
      fsb_camera cl = scaled(r.cam0, h, w);
      rc = trajectory_field64_internal(&cl, t_res, prm->epsilon_scale, 1.0, P.traj[l],
                                       P.traj_ok[l], P.traj_scratch, P.traj_bytes, ss);
      if (rc) return rc;
    }
  }
  rc = fov_mask_internal(&r.cam0, P.mask0, P.iters + 0, st);
  if (rc) return rc;
  rc = fov_mask_internal(&r.cam1, P.mask1, P.iters + 1, st);
  if (rc) return rc;
  rc = calibrate64_internal(rig, i1, P.mask1, i1c, P.i1c_ok, P.iters + 2, st);
  if (rc) return rc;
  k64_and_mask<<<(unsigned)((n0 + 255) / 256), 256, 0, st>>>(P.mask0, P.i1c_ok, n0, P.solve_mask);
  // mask and i1c are final here: publish them early (graph capture only)
  cudaMemcpyAsync(mask_out, P.solve_mask, n0, cudaMemcpyDeviceToDevice, st);
  if (g_early_event) cudaEventRecordWithFlags(g_early_event, st, cudaEventRecordExternal);
  P.lvl_i0[0] = const_cast<double*>(i0);
  P.lvl_i1[0] = i1c;
  P.lvl_mask[0] = P.solve_mask;
  for (int l = 1; l < P.nlev; ++l) {
    const int fh = P.shapes[2 * (l - 1)], fw = P.shapes[2 * (l - 1) + 1];
    const int ch = P.shapes[2 * l], cw = P.shapes[2 * l + 1];
    rc = downsample64_internal(P.lvl_i0[l - 1], P.lvl_mask[l - 1], fh, fw, P.lvl_i0[l],
                               P.lvl_mask[l], ch, cw, st);
    if (rc) return rc;
    rc = downsample64_internal(P.lvl_i1[l - 1], P.lvl_mask[l - 1], fh, fw, P.lvl_i1[l],
                               P.lvl_mask[l], ch, cw, st);
    if (rc) return rc;
  }
  // the level views (coarse -> fine index k) and their setup, on the side stream
  std::vector<L64> lv(P.nlev);
  for (int k = 0; k < P.nlev; ++k) {
    const int l = P.nlev - 1 - k;
    const int h = P.shapes[2 * l], w = P.shapes[2 * l + 1];
    L64& L = lv[k];
    memset(&L, 0, sizeof(L));
    L.h = h; L.w = w; L.n = (size_t)h * w;
    L.i0 = P.lvl_i0[l]; L.i1 = P.lvl_i1[l]; L.mask = P.lvl_mask[l];
    L.traj = traj_dirs ? traj_dirs[k] : P.traj[l];
    L.traj_ok = traj_dirs ? traj_okv[k] : P.traj_ok[l];
    const size_t np = L.n;
    L.T = P.cst[l]; L.S = P.cst[l] + 3 * np;
    L.iu = P.cst[l] + 6 * np; L.rho0 = P.cst[l] + 7 * np; L.uo = P.cst[l] + 8 * np;
    L.u = P.setA; L.v = P.setA + np; L.p = P.setA + 3 * np; L.q = P.setA + 5 * np;
    L.ub = P.setA + 9 * np; L.vb = P.setA + 10 * np;
    L.u2 = P.setB; L.v2 = P.setB + np; L.p2 = P.setB + 3 * np; L.q2 = P.setB + 5 * np;
    L.ub2 = P.setB + 9 * np; L.vb2 = P.setB + 10 * np;
    L.full16 = P.f16l[l];
    L.ecode = P.ecl[l]; L.tiles = P.tll[l]; L.tex = P.texl[l];
    L.lvl_partials = P.lvl_partials; L.lvl_partials_cap = P.lvl_partials_n;
    L.i1w = P.i1w; L.i1w_ok = P.i1w_ok;
    L.dirs = P.dirs; L.dir_ok = P.dir_ok; L.partials = P.partials;
  }
  if (side) {
    cudaEventRecord(ev[kMaxLevels + 1], st);  // pyramids done
    cudaStreamWaitEvent(ss, ev[kMaxLevels + 1], 0);
    for (int k = 0; k < P.nlev; ++k) {
      rc = level_prepare64(lv[k], prm, level_cfg64(lv[k]), P.setup_scratch, P.setup_bytes, ss);
      if (rc) return rc;
      cudaEventRecord(ev[1 + k], ss);
    }
  }
  int64_t pd_off = 0, warp_off = 0;
  int cur = 0, prev_h = 0, prev_w = 0;
  const uint8_t* prev_mask = nullptr;
  for (int k = 0; k < P.nlev; ++k) {
    const int l = P.nlev - 1 - k;
    const int h = P.shapes[2 * l], w = P.shapes[2 * l + 1];
    const size_t np = (size_t)h * w;
    const LevelRange nvtx_range("fsb64 level %dx%d", w, h);  // NVTX range per level
    double* u = P.setA;  // plane 0 of the level's state block
    double* wv = P.wv[cur];
    if (k == 0) {
      cudaMemsetAsync(u, 0, np * sizeof(double), st);
      cudaMemsetAsync(wv, 0, 2 * np * sizeof(double), st);
    } else {
      rc = upsample64_internal(P.carry_u, P.wv[cur ^ 1], prev_mask, prev_h, prev_w,
                               P.lvl_mask[l], h, w, u, wv, st);
      if (rc) return rc;
    }
    L64 L = lv[k];
    L.wv = wv;
    if (side) cudaStreamWaitEvent(st, ev[1 + k], 0);  // join: this level's setup done
    rc = solve_level64(L, prm, diag, pd_off, warp_off, P.setup_scratch, P.setup_bytes, st,
                       tm && tm->level == l ? tm : nullptr, side);
    if (rc) return rc;
    pd_off += (int64_t)N * K;
    warp_off += N;
    prev_h = h; prev_w = w; prev_mask = P.lvl_mask[l];
    if (l > 0) cudaMemcpyAsync(P.carry_u, u, np * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (l == 0) {
      cudaMemcpyAsync(u_out, u, n0 * sizeof(double), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(w_out, wv, 2 * n0 * sizeof(double), cudaMemcpyDeviceToDevice, st);
      k64_interleave<<<(unsigned)((n0 + 255) / 256), 256, 0, st>>>(P.setA + n0, n0, v_out);
    }
    cur ^= 1;
  }
  return launch_status();
}

}  // namespace fsb

using namespace fsb;

extern "C" {

size_t fsb_solve_pyramid_f64_workspace_bytes(const fsb_rig* rig, const fsb_params* prm) {
  return solve_pyramid64_bytes(rig, prm);
}

int fsb_solve_pyramid_f64(const fsb_rig* rig, const fsb_params* prm, const double* i0,
                          const double* i1, const double* const* traj_dirs,
                          const uint8_t* const* traj_ok, void* workspace, size_t workspace_bytes,
                          double* u, double* w, double* v, uint8_t* mask, double* i1c,
                          const fsb_diag* diag, void* stream) {
  return solve_pyramid64(rig, prm, i0, i1, traj_dirs, traj_ok, workspace, workspace_bytes, u, w,
                         v, mask, i1c, diag, as_stream(stream));
}

size_t fsb_warp_linearize_f64_scratch_bytes(int32_t h, int32_t w) {
  return (size_t)h * w * sizeof(double4) + 256;
}

int fsb_warp_linearize_f64(int32_t h, int32_t w, const double* i0, const double* i1,
                           const uint8_t* mask, const double* traj, const uint8_t* traj_ok,
                           const double* wv, double* i1w, uint8_t* i1w_ok, double* dirs,
                           uint8_t* dir_ok, double* iu, double* rho0, void* scratch,
                           size_t scratch_bytes, int32_t kind, void* stream) {
  if (h < 1 || w < 1 || !i0 || !i1 || !mask || !traj || !traj_ok || !wv || !i1w || !i1w_ok ||
      !dirs || !dir_ok || !iu || !rho0 || !scratch ||
      scratch_bytes < fsb_warp_linearize_f64_scratch_bytes(h, w) || (kind != 0 && kind != 1))
    return FSB_EINVAL;
  cudaStream_t st = as_stream(stream);
  const size_t n = (size_t)h * w;
  if (kind == 1) {  // NaN-encoded texels (sample64.cu)
    if (reinterpret_cast<uintptr_t>(scratch) & 31) return FSB_EINVAL;
    double4* tex = reinterpret_cast<double4*>(scratch);
    int rc = pack64_internal(i1, mask, traj, traj_ok, h, w, tex, st);
    if (rc) return rc;
    P64 PL;
    PL.h = h; PL.w = w; PL.i0 = i0; PL.mask = mask; PL.tex = tex; PL.wv = wv;
    PL.i1wn = i1w; PL.dirs = dirs; PL.dir_ok = dir_ok; PL.iu = iu; PL.rho0 = rho0;
    rc = sample_nan64_internal(PL, kBX, kBY, st);
    if (rc) return rc;
    rc = linearize_nan64_internal(PL, kBX, kBY, st);
    if (rc) return rc;
    k64_nan_split<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(i1w, i1w_ok, n);
    return launch_status();
  }
  L64 L;  // masked-gather kernels (k64_sample / k64_linearize) with all-16-valid flags
  memset(&L, 0, sizeof(L));
  L.h = h; L.w = w; L.n = n;
  L.i0 = i0; L.i1 = i1; L.mask = mask; L.traj = traj; L.traj_ok = traj_ok;
  L.wv = const_cast<double*>(wv); L.i1w = i1w; L.i1w_ok = i1w_ok; L.dirs = dirs;
  L.dir_ok = dir_ok; L.iu = iu; L.rho0 = rho0;
  L.full16 = reinterpret_cast<uint8_t*>(scratch);
  dim3 blk(kBX, kBY), grd = grid2d(w, h, blk);
  k64_full16<<<grd, blk, 0, st>>>(L);
  k64_sample<<<grd, blk, 0, st>>>(L);
  k64_linearize<<<grd, blk, 0, st>>>(L, false);
  return launch_status();
}

int fsb_phase_timer_create(int32_t level, int32_t max_warps, fsb_phase_timer** out) {
  if (!out || level < 0 || max_warps < 1) return FSB_EINVAL;
  fsb_phase_timer* t = new fsb_phase_timer();
  t->level = level; t->cap = max_warps; t->used = 0; t->pd_launches = 0;
  t->ev = new cudaEvent_t[3 * (size_t)max_warps]();
  for (int k = 0; k < 3 * max_warps; ++k) {
    cudaError_t e = cudaEventCreate(&t->ev[k]);
    if (e != cudaSuccess) {
      for (int j = 0; j < k; ++j) cudaEventDestroy(t->ev[j]);
      delete[] t->ev;
      delete t;
      return (int)e;
    }
  }
  *out = t;
  return FSB_OK;
}

int fsb_phase_timer_read(fsb_phase_timer* t, double* sample_ms, double* pd_ms, int32_t* warps,
                         int32_t* pd_launches_per_warp, int32_t* level_h, int32_t* level_w) {
  if (!t) return FSB_EINVAL;
  double a = 0.0, b = 0.0;
  for (int wi = 0; wi < t->used; ++wi) {
    float x = 0.f, y = 0.f;
    cudaError_t e = cudaEventElapsedTime(&x, t->ev[3 * wi], t->ev[3 * wi + 1]);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&y, t->ev[3 * wi + 1], t->ev[3 * wi + 2]);
    if (e != cudaSuccess) return (int)e;
    a += x; b += y;
  }
  if (sample_ms) *sample_ms = a;
  if (pd_ms) *pd_ms = b;
  if (warps) *warps = t->used;
  if (pd_launches_per_warp) *pd_launches_per_warp = t->pd_launches;
  if (level_h) *level_h = t->level_h;
  if (level_w) *level_w = t->level_w;
  return FSB_OK;
}

int fsb_phase_timer_destroy(fsb_phase_timer* t) {
  if (!t) return FSB_OK;
  for (int k = 0; k < 3 * t->cap; ++k) cudaEventDestroy(t->ev[k]);
  delete[] t->ev;
  delete t;
  return FSB_OK;
}

int fsb_solve_pyramid_f64_timed(const fsb_rig* rig, const fsb_params* prm, const double* i0,
                                const double* i1, void* workspace, size_t workspace_bytes,
                                double* u, double* w, double* v, uint8_t* mask, double* i1c,
                                fsb_phase_timer* timer, void* stream) {
  if (!timer) return FSB_EINVAL;
  timer->used = 0;
  return solve_pyramid64(rig, prm, i0, i1, nullptr, nullptr, workspace, workspace_bytes, u, w,
                         v, mask, i1c, nullptr, as_stream(stream), timer);
}

}  // extern "C"
