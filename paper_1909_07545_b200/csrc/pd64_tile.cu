// Temporally blocked float64 primal-dual tiles, issue-lean (the float64 path's
// hot kernel).
//
// Same cycle as k64_block (pd64_block.cu) and the reference's
// primal_dual_iterate (solver.py:279-303: dual ascent with forward
// differences + unit-ball projection, backward divergence, data-term
// shrinkage, over-relaxation) on a 32-wide tile with an R-pixel halo, `iters`
// <= R cycles per launch, state in registers. What changes is how little the
// SM issues per pixel-cycle:
//   * x-neighbours come from warp shuffles (a tile row is a warp), so only the
//     y-neighbours go through shared memory: 3 doubles published per thread
//     row for the dual (u_bar, v_bar of its first pixel row) and 3 for the
//     primal (the y-fluxes of its last pixel row), 2 barriers per cycle;
//   * PY pixels per thread stacked vertically: the y-neighbours inside a
//     thread stay in registers (PY = 2 halves the shared traffic and gives two
//     independent dependency chains per thread);
//   * the nine per-pixel constants stay in shared memory (registers hold the
//     12 state doubles per pixel);
//   * edge indicators and the skip of masked pixels are predicates decided
//     once per launch; tiles whose interior holds no solve-mask pixel return
//     right after the mask test (their state is exactly zero, see
//     pd64_block.cu);
//   * compiled with FMA contraction (this translation unit is not -fmad=false):
//     the float64 arithmetic keeps ~53-bit rounding, far below the parity gate
//     (tests/test_gpu_c3_parity.py holds it against the reference at C3).
//
// Reference: solver.py:279-303, 347-360 (warp-start resets and clip/accumulate
// epilogue, fused as in k64_block), rasters.py:144-182.

#include "pd64_block.cuh"
#include "pd_math.cuh"

#include <stddef.h>
#include <stdlib.h>
#include <string.h>

namespace fsb {

namespace {

constexpr int kW = 32;   // tile width = warp width

template <int kTR, int PY>
struct SmemT {
  static constexpr int TH = kTR * PY;
  double ub[kTR][kW], vb0[kTR][kW], vb1[kTR][kW];  // first pixel row of each thread row
  double fy[3][kTR][kW];                            // y-fluxes of the last pixel row
  double c[9][TH][kW];                              // a b c sp tu tv g rho0 u_omega
};

int sm_count() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  }
  return v;
}

FSB_INLINE double shfl_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
FSB_INLINE double shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

// One tile (bx, by) of the level: load, `iters` cycles, epilogue, stores.
template <int R, int PY, int kTR, bool DIAG>
FSB_INLINE void tile_work(const B64& A, SmemT<kTR, PY>& S, int bx, int by, int tile_id) {
  constexpr int TH = kTR * PY;
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const size_t n = A.n;
  const int W = A.w, H = A.h;
  const int gx = bx * OW - R + lane;
  const int gy0 = by * OH - R + ty * PY;

  double u[PY], ub[PY], v0[PY], v1[PY], vb0[PY], vb1[PY], p0[PY], p1[PY];
  double q0[PY], q1[PY], q2[PY], q3[PY];
  bool m[PY], ex[PY], ey[PY], inner[PY];
  uint32_t idx[PY];
  const double alpha1 = A.alpha1;
  if (A.ecode) {
    // Speculative loads: the work list guarantees mask pixels in the interior,
    // and masked pixels hold exactly zero state (and I_u = 0), so every
    // in-image pixel loads unconditionally — one memory round trip, no
    // dependency on the mask.
#pragma unroll
    // 32-bit pixel offsets from kernel-uniform plane pointers: one address
    // instruction per plane. Out-of-image threads read pixel 0 (finite values)
    // and get edge code 0, so nothing they compute reaches an in-image pixel.
    const double* __restrict__ sv1 = A.sv + n;
    const double* __restrict__ sp1 = A.sp + n;
    const double* __restrict__ sq1 = A.sq + n;
    const double* __restrict__ sq2 = A.sq + 2 * n;
    const double* __restrict__ sq3 = A.sq + 3 * n;
    const double* __restrict__ t1 = A.T + n;
    const double* __restrict__ t2 = A.T + 2 * n;
    const double* __restrict__ s1 = A.S + n;
    const double* __restrict__ s2 = A.S + 2 * n;
    const double* __restrict__ svb1 = A.svb + n;
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int gy = gy0 + j;
      const bool in = (unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H;
      const uint32_t i = in ? (uint32_t)gy * (uint32_t)W + (uint32_t)gx : 0u;
      FSB_CHECK(i < n);
      idx[j] = i;
      const int ry = ty * PY + j;
      inner[j] = lane >= R && lane < kW - R && ry >= R && ry < TH - R && in;
      const uint32_t code = in ? A.ecode[i] : 0u;
      u[j] = A.su[i];
      v0[j] = A.sv[i]; v1[j] = sv1[i];
      p0[j] = A.sp[i]; p1[j] = sp1[i];
      q0[j] = A.sq[i]; q1[j] = sq1[i]; q2[j] = sq2[i]; q3[j] = sq3[i];
      double cc[9];
      cc[0] = A.T[i]; cc[1] = t1[i]; cc[2] = t2[i];
      cc[3] = A.S[i] * alpha1; cc[4] = s1[i]; cc[5] = s2[i];
      cc[6] = A.iu[i]; cc[7] = A.rho0[i];
      if (A.first) {
        ub[j] = u[j]; vb0[j] = v0[j]; vb1[j] = v1[j]; cc[8] = u[j];
      } else {
        ub[j] = A.sub[i]; vb0[j] = A.svb[i]; vb1[j] = svb1[i]; cc[8] = A.uo[i];
      }
      m[j] = code & 1u;
      ex[j] = code & 2u;
      ey[j] = code & 4u;
#pragma unroll
      for (int k = 0; k < 9; ++k) S.c[k][ry][lane] = cc[k];
    }
  } else {
    bool any = false;
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int gy = gy0 + j;
      const bool in = (unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H;
      const size_t i = in ? (size_t)gy * W + gx : 0;
      idx[j] = (uint32_t)i;
      m[j] = in && A.mask[i];
      ex[j] = m[j] && gx + 1 < W && A.mask[i + 1];
      ey[j] = m[j] && gy + 1 < H && A.mask[i + W];
      const int ry = ty * PY + j;
      inner[j] = lane >= R && lane < kW - R && ry >= R && ry < TH - R && in;
      any = any || (inner[j] && m[j]);
    }
    // no solve-mask pixel in the interior: nothing to update or store
    if (!__syncthreads_or(any)) {
      if (A.fin && DIAG && (A.diag_du || A.diag_du64) && lane == 0 && ty == 0) A.partials[tile_id] = 0.0;
      return;
    }
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      double cc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      u[j] = ub[j] = v0[j] = v1[j] = vb0[j] = vb1[j] = p0[j] = p1[j] = 0.0;
      q0[j] = q1[j] = q2[j] = q3[j] = 0.0;
      if (m[j]) {
        const size_t i = idx[j];
        u[j] = A.su[i];
        v0[j] = A.sv[i]; v1[j] = A.sv[n + i];
        p0[j] = A.sp[i]; p1[j] = A.sp[n + i];
        q0[j] = A.sq[i]; q1[j] = A.sq[n + i]; q2[j] = A.sq[2 * n + i]; q3[j] = A.sq[3 * n + i];
        cc[0] = A.T[i]; cc[1] = A.T[n + i]; cc[2] = A.T[2 * n + i];
        cc[3] = A.S[i] * alpha1; cc[4] = A.S[n + i]; cc[5] = A.S[2 * n + i];
        cc[6] = A.iu[i]; cc[7] = A.rho0[i];
        if (A.first) {  // warp-start reset (solver.py:344-346): u0 = u, u_bar = u, v_bar = v
          ub[j] = u[j]; vb0[j] = v0[j]; vb1[j] = v1[j]; cc[8] = u[j];
        } else {
          ub[j] = A.sub[i]; vb0[j] = A.svb[i]; vb1[j] = A.svb[n + i]; cc[8] = A.uo[i];
        }
      }
      const int ry = ty * PY + j;
#pragma unroll
      for (int k = 0; k < 9; ++k) S.c[k][ry][lane] = cc[k];
    }
  }
  const double sq = A.sigma_q * A.alpha0, heps = A.heps;
  const double lam = A.lam, alpha0 = A.alpha0, theta = A.theta;
  const int tyd = ty + 1 < kTR ? ty + 1 : ty;
  for (int it = 0; it < A.iters; ++it) {
    S.ub[ty][lane] = ub[0];
    S.vb0[ty][lane] = vb0[0];
    S.vb1[ty][lane] = vb1[0];
    __syncthreads();
    double fx0[PY], fx1[PY], fx2[PY], fy0[PY], fy1[PY], fy2[PY];
    double pmax = 0.0, qmax = 0.0;
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int ry = ty * PY + j;
      const double a = S.c[0][ry][lane], b = S.c[1][ry][lane], c = S.c[2][ry][lane];
      const double sp = S.c[3][ry][lane];
      // forward differences (rasters.py:144-155), zero where the edge leaves the mask
      const double ubx = shfl_dn(ub[j]), vbx0 = shfl_dn(vb0[j]), vbx1 = shfl_dn(vb1[j]);
      double uby, vby0, vby1;
      if (j + 1 < PY) {
        uby = ub[j + 1]; vby0 = vb0[j + 1]; vby1 = vb1[j + 1];
      } else {
        uby = S.ub[tyd][lane]; vby0 = S.vb0[tyd][lane]; vby1 = S.vb1[tyd][lane];
      }
      const double gxx = ex[j] ? ubx - ub[j] : 0.0, gyy = ey[j] ? uby - ub[j] : 0.0;
      const double g00 = ex[j] ? vbx0 - vb0[j] : 0.0, g01 = ey[j] ? vby0 - vb0[j] : 0.0;
      const double g10 = ex[j] ? vbx1 - vb1[j] : 0.0, g11 = ey[j] ? vby1 - vb1[j] : 0.0;
      dual_update_exact<double>(a, b, c, sp, sq, gxx, gyy, g00, g01, g10, g11, vb0[j], vb1[j],
                                p0[j], p1[j], q0[j], q1[j], q2[j], q3[j], heps);
      fx0[j] = ex[j] ? a * p0[j] + b * p1[j] : 0.0;
      fy0[j] = ey[j] ? b * p0[j] + c * p1[j] : 0.0;
      fx1[j] = ex[j] ? q0[j] : 0.0;
      fy1[j] = ey[j] ? q1[j] : 0.0;
      fx2[j] = ex[j] ? q2[j] : 0.0;
      fy2[j] = ey[j] ? q3[j] : 0.0;
      if (DIAG && inner[j]) {
        pmax = fmax(pmax, sqrt(p0[j] * p0[j] + p1[j] * p1[j]));
        qmax = fmax(qmax, sqrt(((q0[j] * q0[j] + q1[j] * q1[j]) + q2[j] * q2[j]) + q3[j] * q3[j]));
      }
    }
    S.fy[0][ty][lane] = fy0[PY - 1];
    S.fy[1][ty][lane] = fy1[PY - 1];
    S.fy[2][ty][lane] = fy2[PY - 1];
    if (DIAG) {
      pmax = warp_max(pmax);
      qmax = warp_max(qmax);
      if (lane == 0 && A.diag_p) {
        atomic_max_nonneg(A.diag_p + it, (float)pmax);
        atomic_max_nonneg(A.diag_q + it, (float)qmax);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int ry = ty * PY + j;
      // backward divergence (rasters.py:158-172); the column left of / row above
      // the tile feed only halo pixels
      const double lx0 = shfl_up(fx0[j]), lx1 = shfl_up(fx1[j]), lx2 = shfl_up(fx2[j]);
      double uy0, uy1, uy2;
      if (j > 0) {
        uy0 = fy0[j - 1]; uy1 = fy1[j - 1]; uy2 = fy2[j - 1];
      } else if (ty > 0) {
        uy0 = S.fy[0][ty - 1][lane]; uy1 = S.fy[1][ty - 1][lane]; uy2 = S.fy[2][ty - 1][lane];
      } else {
        uy0 = uy1 = uy2 = 0.0;
      }
      const double dvv = ((fx0[j] - lx0) + fy0[j]) - uy0;
      const double d0 = ((fx1[j] - lx1) + fy1[j]) - uy1;
      const double d1 = ((fx2[j] - lx2) + fy2[j]) - uy2;
      const double tu = S.c[4][ry][lane], tv = S.c[5][ry][lane], g = S.c[6][ry][lane];
      const double rh = S.c[7][ry][lane], uo = S.c[8][ry][lane];
      primal_update_exact<double>(dvv, d0, d1, tu, tv, g, rh, uo, p0[j], p1[j], lam, alpha0,
                                  alpha1, theta, u[j], v0[j], v1[j], ub[j], vb0[j], vb1[j]);
    }
  }
  double adu = 0.0, amax = 0.0;
#pragma unroll
  for (int j = 0; j < PY; ++j) {
    const int ry = ty * PY + j;
    const uint32_t i = idx[j];
    const bool st = inner[j] && m[j];
    const double uo = S.c[8][ry][lane];
    if (A.fin && st) {  // clip / accumulate (solver.py:356-360) on the interior
      const double du = fmin(fmax(u[j] - uo, -A.du_max), A.du_max);
      u[j] = uo + du;
      amax = fmax(amax, fabs(du));
      const double2 dd = reinterpret_cast<const double2*>(A.dirs)[i];
      double2 wv = reinterpret_cast<double2*>(A.wv)[i];
      wv.x = wv.x + du * dd.x;
      wv.y = wv.y + du * dd.y;
      reinterpret_cast<double2*>(A.wv)[i] = wv;
      adu += fabs(du);
    }
    if (!st) continue;
    if (A.first) A.uo[i] = uo;
    A.du[i] = u[j];
    A.dv[i] = v0[j]; (A.dv + n)[i] = v1[j];
    A.dp[i] = p0[j]; (A.dp + n)[i] = p1[j];
    A.dq[i] = q0[j]; (A.dq + n)[i] = q1[j]; (A.dq + 2 * n)[i] = q2[j];
    (A.dq + 3 * n)[i] = q3[j];
    if (!A.fin) {  // u_bar / v_bar are reset at the next warp's start: dead after its last cycle
      A.dub[i] = ub[j];
      A.dvb[i] = vb0[j]; (A.dvb + n)[i] = vb1[j];
    }
  }
  if (DIAG && A.fin && (A.diag_du || A.diag_du64)) {
    __shared__ double s_sum[kTR], s_max[kTR];
    const double mx = warp_max(amax), sm = warp_sum(adu);
    if (lane == 0) { s_sum[ty] = sm; s_max[ty] = mx; }
    __syncthreads();
    if (lane == 0 && ty == 0) {
      double t = 0.0, mm = 0.0;
      for (int k = 0; k < kTR; ++k) { t += s_sum[k]; mm = fmax(mm, s_max[k]); }
      A.partials[tile_id] = t;
      if (A.diag_du64) atomic_max_nonneg(A.diag_du64, mm);
        else atomic_max_nonneg(A.diag_du, (float)mm);
    }
  }
}

template <int R, int PY, int kTR, bool DIAG>
__global__ void __launch_bounds__(kW * kTR, kTR * PY <= 16 ? 2 : 1) k64_tile(const B64 A) {
  constexpr int TH = kTR * PY;
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  extern __shared__ double s_raw[];
  SmemT<kTR, PY>& S = *reinterpret_cast<SmemT<kTR, PY>*>(s_raw);
  poison_dynamic_smem(s_raw);  // checked build only
  const int ntx = (A.w + OW - 1) / OW;
  if (!A.tiles) {  // 2-D grid over every tile
    tile_work<R, PY, kTR, DIAG>(A, S, blockIdx.x, blockIdx.y, blockIdx.y * ntx + blockIdx.x);
    return;
  }
  // 1-D grid over the level's work list. With A.persist the grid is 2 CTAs per
  // SM striding over the list, and the second half of the CTAs starts
  // A.persist ns late, so an SM's two CTAs keep opposite phases (one loading
  // while the other cycles) instead of loading in step.
  const int cnt = A.tiles[0];
  const int stride = A.persist ? (int)gridDim.x : cnt;
  if (A.persist && blockIdx.x >= gridDim.x / 2) __nanosleep((unsigned)A.persist);
  for (int k = blockIdx.x; k < cnt; k += stride) {
    const int t = A.tiles[1 + k];
    tile_work<R, PY, kTR, DIAG>(A, S, t % ntx, t / ntx, t);
    if (A.persist) __syncthreads();  // shared tile buffers are reused by the next tile
  }
}

template <int R, int PY, int kTR, bool DIAG>
int launch_tile(const B64& A0, cudaStream_t st) {
  constexpr int TH = kTR * PY;
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  B64 A = A0;
  if (kTR * PY > 16) A.persist = 0;  // the staggered schedule needs 2 CTAs per SM
  const int ntx = (A.w + OW - 1) / OW, nty = (A.h + OH - 1) / OH;
  // with a work list: a 1-D grid of every tile (CTAs past the list's count exit),
  // or 2 persistent CTAs per SM
  const dim3 blk(kW, kTR),
      grd = A.tiles ? dim3(A.persist ? 2 * sm_count() : ntx * nty) : dim3(ntx, nty);
  const size_t dyn = sizeof(SmemT<kTR, PY>);
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k64_tile<R, PY, kTR, DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dyn);
  });
  k64_tile<R, PY, kTR, DIAG><<<grd, blk, dyn, st>>>(A);
  return launch_status();
}

int tile_py() {
  static const int v = [] {
    const char* e = getenv("FSB_PD64_PY");
    return e && e[0] == '2' ? 2 : 1;
  }();
  return v;
}

// thread rows per CTA: 16 for one pixel per thread; FSB_PD64_PY=2 stacks two
// pixels per thread on 8 thread rows (same 32 x 16 tile, 2 CTAs / SM) or, with
// FSB_PD64_PY=2t, on 16 thread rows (32 x 32 tile, 1 CTA / SM)
// Thread rows per CTA (one pixel per thread): 16 (2 CTAs / SM; the large,
// DRAM-streaming levels, with the staggered persistent schedule) or 32 (1 CTA
// / SM, 32 x 32 tiles). 32 rows pay off on levels of 128^2 < n <= 256^2: their
// 32 x 32 tiles fit one wave at R = 5, so a warp takes 2 PD launches instead of
// 4 (C3 256^2: 2.39 -> 2.13 ms); elsewhere 16 rows measured better.
// FSB_PD64_ROWS_L="w:rows,..." overrides per level width; FSB_PD64_PY=2 stacks
// two pixels per thread on 8 rows.
int tile_rows(int w, int h) {
  static const int py2 = [] {
    const char* e = getenv("FSB_PD64_PY");
    return e && e[0] == '2' ? (e[1] == 't' ? 16 : 8) : 0;
  }();
  if (py2) return py2;
  const char* e = getenv("FSB_PD64_ROWS_L");
  for (const char* c = e; c && *c;) {
    const int lw = atoi(c);
    const char* colon = strchr(c, ':');
    if (!colon) break;
    const int r = atoi(colon + 1);
    if (lw == w && (r == 16 || r == 32)) return r;
    c = strchr(colon, ',');
    if (c) ++c;
  }
  const size_t n = (size_t)w * h;
  return n > 128 * 128 && n <= 256 * 256 ? 32 : 16;
}

template <int R>
int launch_r(const B64& A, cudaStream_t st) {
  const bool diag = A.diag_p || A.diag_du || A.diag_du64;
  const int rows = tile_rows(A.w, A.h);
  if (tile_py() == 2 && rows == 8)
    return diag ? launch_tile<R, 2, 8, true>(A, st) : launch_tile<R, 2, 8, false>(A, st);
  if (tile_py() == 2)
    return diag ? launch_tile<R, 2, 16, true>(A, st) : launch_tile<R, 2, 16, false>(A, st);
  if (rows == 32)
    return diag ? launch_tile<R, 1, 32, true>(A, st) : launch_tile<R, 1, 32, false>(A, st);
  return diag ? launch_tile<R, 1, 16, true>(A, st) : launch_tile<R, 1, 16, false>(A, st);
}

// Edge code per pixel of a level: bit0 mask, bit1 x-edge in the mask
// (m(x) & m(x+1)), bit2 y-edge (m(y) & m(y+1)) — rasters.py:175-182.
__global__ void k64_edge_codes(const uint8_t* __restrict__ m, int w, int h,
                               uint32_t* __restrict__ code, double* __restrict__ codef) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w) return;
  const size_t i = (size_t)y * w + x;
  const bool mm = m[i];
  const bool ex = mm && x + 1 < w && m[i + 1];
  const bool ey = mm && y + 1 < h && m[i + w];
  const uint32_t c = (mm ? 1u : 0u) | (ex ? 2u : 0u) | (ey ? 4u : 0u);
  code[i] = c;
  if (codef) codef[i] = (double)c;
}

}  // namespace

int pd64_edge_codes(const uint8_t* mask, int w, int h, uint32_t* code, double* codef,
                    cudaStream_t st) {
  k64_edge_codes<<<dim3((w + 127) / 128, h), 128, 0, st>>>(mask, w, h, code, codef);
  return launch_status();
}

size_t pd64_tile_count(int w, int h, int halo) {
  const int TH = tile_rows(w, h) * tile_py();
  const int OW = kW - 2 * halo, OH = TH - 2 * halo;
  return (size_t)((w + OW - 1) / OW) * ((h + OH - 1) / OH);
}

int tile_list_internal(const uint8_t* mask, int w, int h, int TW, int TH, int* tiles,
                       cudaStream_t st);

int pd64_tile_tile_list(const uint8_t* mask, int w, int h, int halo, int* tiles,
                        cudaStream_t st) {
  return tile_list_internal(mask, w, h, kW - 2 * halo, tile_rows(w, h) * tile_py() - 2 * halo, tiles,
                            st);
}

int pd64_tile_launch_unchecked(const B64& A, int halo, cudaStream_t st) {
  switch (halo) {
    case 2: return launch_r<2>(A, st);
    case 3: return launch_r<3>(A, st);
    default: return FSB_EINVAL;
  }
}

int pd64_tile_launch(const B64& A, int halo, cudaStream_t st) {
  if (A.iters < 1 || A.iters > halo) return FSB_EINVAL;
  switch (halo) {
    case 1: return launch_r<1>(A, st);
    case 2: return launch_r<2>(A, st);
    case 3: return launch_r<3>(A, st);
    case 5: return launch_r<5>(A, st);
    default: return FSB_EINVAL;
  }
}

}  // namespace fsb
