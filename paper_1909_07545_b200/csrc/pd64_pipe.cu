// Persistent, software-pipelined float64 primal-dual tiles (the float64 path's
// hot kernel on the large pyramid levels).
//
// The cycle is the reference's primal_dual_iterate (solver.py:279-303) as in
// k64_block / k64_tile, with the warp-start reset (solver.py:344-346) and the
// clip / accumulate epilogue (solver.py:356-360) fused into the first / last
// launch of a warp. The difference is the memory pipeline:
//   * one CTA per SM walks a per-level work list of the tiles whose interior
//     holds solve-mask pixels (masked pixels keep exactly zero state, see
//     pd64_block.cu), tile k, k + gridDim.x, ...;
//   * the 21 float64 planes of a tile (12 state, 9 constants) and a 32-bit
//     edge code per pixel land in a shared-memory staging tile through
//     cp.async (8-byte copies, zero-filled outside the image); as soon as the
//     threads have moved tile k into registers the copies of tile
//     k + gridDim.x are issued, so the loads of the next tile run under the
//     primal-dual cycles of this one instead of stalling them;
//   * every pixel's state AND constants live in registers during the cycles
//     (one pixel per thread, a tile row per warp): x-neighbours by warp
//     shuffles, y-neighbours through a small exchange buffer (u_bar / v_bar
//     for the dual, the y-fluxes for the primal), two barriers per cycle;
//   * the edge indicators of the masked gradient / divergence (rasters.py:
//     144-182) come precomputed per level (k64_edge_codes), so the kernel
//     never reads a neighbour's mask;
//   * FMA contraction on (this unit is not -fmad=false), IEEE division and
//     square root where the reference divides.
//
// Reference: solver.py:279-303, 344-360, rasters.py:144-182.

#include "pd64_block.cuh"
#include "pd_math.cuh"

#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

namespace fsb {

int tile_list_internal(const uint8_t* mask, int w, int h, int TW, int TH, int* tiles,
                       cudaStream_t st);

namespace {

constexpr int kW = 32;
constexpr int kPlanes = 21;  // staging planes (state 12, constants 9)
// staging plane order
enum { PU, PUB, PV0, PV1, PVB0, PVB1, PP0, PP1, PQ0, PQ1, PQ2, PQ3,
       PA, PB, PC, PSP, PTU, PTV, PIU, PRH, PUO };

template <int TH>
struct PipeSmem {
  double stg[kPlanes][TH][kW];
  uint32_t code[TH][kW];
  double xb[3][TH][kW];  // u_bar, v_bar0, v_bar1 (read by the row above)
  double fy[3][TH][kW];  // y-fluxes (read by the row below)
};

FSB_INLINE uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
FSB_INLINE void cp8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(su32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
FSB_INLINE void cp4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(su32(dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
FSB_INLINE void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FSB_INLINE void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
FSB_INLINE double shfl_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
FSB_INLINE double shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

// Stage tile `tile` (grid ntx wide, OW x OH interiors, R halo) into S.stg / S.code.
template <int R, int TH>
FSB_INLINE void stage(PipeSmem<TH>& S, const B64& A, int tile, int ntx) {
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int gx = (tile % ntx) * OW - R + lane, gy = (tile / ntx) * OH - R + ty;
  const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
  const size_t n = A.n, i = in ? (size_t)gy * A.w + gx : 0;
  cp4(&S.code[ty][lane], A.ecode + i, in);
  cp8(&S.stg[PU][ty][lane], A.su + i, in);
  cp8(&S.stg[PV0][ty][lane], A.sv + i, in);
  cp8(&S.stg[PV1][ty][lane], A.sv + n + i, in);
  if (!A.first) {
    cp8(&S.stg[PUB][ty][lane], A.sub + i, in);
    cp8(&S.stg[PVB0][ty][lane], A.svb + i, in);
    cp8(&S.stg[PVB1][ty][lane], A.svb + n + i, in);
    cp8(&S.stg[PUO][ty][lane], A.uo + i, in);
  }
  cp8(&S.stg[PP0][ty][lane], A.sp + i, in);
  cp8(&S.stg[PP1][ty][lane], A.sp + n + i, in);
#pragma unroll
  for (int k = 0; k < 4; ++k) cp8(&S.stg[PQ0 + k][ty][lane], A.sq + k * n + i, in);
#pragma unroll
  for (int k = 0; k < 3; ++k) cp8(&S.stg[PA + k][ty][lane], A.T + k * n + i, in);
#pragma unroll
  for (int k = 0; k < 3; ++k) cp8(&S.stg[PSP + k][ty][lane], A.S + k * n + i, in);
  cp8(&S.stg[PIU][ty][lane], A.iu + i, in);
  cp8(&S.stg[PRH][ty][lane], A.rho0 + i, in);
  cp_commit();
}

template <int R, int TH, bool DIAG>
__global__ void __launch_bounds__(kW * TH, 1) k64_pipe(const B64 A) {
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  extern __shared__ double s_raw[];
  PipeSmem<TH>& S = *reinterpret_cast<PipeSmem<TH>*>(s_raw);
  const int lane = threadIdx.x, ty = threadIdx.y;
  const size_t n = A.n;
  const int ntx = (A.w + OW - 1) / OW;
  const int cnt = A.tiles ? A.tiles[0] : ntx * ((A.h + OH - 1) / OH);
  const double sq = A.sigma_q * A.alpha0, heps = A.heps, alpha1 = A.alpha1;
  const double lam = A.lam, alpha0 = A.alpha0, theta = A.theta;
  const bool inner_xy = lane >= R && lane < kW - R && ty >= R && ty < TH - R;
  const int tyd = ty + 1 < TH ? ty + 1 : ty;
  double fin_sum = 0.0;
  double fin_max = 0.0;

  int k = blockIdx.x;
  if (k < cnt) stage<R, TH>(S, A, A.tiles ? A.tiles[1 + k] : k, ntx);
  for (; k < cnt; k += gridDim.x) {
    const int tile = A.tiles ? A.tiles[1 + k] : k;
    const int gx = (tile % ntx) * OW - R + lane, gy = (tile / ntx) * OH - R + ty;
    const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
    const size_t i = in ? (size_t)gy * A.w + gx : 0;
    cp_wait_all();
    __syncthreads();
    const uint32_t code = S.code[ty][lane];
    const bool m = code & 1u, ex = code & 2u, ey = code & 4u;
    double u = S.stg[PU][ty][lane], v0 = S.stg[PV0][ty][lane], v1 = S.stg[PV1][ty][lane];
    double ub, vb0, vb1, uo;
    if (A.first) {  // warp-start reset (solver.py:344-346)
      ub = u; vb0 = v0; vb1 = v1; uo = u;
    } else {
      ub = S.stg[PUB][ty][lane]; vb0 = S.stg[PVB0][ty][lane]; vb1 = S.stg[PVB1][ty][lane];
      uo = S.stg[PUO][ty][lane];
    }
    double p0 = S.stg[PP0][ty][lane], p1 = S.stg[PP1][ty][lane];
    double q0 = S.stg[PQ0][ty][lane], q1 = S.stg[PQ1][ty][lane];
    double q2 = S.stg[PQ2][ty][lane], q3 = S.stg[PQ3][ty][lane];
    const double a = S.stg[PA][ty][lane], b = S.stg[PB][ty][lane], c = S.stg[PC][ty][lane];
    const double sp = S.stg[PSP][ty][lane] * alpha1;
    const double tu = S.stg[PTU][ty][lane], tv = S.stg[PTV][ty][lane];
    const double g = S.stg[PIU][ty][lane], rh = S.stg[PRH][ty][lane];
    __syncthreads();  // staging consumed: the next tile's copies run under the cycles
    if (k + (int)gridDim.x < cnt)
      stage<R, TH>(S, A, A.tiles ? A.tiles[1 + k + gridDim.x] : k + gridDim.x, ntx);

    for (int it = 0; it < A.iters; ++it) {
      S.xb[0][ty][lane] = ub;
      S.xb[1][ty][lane] = vb0;
      S.xb[2][ty][lane] = vb1;
      __syncthreads();
      const double ubx = shfl_dn(ub), vbx0 = shfl_dn(vb0), vbx1 = shfl_dn(vb1);
      const double uby = S.xb[0][tyd][lane], vby0 = S.xb[1][tyd][lane];
      const double vby1 = S.xb[2][tyd][lane];
      const double gxx = ex ? ubx - ub : 0.0, gyy = ey ? uby - ub : 0.0;
      const double g00 = ex ? vbx0 - vb0 : 0.0, g01 = ey ? vby0 - vb0 : 0.0;
      const double g10 = ex ? vbx1 - vb1 : 0.0, g11 = ey ? vby1 - vb1 : 0.0;
      dual_update_exact<double>(a, b, c, sp, sq, gxx, gyy, g00, g01, g10, g11, vb0, vb1, p0, p1,
                                q0, q1, q2, q3, heps);
      const double fx0 = ex ? a * p0 + b * p1 : 0.0, fy0 = ey ? b * p0 + c * p1 : 0.0;
      const double fx1 = ex ? q0 : 0.0, fy1 = ey ? q1 : 0.0;
      const double fx2 = ex ? q2 : 0.0, fy2 = ey ? q3 : 0.0;
      S.fy[0][ty][lane] = fy0;
      S.fy[1][ty][lane] = fy1;
      S.fy[2][ty][lane] = fy2;
      if (DIAG) {
        double pn = 0.0, qn = 0.0;
        if (inner_xy && in) {
          pn = sqrt(p0 * p0 + p1 * p1);
          qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
        }
        pn = warp_max(pn);
        qn = warp_max(qn);
        if (lane == 0 && A.diag_p) {
          atomic_max_nonneg(A.diag_p + it, (float)pn);
          atomic_max_nonneg(A.diag_q + it, (float)qn);
        }
      }
      __syncthreads();
      const double lx0 = shfl_up(fx0), lx1 = shfl_up(fx1), lx2 = shfl_up(fx2);
      double uy0 = 0.0, uy1 = 0.0, uy2 = 0.0;
      if (ty > 0) { uy0 = S.fy[0][ty - 1][lane]; uy1 = S.fy[1][ty - 1][lane]; uy2 = S.fy[2][ty - 1][lane]; }
      const double dvv = ((fx0 - lx0) + fy0) - uy0;
      const double d0 = ((fx1 - lx1) + fy1) - uy1;
      const double d1 = ((fx2 - lx2) + fy2) - uy2;
      primal_update_exact<double>(dvv, d0, d1, tu, tv, g, rh, uo, p0, p1, lam, alpha0, alpha1,
                                  theta, u, v0, v1, ub, vb0, vb1);
    }
    const bool st = inner_xy && in && m;
    if (A.fin && st) {  // clip / accumulate (solver.py:356-360)
      const double du = fmin(fmax(u - uo, -A.du_max), A.du_max);
      u = uo + du;
      const double2 dd = reinterpret_cast<const double2*>(A.dirs)[i];
      double2 wv = reinterpret_cast<double2*>(A.wv)[i];
      wv.x = wv.x + du * dd.x;
      wv.y = wv.y + du * dd.y;
      reinterpret_cast<double2*>(A.wv)[i] = wv;
      if (DIAG) {
        fin_sum += fabs(du);
        fin_max = fmax(fin_max, fabs(du));
      }
    }
    if (st) {
      if (A.first) A.uo[i] = uo;
      A.du[i] = u;
      A.dv[i] = v0; A.dv[n + i] = v1;
      A.dp[i] = p0; A.dp[n + i] = p1;
      A.dq[i] = q0; A.dq[n + i] = q1; A.dq[2 * n + i] = q2; A.dq[3 * n + i] = q3;
      if (!A.fin) {  // u_bar / v_bar are reset at the next warp's start
        A.dub[i] = ub;
        A.dvb[i] = vb0; A.dvb[n + i] = vb1;
      }
    }
    if (DIAG && A.fin && (A.diag_du || A.diag_du64)) {  // per-tile sum of |du| (fixed order), global max
      __shared__ double s_sum[TH];
      __shared__ double s_max[TH];
      const double sm = warp_sum(fin_sum);
      const double mx = warp_max(fin_max);
      if (lane == 0) { s_sum[ty] = sm; s_max[ty] = mx; }
      __syncthreads();
      if (lane == 0 && ty == 0) {
        double t = 0.0, mm = 0.0;
        for (int r = 0; r < TH; ++r) { t += s_sum[r]; mm = fmax(mm, s_max[r]); }
        A.partials[tile] = t;
        if (A.diag_du64) atomic_max_nonneg(A.diag_du64, mm);
        else atomic_max_nonneg(A.diag_du, (float)mm);
      }
      fin_sum = 0.0;
      fin_max = 0.0;
    }
  }
  cp_wait_all();
}

// ---- two CTAs per SM: constants in shared memory, state pipelined -----------
// The variant for 2 CTAs per SM (64 registers, 110 KB of shared memory each):
// the 12 state planes of tile k + gridDim.x are copied while tile k cycles (its
// state lives in registers); the 9 constant planes stay in shared memory for the
// cycles and the next tile's constants are copied in after the last cycle, under
// the epilogue stores. Two CTAs per SM desynchronise the barriers.
template <int TH>
struct PipeSmemCS {
  double stg[12][TH][kW];  // state staging (next tile)
  double cst[9][TH][kW];   // constants of the current tile
  uint32_t code[TH][kW];
  double xb[3][TH][kW];
  double fy[3][TH][kW];
};

template <int R, int TH>
FSB_INLINE void stage_state(PipeSmemCS<TH>& S, const B64& A, int tile, int ntx) {
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int gx = (tile % ntx) * OW - R + lane, gy = (tile / ntx) * OH - R + ty;
  const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
  const size_t n = A.n, i = in ? (size_t)gy * A.w + gx : 0;
  cp4(&S.code[ty][lane], A.ecode + i, in);
  cp8(&S.stg[PU][ty][lane], A.su + i, in);
  cp8(&S.stg[PV0][ty][lane], A.sv + i, in);
  cp8(&S.stg[PV1][ty][lane], A.sv + n + i, in);
  if (!A.first) {
    cp8(&S.stg[PUB][ty][lane], A.sub + i, in);
    cp8(&S.stg[PVB0][ty][lane], A.svb + i, in);
    cp8(&S.stg[PVB1][ty][lane], A.svb + n + i, in);
  }
  cp8(&S.stg[PP0][ty][lane], A.sp + i, in);
  cp8(&S.stg[PP1][ty][lane], A.sp + n + i, in);
#pragma unroll
  for (int k = 0; k < 4; ++k) cp8(&S.stg[PQ0 + k][ty][lane], A.sq + k * n + i, in);
  cp_commit();
}

template <int R, int TH>
FSB_INLINE void stage_const(PipeSmemCS<TH>& S, const B64& A, int tile, int ntx) {
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int gx = (tile % ntx) * OW - R + lane, gy = (tile / ntx) * OH - R + ty;
  const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
  const size_t n = A.n, i = in ? (size_t)gy * A.w + gx : 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) cp8(&S.cst[k][ty][lane], A.T + k * n + i, in);
#pragma unroll
  for (int k = 0; k < 3; ++k) cp8(&S.cst[3 + k][ty][lane], A.S + k * n + i, in);
  cp8(&S.cst[6][ty][lane], A.iu + i, in);
  cp8(&S.cst[7][ty][lane], A.rho0 + i, in);
  // u_omega: the warp's first launch takes it from u (solver.py:344-346)
  cp8(&S.cst[8][ty][lane], (A.first ? A.su : A.uo) + i, in);
  cp_commit();
}

template <int R, int TH, bool DIAG>
__global__ void __launch_bounds__(kW * TH, 2) k64_pipe_cs(const B64 A) {
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  extern __shared__ double s_raw[];
  PipeSmemCS<TH>& S = *reinterpret_cast<PipeSmemCS<TH>*>(s_raw);
  const int lane = threadIdx.x, ty = threadIdx.y;
  const size_t n = A.n;
  const int ntx = (A.w + OW - 1) / OW;
  const int cnt = A.tiles ? A.tiles[0] : ntx * ((A.h + OH - 1) / OH);
  const double sq = A.sigma_q * A.alpha0, heps = A.heps, alpha1 = A.alpha1;
  const double lam = A.lam, alpha0 = A.alpha0, theta = A.theta;
  const bool inner_xy = lane >= R && lane < kW - R && ty >= R && ty < TH - R;
  const int tyd = ty + 1 < TH ? ty + 1 : ty;
  double fin_sum = 0.0, fin_max = 0.0;

  int k = blockIdx.x;
  if (k < cnt) {
    const int t0 = A.tiles ? A.tiles[1 + k] : k;
    stage_state<R, TH>(S, A, t0, ntx);
    stage_const<R, TH>(S, A, t0, ntx);
  }
  for (; k < cnt; k += gridDim.x) {
    const int tile = A.tiles ? A.tiles[1 + k] : k;
    const int gx = (tile % ntx) * OW - R + lane, gy = (tile / ntx) * OH - R + ty;
    const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
    const size_t i = in ? (size_t)gy * A.w + gx : 0;
    const bool more = k + (int)gridDim.x < cnt;
    const int nxt = more ? (A.tiles ? A.tiles[1 + k + gridDim.x] : k + gridDim.x) : 0;
    cp_wait_all();
    __syncthreads();
    const uint32_t code = S.code[ty][lane];
    const bool m = code & 1u, ex = code & 2u, ey = code & 4u;
    double u = S.stg[PU][ty][lane], v0 = S.stg[PV0][ty][lane], v1 = S.stg[PV1][ty][lane];
    double ub, vb0, vb1;
    if (A.first) {
      ub = u; vb0 = v0; vb1 = v1;
    } else {
      ub = S.stg[PUB][ty][lane]; vb0 = S.stg[PVB0][ty][lane]; vb1 = S.stg[PVB1][ty][lane];
    }
    double p0 = S.stg[PP0][ty][lane], p1 = S.stg[PP1][ty][lane];
    double q0 = S.stg[PQ0][ty][lane], q1 = S.stg[PQ1][ty][lane];
    double q2 = S.stg[PQ2][ty][lane], q3 = S.stg[PQ3][ty][lane];
    __syncthreads();  // state staging consumed: the next tile's state copies run under the cycles
    if (more) stage_state<R, TH>(S, A, nxt, ntx);

    for (int it = 0; it < A.iters; ++it) {
      S.xb[0][ty][lane] = ub;
      S.xb[1][ty][lane] = vb0;
      S.xb[2][ty][lane] = vb1;
      __syncthreads();
      const double a = S.cst[0][ty][lane], b = S.cst[1][ty][lane], c = S.cst[2][ty][lane];
      const double sp = S.cst[3][ty][lane] * alpha1;
      const double ubx = shfl_dn(ub), vbx0 = shfl_dn(vb0), vbx1 = shfl_dn(vb1);
      const double uby = S.xb[0][tyd][lane], vby0 = S.xb[1][tyd][lane];
      const double vby1 = S.xb[2][tyd][lane];
      const double gxx = ex ? ubx - ub : 0.0, gyy = ey ? uby - ub : 0.0;
      const double g00 = ex ? vbx0 - vb0 : 0.0, g01 = ey ? vby0 - vb0 : 0.0;
      const double g10 = ex ? vbx1 - vb1 : 0.0, g11 = ey ? vby1 - vb1 : 0.0;
      dual_update_exact<double>(a, b, c, sp, sq, gxx, gyy, g00, g01, g10, g11, vb0, vb1, p0, p1,
                                q0, q1, q2, q3, heps);
      const double fx0 = ex ? a * p0 + b * p1 : 0.0, fy0 = ey ? b * p0 + c * p1 : 0.0;
      const double fx1 = ex ? q0 : 0.0, fy1 = ey ? q1 : 0.0;
      const double fx2 = ex ? q2 : 0.0, fy2 = ey ? q3 : 0.0;
      S.fy[0][ty][lane] = fy0;
      S.fy[1][ty][lane] = fy1;
      S.fy[2][ty][lane] = fy2;
      if (DIAG) {
        double pn = 0.0, qn = 0.0;
        if (inner_xy && in) {
          pn = sqrt(p0 * p0 + p1 * p1);
          qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
        }
        pn = warp_max(pn);
        qn = warp_max(qn);
        if (lane == 0 && A.diag_p) {
          atomic_max_nonneg(A.diag_p + it, (float)pn);
          atomic_max_nonneg(A.diag_q + it, (float)qn);
        }
      }
      __syncthreads();
      const double lx0 = shfl_up(fx0), lx1 = shfl_up(fx1), lx2 = shfl_up(fx2);
      double uy0 = 0.0, uy1 = 0.0, uy2 = 0.0;
      if (ty > 0) { uy0 = S.fy[0][ty - 1][lane]; uy1 = S.fy[1][ty - 1][lane]; uy2 = S.fy[2][ty - 1][lane]; }
      const double dvv = ((fx0 - lx0) + fy0) - uy0;
      const double d0 = ((fx1 - lx1) + fy1) - uy1;
      const double d1 = ((fx2 - lx2) + fy2) - uy2;
      const double tu = S.cst[4][ty][lane], tv = S.cst[5][ty][lane], g = S.cst[6][ty][lane];
      const double rh = S.cst[7][ty][lane], uo_ = S.cst[8][ty][lane];
      primal_update_exact<double>(dvv, d0, d1, tu, tv, g, rh, uo_, p0, p1, lam, alpha0, alpha1,
                                  theta, u, v0, v1, ub, vb0, vb1);
    }
    const double uo = S.cst[8][ty][lane];
    __syncthreads();  // constants consumed: the next tile's constants copy under the stores
    if (more) stage_const<R, TH>(S, A, nxt, ntx);
    const bool st = inner_xy && in && m;
    if (A.fin && st) {  // clip / accumulate (solver.py:356-360)
      const double du = fmin(fmax(u - uo, -A.du_max), A.du_max);
      u = uo + du;
      const double2 dd = reinterpret_cast<const double2*>(A.dirs)[i];
      double2 wv = reinterpret_cast<double2*>(A.wv)[i];
      wv.x = wv.x + du * dd.x;
      wv.y = wv.y + du * dd.y;
      reinterpret_cast<double2*>(A.wv)[i] = wv;
      if (DIAG) {
        fin_sum += fabs(du);
        fin_max = fmax(fin_max, fabs(du));
      }
    }
    if (st) {
      if (A.first) A.uo[i] = uo;
      A.du[i] = u;
      A.dv[i] = v0; A.dv[n + i] = v1;
      A.dp[i] = p0; A.dp[n + i] = p1;
      A.dq[i] = q0; A.dq[n + i] = q1; A.dq[2 * n + i] = q2; A.dq[3 * n + i] = q3;
      if (!A.fin) {
        A.dub[i] = ub;
        A.dvb[i] = vb0; A.dvb[n + i] = vb1;
      }
    }
    if (DIAG && A.fin && (A.diag_du || A.diag_du64)) {
      __shared__ double s_sum[TH], s_max[TH];
      const double sm = warp_sum(fin_sum), mx = warp_max(fin_max);
      if (lane == 0) { s_sum[ty] = sm; s_max[ty] = mx; }
      __syncthreads();
      if (lane == 0 && ty == 0) {
        double t = 0.0, mm = 0.0;
        for (int r = 0; r < TH; ++r) { t += s_sum[r]; mm = fmax(mm, s_max[r]); }
        A.partials[tile] = t;
        if (A.diag_du64) atomic_max_nonneg(A.diag_du64, mm);
        else atomic_max_nonneg(A.diag_du, (float)mm);
      }
      fin_sum = 0.0;
      fin_max = 0.0;
    }
  }
  cp_wait_all();
}

// Edge code per pixel of a level: bit0 mask, bit1 x-edge in the mask
// (m(x) & m(x+1)), bit2 y-edge (m(y) & m(y+1)) — rasters.py:175-182.
__global__ void k64_edge_codes(const uint8_t* __restrict__ m, int w, int h,
                               uint32_t* __restrict__ code) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= w) return;
  const size_t i = (size_t)y * w + x;
  const bool mm = m[i];
  const bool ex = mm && x + 1 < w && m[i + 1];
  const bool ey = mm && y + 1 < h && m[i + w];
  code[i] = (mm ? 1u : 0u) | (ex ? 2u : 0u) | (ey ? 4u : 0u);
}

template <int R, int TH, bool DIAG>
int launch_pipe_cs(const B64& A, cudaStream_t st) {
  const size_t dyn = sizeof(PipeSmemCS<TH>);
  static std::atomic<unsigned long long> attr{0};
  static int sms = 0;
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k64_pipe_cs<R, TH, DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dyn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  const int ntiles = ((A.w + OW - 1) / OW) * ((A.h + OH - 1) / OH);
  const int grid = ntiles < 2 * sms ? ntiles : 2 * sms;
  k64_pipe_cs<R, TH, DIAG><<<grid, dim3(kW, TH), dyn, st>>>(A);
  return launch_status();
}

template <int R, int TH, bool DIAG>
int launch_pipe(const B64& A, cudaStream_t st) {
  const size_t dyn = sizeof(PipeSmem<TH>);
  static std::atomic<unsigned long long> attr{0};
  static int sms = 0;
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k64_pipe<R, TH, DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dyn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  constexpr int OW = kW - 2 * R, OH = TH - 2 * R;
  const int ntiles = ((A.w + OW - 1) / OW) * ((A.h + OH - 1) / OH);
  const int grid = ntiles < sms ? ntiles : sms;
  k64_pipe<R, TH, DIAG><<<grid, dim3(kW, TH), dyn, st>>>(A);
  return launch_status();
}

int pipe_th() {
  static const int v = [] {
    const char* e = getenv("FSB_PD64_TH");
    return e ? atoi(e) : 24;
  }();
  return v;
}

template <int R, int TH>
int launch_th(const B64& A, cudaStream_t st) {
  const bool diag = A.diag_p || A.diag_du || A.diag_du64;
  return diag ? launch_pipe<R, TH, true>(A, st) : launch_pipe<R, TH, false>(A, st);
}

template <int R>
int launch_r(const B64& A, cudaStream_t st) {
  if (pipe_th() == 116) {  // FSB_PD64_TH=116: 2 CTAs / SM, 16-row tiles, constants in smem
    const bool diag = A.diag_p || A.diag_du || A.diag_du64;
    return diag ? launch_pipe_cs<R, 16, true>(A, st) : launch_pipe_cs<R, 16, false>(A, st);
  }
  switch (pipe_th()) {
    case 16: return launch_th<R, 16>(A, st);
    case 32: return launch_th<R, 32>(A, st);
    default: return launch_th<R, 24>(A, st);
  }
}

}  // namespace

size_t pd64_pipe_count(int w, int h, int halo) {
  const int TH = pipe_th() == 116 ? 16 : pipe_th();
  const int OW = kW - 2 * halo, OH = TH - 2 * halo;
  return (size_t)((w + OW - 1) / OW) * ((h + OH - 1) / OH);
}

int pd64_pipe_tile_list(const uint8_t* mask, int w, int h, int halo, int* tiles,
                        cudaStream_t st) {
  return tile_list_internal(mask, w, h, kW - 2 * halo,
                            (pipe_th() == 116 ? 16 : pipe_th()) - 2 * halo, tiles, st);
}

int pd64_edge_codes(const uint8_t* mask, int w, int h, uint32_t* code, cudaStream_t st) {
  k64_edge_codes<<<dim3((w + 127) / 128, h), 128, 0, st>>>(mask, w, h, code);
  return launch_status();
}

int pd64_pipe_launch(const B64& A, int halo, cudaStream_t st) {
  if (A.iters < 1 || A.iters > halo || !A.ecode) return FSB_EINVAL;
  switch (halo) {
    case 2: return launch_r<2>(A, st);
    case 3: return launch_r<3>(A, st);
    default: return FSB_EINVAL;
  }
}

}  // namespace fsb
