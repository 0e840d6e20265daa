// k64_level: the whole warp loop of a small float64 pyramid level in one
// cluster launch.
//
// On the small levels (C3: 64^2) every warp is four dependent launches
// (sampling, linearisation, two primal-dual launches) over a grid that fills a
// fraction of the GPU, so a warp costs launch and memory latencies, not work.
// Here one cluster of up to 16 CTAs holds the whole level: each CTA one
// 32 x kH tile, one pixel per thread, the primal-dual state, the warp and the
// per-level constants in registers for all N warps. Per warp:
//   * sampling at x + w from the level's NaN-encoded texels (sample_nan_px);
//     the sampled image goes to a global scratch plane (double-buffered by
//     warp parity) and a release / acquire cluster barrier publishes it;
//   * linearisation from that plane (linearize_nan_px; plain coherent loads);
//   * K cycles: in-CTA exchange through shared memory with 2 barriers per
//     cycle; across CTA edges the row / column values are pushed with
//     st.async into the neighbour's shared memory and counted on its
//     mbarrier (as k64_ctile), double-buffered by cycle parity;
//   * clip / accumulate of w in registers.
// u, v and w are written once at the end. No halo: the cluster covers the
// level, so the cluster's border is the image border (fluxes across it are 0).
//
// Reference: solver.py:331-365 (solve_level warp loop), 279-303
// (primal_dual_iterate), 332-346 and 192-202 (warp prologue).

#include <cooperative_groups.h>
#include <stdlib.h>
#include <string.h>

#include "pd64_block.cuh"
#include "pd_math.cuh"
#include "sample64.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace fsb {

namespace {

constexpr int kW = 32;

template <int kH>
struct LvlSmem {
  double ub[kH][kW], vb0[kH][kW], vb1[kH][kW];  // dual step: u_bar, v_bar rows
  double fy[3][kH][kW];                         // primal step: y-fluxes
  double dn[2][3][kW];  // dual: row 0 of the CTA below (st.async)
  double rt[2][3][kH];  // dual: column 0 of the CTA to the right
  double up[2][3][kW];  // primal: last-row y-fluxes of the CTA above
  double lf[2][3][kH];  // primal: column 31 x-fluxes of the CTA to the left
  double red_sum[kH], red_max[kH];  // diagnostics: per-warp |du| sums / maxima
  uint64_t bd[2], bp[2];
};

FSB_INLINE double shfl_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
FSB_INLINE double shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

// A CTA's place in its cluster and the neighbours it exchanges with.
struct Nbr {
  int rank, cx_n;  // rank; cluster width in CTAs
  bool has_r, has_l, has_d, has_u;
  uint32_t dual_bytes, primal_bytes;  // bytes each exchange phase receives
};
template <int kH>
FSB_INLINE Nbr make_nbr(int rank, int CX, int CY) {
  Nbr e;
  const int cx = rank % CX, cy = rank / CX;
  e.rank = rank; e.cx_n = CX;
  e.has_r = cx + 1 < CX; e.has_l = cx > 0; e.has_d = cy + 1 < CY; e.has_u = cy > 0;
  e.dual_bytes = (e.has_d ? 3 * kW * 8 : 0) + (e.has_r ? 3 * kH * 8 : 0);
  e.primal_bytes = (e.has_u ? 3 * kW * 8 : 0) + (e.has_l ? 3 * kH * 8 : 0);
  return e;
}
struct PdConst {  // per-pixel constants of the cycles
  double a, b, c, sp, tu, tv, g, rh, uo;
  bool ex, ey;
};
struct PdScal {
  double sq, heps, lam, alpha0, alpha1, theta;
};

// K primal-dual cycles (solver.py:279-303) of a warp, starting from the
// warp-start reset u_bar = u, v_bar = v; in-CTA y-neighbours through shared
// memory, x-neighbours by shuffle, across CTA edges by st.async pushes counted
// on the receiver's mbarriers (parity buffers by the running cycle index cyc).
// Left of column 0 / above row 0 without a neighbour CTA the fluxes are 0 (the
// image border; at a region border these are halo pixels).
// DIAG: per-cycle maxima of |p| and |q| over the CTA's pixels into dp[cyc],
// dq[cyc] (solver.py:350-354; out-of-image threads hold p = q = 0).
template <int kH, bool DIAG>
FSB_INLINE void pd_cycles(LvlSmem<kH>& S, const Nbr& E, const PdConst& C, const PdScal& Q, int K,
                          int& cyc, double& u, double& v0, double& v1, double& p0, double& p1,
                          double& q0, double& q1, double& q2, double& q3, float* dp = nullptr,
                          float* dq = nullptr) {
  const int lane = threadIdx.x, ty = threadIdx.y, tid = ty * kW + lane;
  const int tyd = ty + 1 < kH ? ty + 1 : ty;
  const bool ex = C.ex, ey = C.ey;
  double ub = u, vb0 = v0, vb1 = v1;
  for (int it = 0; it < K; ++it, ++cyc) {
    const int par = cyc & 1;
    const uint32_t ph = (uint32_t)(cyc >> 1) & 1u;
    S.ub[ty][lane] = ub;
    S.vb0[ty][lane] = vb0;
    S.vb1[ty][lane] = vb1;
    if (ty == 0 && E.has_u) {
      const int rk = E.rank - E.cx_n;
      const uint32_t bar = mapa(&S.bd[par], rk);
      st_async(mapa(&S.dn[par][0][lane], rk), ub, bar);
      st_async(mapa(&S.dn[par][1][lane], rk), vb0, bar);
      st_async(mapa(&S.dn[par][2][lane], rk), vb1, bar);
    }
    if (lane == 0 && E.has_l) {
      const int rk = E.rank - 1;
      const uint32_t bar = mapa(&S.bd[par], rk);
      st_async(mapa(&S.rt[par][0][ty], rk), ub, bar);
      st_async(mapa(&S.rt[par][1][ty], rk), vb0, bar);
      st_async(mapa(&S.rt[par][2][ty], rk), vb1, bar);
    }
    if (tid == 0) mbar_expect_tx(&S.bd[par], E.dual_bytes);
    __syncthreads();
    // forward differences (rasters.py:144-155), zero where the edge leaves the mask
    double ubx = shfl_dn(ub), vbx0 = shfl_dn(vb0), vbx1 = shfl_dn(vb1);
    double uby = S.ub[tyd][lane], vby0 = S.vb0[tyd][lane], vby1 = S.vb1[tyd][lane];
    if (E.has_r || (ty == kH - 1 && E.has_d)) {  // warp-uniform wait
      mbar_wait(&S.bd[par], ph);
      if (lane == kW - 1 && E.has_r) {
        ubx = S.rt[par][0][ty]; vbx0 = S.rt[par][1][ty]; vbx1 = S.rt[par][2][ty];
      }
      if (ty == kH - 1 && E.has_d) {
        uby = S.dn[par][0][lane]; vby0 = S.dn[par][1][lane]; vby1 = S.dn[par][2][lane];
      }
    }
    const double gxx = ex ? ubx - ub : 0.0, gyy = ey ? uby - ub : 0.0;
    const double g00 = ex ? vbx0 - vb0 : 0.0, g01 = ey ? vby0 - vb0 : 0.0;
    const double g10 = ex ? vbx1 - vb1 : 0.0, g11 = ey ? vby1 - vb1 : 0.0;
    dual_update_exact<double>(C.a, C.b, C.c, C.sp, Q.sq, gxx, gyy, g00, g01, g10, g11, vb0, vb1,
                              p0, p1, q0, q1, q2, q3, Q.heps);
    const double fx0 = ex ? C.a * p0 + C.b * p1 : 0.0;
    const double fy0 = ey ? C.b * p0 + C.c * p1 : 0.0;
    const double fx1 = ex ? q0 : 0.0, fy1 = ey ? q1 : 0.0;
    const double fx2 = ex ? q2 : 0.0, fy2 = ey ? q3 : 0.0;
    S.fy[0][ty][lane] = fy0;
    S.fy[1][ty][lane] = fy1;
    S.fy[2][ty][lane] = fy2;
    if (DIAG) {
      const double pmax = warp_max(sqrt(p0 * p0 + p1 * p1));
      const double qmax = warp_max(sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3));
      if (lane == 0) {
        atomic_max_nonneg(dp + cyc, (float)pmax);
        atomic_max_nonneg(dq + cyc, (float)qmax);
      }
    }
    if (ty == kH - 1 && E.has_d) {
      const int rk = E.rank + E.cx_n;
      const uint32_t bar = mapa(&S.bp[par], rk);
      st_async(mapa(&S.up[par][0][lane], rk), fy0, bar);
      st_async(mapa(&S.up[par][1][lane], rk), fy1, bar);
      st_async(mapa(&S.up[par][2][lane], rk), fy2, bar);
    }
    if (lane == kW - 1 && E.has_r) {
      const int rk = E.rank + 1;
      const uint32_t bar = mapa(&S.bp[par], rk);
      st_async(mapa(&S.lf[par][0][ty], rk), fx0, bar);
      st_async(mapa(&S.lf[par][1][ty], rk), fx1, bar);
      st_async(mapa(&S.lf[par][2][ty], rk), fx2, bar);
    }
    if (tid == 0) mbar_expect_tx(&S.bp[par], E.primal_bytes);
    __syncthreads();
    // backward divergence (rasters.py:158-172)
    double lx0 = shfl_up(fx0), lx1 = shfl_up(fx1), lx2 = shfl_up(fx2);
    if (lane == 0) lx0 = lx1 = lx2 = 0.0;
    double uy0 = 0.0, uy1 = 0.0, uy2 = 0.0;
    if (ty > 0) {
      uy0 = S.fy[0][ty - 1][lane]; uy1 = S.fy[1][ty - 1][lane]; uy2 = S.fy[2][ty - 1][lane];
    }
    if (E.has_l || (ty == 0 && E.has_u)) {
      mbar_wait(&S.bp[par], ph);
      if (lane == 0 && E.has_l) {
        lx0 = S.lf[par][0][ty]; lx1 = S.lf[par][1][ty]; lx2 = S.lf[par][2][ty];
      }
      if (ty == 0 && E.has_u) {
        uy0 = S.up[par][0][lane]; uy1 = S.up[par][1][lane]; uy2 = S.up[par][2][lane];
      }
    }
    const double dvv = ((fx0 - lx0) + fy0) - uy0;
    const double dd0 = ((fx1 - lx1) + fy1) - uy1;
    const double dd1 = ((fx2 - lx2) + fy2) - uy2;
    primal_update_exact<double>(dvv, dd0, dd1, C.tu, C.tv, C.g, C.rh, C.uo, p0, p1, Q.lam,
                                Q.alpha0, Q.alpha1, Q.theta, u, v0, v1, ub, vb0, vb1);
  }
}

struct LvlArgs {
  P64 P;                    // the level's prologue view (tex, i0, mask, h, w)
  const double* T;          // tensor a, b, c planes
  const double* S;          // sigma_p, tau_u, tau_v planes
  const uint32_t* ecode;    // edge codes (bit0 mask, bit1 x-edge, bit2 y-edge)
  double* u;                // in: level start; out: result
  double* v;                // out: v (2 planes)
  double* wv;               // in / out: (h, w, 2)
  double* i1wn[2];          // scratch planes: the sampled image by warp parity
  double lam, alpha0, alpha1, theta, sigma_q, heps, du_max;
  int N, K;
  // diagnostics (nullptr = off): per-cycle |p| / |q| maxima, per-warp max |du|
  // (float or float64) and per-warp per-CTA partial sums of |du| (N x CTAs)
  float* diag_p; float* diag_q; float* diag_du; double* diag_du64; double* partials;
};

template <int kH, int CX, bool DIAG>
__global__ void __launch_bounds__(kW * kH, 1) k64_level(const LvlArgs A) {
  extern __shared__ unsigned char smem_raw[];
  poison_dynamic_smem(smem_raw);  // checked build only
  LvlSmem<kH>& S = *reinterpret_cast<LvlSmem<kH>*>(smem_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), ncta = (int)cl.num_blocks();
  const int cx = rank % CX, cy = rank / CX, CY = ncta / CX;
  const int lane = threadIdx.x, ty = threadIdx.y, tid = ty * kW + lane;
  const int W = A.P.w, H = A.P.h;
  const size_t n = (size_t)W * H;
  const int x = cx * kW + lane, y = cy * kH + ty;
  const bool in = x < W && y < H;
  const size_t i = in ? (size_t)y * W + x : 0;
  const Nbr E = make_nbr<kH>(rank, CX, CY);
  if (tid == 0) {
    for (int j = 0; j < 2; ++j) {
      mbar_init(&S.bd[j], 1);
      mbar_init(&S.bp[j], 1);
    }
    mbar_init_fence();
  }
  // per-pixel constants, state and warp (v, p, q start at zero: solver.py:323-327)
  const uint32_t code = in ? A.ecode[i] : 0u;
  const bool m = code & 1u, ex = code & 2u, ey = code & 4u;
  const double a = in ? A.T[i] : 0.0, b = in ? A.T[n + i] : 0.0, c = in ? A.T[2 * n + i] : 0.0;
  const double sp = in ? A.S[i] * A.alpha1 : 0.0;
  const double tu = in ? A.S[n + i] : 0.0, tv = in ? A.S[2 * n + i] : 0.0;
  const double i0 = in ? A.P.i0[i] : 0.0;
  double u = in ? A.u[i] : 0.0, v0 = 0.0, v1 = 0.0, p0 = 0.0, p1 = 0.0;
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
  double2 wv = in ? reinterpret_cast<const double2*>(A.wv)[i] : make_double2(0.0, 0.0);
  const PdScal Q{A.sigma_q * A.alpha0, A.heps, A.lam, A.alpha0, A.alpha1, A.theta};
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  cluster_sync_rel_acq();  // every CTA's mbarriers are initialised

  int cyc = 0;  // running cycle index: exchange buffer parity and mbarrier phase
  for (int wi = 0; wi < A.N; ++wi) {
    // ---- sampling at x + w (solver.py:332-337)
    double iwn = nan, d0 = 0.0, d1 = 0.0;
    bool dok = false;
    if (in && m) sample_nan_px(A.P, x, y, wv, iwn, d0, d1, dok);
    double* i1wn = A.i1wn[wi & 1];
    if (in) i1wn[i] = iwn;
    cluster_sync_rel_acq();  // the sampled image of the whole level is visible
    // ---- I_u and rho0 (solver.py:339-343, image_derivative_along 192-202)
    double g = 0.0, rh = 0.0;
    if (in) {
      auto tap = [&](int r, int cc) {
        return ((unsigned)r < (unsigned)H && (unsigned)cc < (unsigned)W)
                   ? i1wn[(size_t)r * W + cc]
                   : nan;
      };
      linearize_nan_px(A.P, x, y, iwn, i0, make_double2(d0, d1), dok, tap, g, rh);
    }
    // warp-start reset (solver.py:344-346): u0 = u, u_bar = u, v_bar = v
    const double uo = u;
    const PdConst C{a, b, c, sp, tu, tv, g, rh, uo, ex, ey};
    pd_cycles<kH, DIAG>(S, E, C, Q, A.K, cyc, u, v0, v1, p0, p1, q0, q1, q2, q3, A.diag_p,
                        A.diag_q);
    // ---- clip and accumulate (solver.py:356-360)
    double adu = 0.0;
    if (in && m) {
      const double du = fmin(fmax(u - uo, -A.du_max), A.du_max);
      u = uo + du;
      wv.x = wv.x + du * d0;
      wv.y = wv.y + du * d1;
      adu = fabs(du);
    }
    if (DIAG && A.partials) {  // max |du| and this CTA's sum of |du| for warp wi
      const double mx = warp_max(adu), sm = warp_sum(adu);
      if (lane == 0) { S.red_sum[ty] = sm; S.red_max[ty] = mx; }
      __syncthreads();
      if (tid == 0) {
        double tsum = 0.0, mm = 0.0;
        for (int j = 0; j < kH; ++j) { tsum += S.red_sum[j]; mm = fmax(mm, S.red_max[j]); }
        A.partials[(size_t)wi * ncta + rank] = tsum;
        if (A.diag_du64) atomic_max_nonneg(A.diag_du64 + wi, mm);
        else atomic_max_nonneg(A.diag_du + wi, (float)mm);
      }
      __syncthreads();  // the reduction slots are reused by the next warp
    }
  }
  if (in) {
    A.u[i] = u;
    A.v[i] = v0;
    A.v[n + i] = v1;
    reinterpret_cast<double2*>(A.wv)[i] = wv;
  }
  // no CTA may leave while a neighbour's last pushes target its shared memory:
  // every push was awaited by its receiver, so only the receivers' own exits
  // matter, and each CTA waited for everything sent to it
}

struct LvlShape {
  int th, cx, cy;
};

// Tiles of 32 x kH (kH 8 or 16) covering the level with at most 16 CTAs, the
// most CTAs first; {0, 0, 0} if the level does not fit one cluster. (32-row
// tiles — 1024 threads, 64 registers — spill the sampler: C3 128^2 took
// 47.6 instead of 26.1 us per warp.)
LvlShape level_shape(int w, int h) {
  const int cx = (w + kW - 1) / kW;
  for (int th : {8, 16}) {
    const int cy = (h + th - 1) / th;
    if (cx * cy <= 16 && cx <= 4) return {th, cx, cy};
  }
  return {0, 0, 0};
}

template <int kH, int CX>
int launch_level(const LvlArgs& A, int cy, cudaStream_t st) {
  const bool diag = A.diag_p || A.partials;
  auto kern = diag ? k64_level<kH, CX, true> : k64_level<kH, CX, false>;
  const int nc = CX * cy;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [&] {
    for (auto k : {k64_level<kH, CX, true>, k64_level<kH, CX, false>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(LvlSmem<kH>));
    }
  });
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)nc);
  cfg.blockDim = dim3(kW, kH);
  cfg.dynamicSmemBytes = sizeof(LvlSmem<kH>);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, A);
  if (e != cudaSuccess) return (int)e;
  return launch_status();
}

template <int kH>
int launch_level_th(const LvlArgs& A, const LvlShape& s, cudaStream_t st) {
  switch (s.cx) {
    case 1: return launch_level<kH, 1>(A, s.cy, st);
    case 2: return launch_level<kH, 2>(A, s.cy, st);
    case 3: return launch_level<kH, 3>(A, s.cy, st);
    case 4: return launch_level<kH, 4>(A, s.cy, st);
    default: return FSB_EINVAL;
  }
}

}  // namespace

int pd64_level_ctas(int w, int h) {
  const LvlShape s = level_shape(w, h);
  return s.cx * s.cy;
}

bool pd64_level_fits(int w, int h) {
  static const bool on = [] {
    const char* e = getenv("FSB_LEVEL64");
    return !(e && e[0] == '0');
  }();
  return on && level_shape(w, h).th > 0;
}

int pd64_level_launch(const P64& P, const double* T, const double* S, const uint32_t* ecode,
                      double* u, double* v, double* wv, double* scratch2, double lam,
                      double alpha0, double alpha1, double theta, double sigma_q, double heps,
                      double du_max, int N, int K, const LvlDiag* diag, cudaStream_t st) {
  const LvlShape s = level_shape(P.w, P.h);
  if (!s.th) return FSB_EINVAL;
  LvlArgs A;
  memset(&A, 0, sizeof(A));
  A.P = P; A.T = T; A.S = S; A.ecode = ecode; A.u = u; A.v = v; A.wv = wv;
  A.i1wn[0] = scratch2;
  A.i1wn[1] = scratch2 + (size_t)P.w * P.h;
  A.lam = lam; A.alpha0 = alpha0; A.alpha1 = alpha1; A.theta = theta; A.sigma_q = sigma_q;
  A.heps = heps; A.du_max = du_max; A.N = N; A.K = K;
  if (diag) {
    A.diag_p = diag->p; A.diag_q = diag->q; A.diag_du = diag->du; A.diag_du64 = diag->du64;
    A.partials = diag->partials;
  }
  return s.th == 8 ? launch_level_th<8>(A, s, st) : launch_level_th<16>(A, s, st);
}

}  // namespace fsb
