// k64_ctile: the float64 primal-dual kernel of the large levels (512^2 and up)
// as cluster tiles — halo exchange through distributed shared memory inside a
// cluster, redundant halo cycles only at the cluster's border.
//
// k64_tile / k64_tma run R = 2 cycles per launch on 32 x 16 tiles: every tile
// recomputes a 2-pixel halo, and a warp's K = 10 cycles cost 5 round trips of
// the 12 state + 10 constant planes through HBM — the launch is bound by that
// traffic (profiles/r02_pd64_ncu.txt). Here a cluster of CX x CY CTAs covers
// one region of (CX 32) x (CY kH) pixels (each CTA one 32 x kH tile, one pixel
// per thread, state in registers, constants in shared memory) and runs R = 5
// cycles per launch: a warp is 2 launches instead of 5, and only the region's
// outer R-pixel border is halo. Default: 2 x 8 clusters of 32 x 8 CTAs (256
// threads, 4 CTAs per SM) — a 64 x 64 region with a 54 x 54 interior, 1.40
// pixel-cycles per solved pixel-cycle against k64_tile's 1.52.
//
// Across a CTA edge the neighbour values of a half-cycle (dual: the u_bar /
// v_bar row 0 and column 0; primal: the y-fluxes of the last row and the
// x-fluxes of column 31) are PUSHED into the neighbour CTA's shared memory
// with st.async, completing bytes on its mbarrier; the receiver waits on that
// mbarrier, and inside the CTA two __syncthreads per cycle remain. No cluster
// barrier in the cycles: a release-ordered barrier.cluster costs a MEMBAR.GPU
// per use, which made a first version with 2 cluster barriers per cycle slower
// than k64_tile. Receive buffers and mbarriers are double-buffered by cycle
// parity; a neighbour can run at most one half-cycle ahead, because every push
// direction has a reverse one between the same two CTAs.
//
// Loads: two TMA boxes per CTA (state: 12 planes, the warp's first launch 9;
// constants: 10 planes with the edge codes) 34 columns wide from an even
// column (16-B aligned rows), zero outside the image. Stores: the region
// interior, per pixel from registers. Arithmetic and neighbour values are
// those of k64_tile, so interior results agree with it to FMA-contraction
// round-off (tests/test_gpu_variants.py).
//
// Reference: solver.py:279-303 (primal_dual_iterate), 344-360 (warp-start
// reset, clip / accumulate epilogue), rasters.py:144-182.

#include <cooperative_groups.h>
#include <stdlib.h>
#include <string.h>

#include "pd64_block.cuh"
#include "pd_math.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace fsb {

bool make_map64(CUtensorMap* m, const double* base, int w, int h, int planes, int bw, int bh,
                int bp);
int tile_list_internal(const uint8_t* mask, int w, int h, int TW, int TH, int* tiles,
                       cudaStream_t st);

namespace {

constexpr int kW = 32, kBW = kW + 2;  // load box: 2 spare columns for the even start
constexpr int kSt = 12, kSt0 = 9, kCst = 10;
enum { PU, PV0, PV1, PP0, PP1, PQ0, PQ1, PQ2, PQ3, PUB, PVB0, PVB1 };
enum { CA, CB, CC, CSP, CTU, CTV, CIU, CRH, CUO, CCODE };

// in-CTA exchange buffers, aliased on the state box once the tile is in registers
template <int kH>
struct XchC {
  double ub[kH][kW], vb0[kH][kW], vb1[kH][kW];  // dual step: u_bar, v_bar rows
  double fy[3][kH][kW];                         // primal step: y-fluxes
};
// Cross-CTA values, pushed by the neighbour CTA with st.async (double-buffered
// by cycle parity; each buffer completes one mbarrier phase per 2 cycles).
template <int kH>
struct RecvC {
  double dn[2][3][kW];  // dual: row 0 (u_bar, v_bar) of the CTA below
  double rt[2][3][kH];  // dual: column 0 of the CTA to the right
  double up[2][3][kW];  // primal: row 15 y-fluxes of the CTA above
  double lf[2][3][kH];  // primal: column 31 x-fluxes of the CTA to the left
  uint64_t bd[2], bp[2];  // dual / primal mbarriers
};
template <int kH>
struct SmemC {
  static constexpr int kPl = kBW * kH;  // doubles per staged plane
  double st[kSt][kPl];   // state box | XchC
  double cs[kCst][kPl];  // constant box, read through the cycles
  RecvC<kH> rv;
  double red_sum[kH], red_max[kH];
  uint64_t bar;
  static_assert(sizeof(XchC<kH>) <= sizeof(double) * kSt * kPl, "exchange aliases the state box");
  static_assert(sizeof(double) * kSt * kPl % 128 == 0, "TMA boxes must stay 128-byte aligned");
};
template <int kH>
constexpr size_t smem_bytes() { return sizeof(SmemC<kH>) + 128; }

FSB_INLINE double shfl_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
FSB_INLINE double shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

// kH rows per CTA: 16 (512 threads, 2 CTAs per SM), 8 (256 threads, 4 per SM) or 4
template <int R, int CX, int CY, int kH, bool DIAG>
__global__ void __launch_bounds__(kW * kH, 1024 / (kW * kH))
    k64_ctile(const B64 A, const __grid_constant__ CUtensorMap m_ld,
              const __grid_constant__ CUtensorMap m_cst, int nrx) {
  constexpr int NC = CX * CY, RW = CX * kW, RH = CY * kH, IW = RW - 2 * R, IH = RH - 2 * R;
  extern __shared__ unsigned char smem_raw[];
  poison_dynamic_smem(smem_raw);  // checked build only
  constexpr int kPl = SmemC<kH>::kPl;
  SmemC<kH>& S =
      *reinterpret_cast<SmemC<kH>*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  XchC<kH>& X = *reinterpret_cast<XchC<kH>*>(&S.st[0][0]);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), cx = rank % CX, cy = rank / CX;
  const int k = (int)blockIdx.x / NC;  // the cluster's work-list entry
  if (k >= A.tiles[0]) return;         // uniform over the cluster
  const int r = A.tiles[1 + k], rx = r % nrx, ry = r / nrx;
  const int ox = rx * IW - R + cx * kW, oy = ry * IH - R + cy * kH;  // tile origin
  const int bx0 = ox & ~1;                                         // even box start
  const int lane = threadIdx.x, ty = threadIdx.y, tid = ty * kW + lane;
  const int s = ty * kBW + lane + (ox - bx0);
  const bool first = A.first, fin = A.fin;
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    for (int j = 0; j < 2; ++j) {
      mbar_init(&S.rv.bd[j], 1);
      mbar_init(&S.rv.bp[j], 1);
    }
    mbar_init_fence();
    mbar_expect_tx(&S.bar, (uint32_t)(((first ? kSt0 : kSt) + kCst) * kPl * sizeof(double)));
    tma_load_3d(&S.st[0][0], &m_ld, bx0, oy, 0, &S.bar);
    tma_load_3d(&S.cs[0][0], &m_cst, bx0, oy, 0, &S.bar);
  }
  const int W = A.w, H = A.h;
  const int gx = ox + lane, gy = oy + ty;
  const int qx = cx * kW + lane, qy = cy * kH + ty;  // position in the region
  const bool inner = qx >= R && qx < RW - R && qy >= R && qy < RH - R &&
                     (unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H;
  const double alpha1 = A.alpha1, sq = A.sigma_q * A.alpha0, heps = A.heps;
  const double lam = A.lam, alpha0 = A.alpha0, theta = A.theta;
  const bool has_r = cx + 1 < CX, has_l = cx > 0, has_d = cy + 1 < CY, has_u = cy > 0;
  // bytes each exchange phase brings in from the neighbours
  const uint32_t dual_bytes = (has_d ? 3 * kW * 8 : 0) + (has_r ? 3 * kH * 8 : 0);
  const uint32_t primal_bytes = (has_u ? 3 * kW * 8 : 0) + (has_l ? 3 * kH * 8 : 0);
  // every CTA's mbarriers are initialised before any neighbour pushes into it
  cluster_arrive_relaxed();
  cluster_wait();
  mbar_wait(&S.bar, 0);
  double u = S.st[PU][s], v0 = S.st[PV0][s], v1 = S.st[PV1][s];
  double p0 = S.st[PP0][s], p1 = S.st[PP1][s];
  double q0 = S.st[PQ0][s], q1 = S.st[PQ1][s], q2 = S.st[PQ2][s], q3 = S.st[PQ3][s];
  double ub, vb0, vb1;
  if (first) {  // warp-start reset (solver.py:344-346): u0 = u, u_bar = u, v_bar = v
    ub = u; vb0 = v0; vb1 = v1;
    S.cs[CUO][s] = u;  // read back by this thread only
  } else {
    ub = S.st[PUB][s]; vb0 = S.st[PVB0][s]; vb1 = S.st[PVB1][s];
  }
  const double sp = S.cs[CSP][s] * alpha1;
  const uint32_t code = (uint32_t)S.cs[CCODE][s];  // 0 outside the image (zero fill)
  const bool m = code & 1u, ex = code & 2u, ey = code & 4u;
  __syncthreads();  // the state box is in registers: it becomes the exchange buffers

  for (int it = 0; it < A.iters; ++it) {
    const int par = it & 1;
    const uint32_t ph = (uint32_t)(it >> 1) & 1u;  // phase parity of the par buffers
    X.ub[ty][lane] = ub;
    X.vb0[ty][lane] = vb0;
    X.vb1[ty][lane] = vb1;
    // push this CTA's row 0 up and column 0 left (the neighbours' y+1 / x+1 values)
    if (ty == 0 && has_u) {
      const int rk = rank - CX;
      const uint32_t bar = mapa(&S.rv.bd[par], rk);
      st_async(mapa(&S.rv.dn[par][0][lane], rk), ub, bar);
      st_async(mapa(&S.rv.dn[par][1][lane], rk), vb0, bar);
      st_async(mapa(&S.rv.dn[par][2][lane], rk), vb1, bar);
    }
    if (lane == 0 && has_l) {
      const int rk = rank - 1;
      const uint32_t bar = mapa(&S.rv.bd[par], rk);
      st_async(mapa(&S.rv.rt[par][0][ty], rk), ub, bar);
      st_async(mapa(&S.rv.rt[par][1][ty], rk), vb0, bar);
      st_async(mapa(&S.rv.rt[par][2][ty], rk), vb1, bar);
    }
    if (tid == 0) mbar_expect_tx(&S.rv.bd[par], dual_bytes);
    __syncthreads();
    const double a = S.cs[CA][s], b = S.cs[CB][s], c = S.cs[CC][s];
    // forward differences (rasters.py:144-155), zero where the edge leaves the
    // mask; across a CTA edge the neighbour's values arrive by st.async
    double ubx = shfl_dn(ub), vbx0 = shfl_dn(vb0), vbx1 = shfl_dn(vb1);
    double uby, vby0, vby1;
    if (ty + 1 < kH) {
      uby = X.ub[ty + 1][lane]; vby0 = X.vb0[ty + 1][lane]; vby1 = X.vb1[ty + 1][lane];
    } else {  // region border: halo pixel (own values)
      uby = ub; vby0 = vb0; vby1 = vb1;
    }
    // warp-uniform wait (a lane-divergent one splits the warp through the cycle)
    if (has_r || (ty == kH - 1 && has_d)) {
      mbar_wait(&S.rv.bd[par], ph);
      if (lane == kW - 1 && has_r) {
        ubx = S.rv.rt[par][0][ty]; vbx0 = S.rv.rt[par][1][ty]; vbx1 = S.rv.rt[par][2][ty];
      }
      if (ty == kH - 1 && has_d) {
        uby = S.rv.dn[par][0][lane]; vby0 = S.rv.dn[par][1][lane]; vby1 = S.rv.dn[par][2][lane];
      }
    }
    const double gxx = ex ? ubx - ub : 0.0, gyy = ey ? uby - ub : 0.0;
    const double g00 = ex ? vbx0 - vb0 : 0.0, g01 = ey ? vby0 - vb0 : 0.0;
    const double g10 = ex ? vbx1 - vb1 : 0.0, g11 = ey ? vby1 - vb1 : 0.0;
    dual_update_exact<double>(a, b, c, sp, sq, gxx, gyy, g00, g01, g10, g11, vb0, vb1, p0, p1, q0,
                              q1, q2, q3, heps);
    const double fx0 = ex ? a * p0 + b * p1 : 0.0;
    const double fy0 = ey ? b * p0 + c * p1 : 0.0;
    const double fx1 = ex ? q0 : 0.0, fy1 = ey ? q1 : 0.0;
    const double fx2 = ex ? q2 : 0.0, fy2 = ey ? q3 : 0.0;
    X.fy[0][ty][lane] = fy0;
    X.fy[1][ty][lane] = fy1;
    X.fy[2][ty][lane] = fy2;
    // push row 15's y-fluxes down and column 31's x-fluxes right
    if (ty == kH - 1 && has_d) {
      const int rk = rank + CX;
      const uint32_t bar = mapa(&S.rv.bp[par], rk);
      st_async(mapa(&S.rv.up[par][0][lane], rk), fy0, bar);
      st_async(mapa(&S.rv.up[par][1][lane], rk), fy1, bar);
      st_async(mapa(&S.rv.up[par][2][lane], rk), fy2, bar);
    }
    if (lane == kW - 1 && has_r) {
      const int rk = rank + 1;
      const uint32_t bar = mapa(&S.rv.bp[par], rk);
      st_async(mapa(&S.rv.lf[par][0][ty], rk), fx0, bar);
      st_async(mapa(&S.rv.lf[par][1][ty], rk), fx1, bar);
      st_async(mapa(&S.rv.lf[par][2][ty], rk), fx2, bar);
    }
    if (tid == 0) mbar_expect_tx(&S.rv.bp[par], primal_bytes);
    if (DIAG) {
      double pmax = 0.0, qmax = 0.0;
      if (inner) {
        pmax = sqrt(p0 * p0 + p1 * p1);
        qmax = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
      }
      pmax = warp_max(pmax);
      qmax = warp_max(qmax);
      if (lane == 0 && A.diag_p) {
        atomic_max_nonneg(A.diag_p + it, (float)pmax);
        atomic_max_nonneg(A.diag_q + it, (float)qmax);
      }
    }
    __syncthreads();
    // backward divergence (rasters.py:158-172)
    double lx0 = shfl_up(fx0), lx1 = shfl_up(fx1), lx2 = shfl_up(fx2);
    double uy0 = 0.0, uy1 = 0.0, uy2 = 0.0;
    if (ty > 0) {
      uy0 = X.fy[0][ty - 1][lane]; uy1 = X.fy[1][ty - 1][lane]; uy2 = X.fy[2][ty - 1][lane];
    }
    if (has_l || (ty == 0 && has_u)) {
      mbar_wait(&S.rv.bp[par], ph);
      if (lane == 0 && has_l) {
        lx0 = S.rv.lf[par][0][ty]; lx1 = S.rv.lf[par][1][ty]; lx2 = S.rv.lf[par][2][ty];
      }
      if (ty == 0 && has_u) {
        uy0 = S.rv.up[par][0][lane]; uy1 = S.rv.up[par][1][lane]; uy2 = S.rv.up[par][2][lane];
      }
    }
    const double dvv = ((fx0 - lx0) + fy0) - uy0;
    const double d0 = ((fx1 - lx1) + fy1) - uy1;
    const double d1 = ((fx2 - lx2) + fy2) - uy2;
    const double tu = S.cs[CTU][s], tv = S.cs[CTV][s], g = S.cs[CIU][s];
    const double rh = S.cs[CRH][s], uo = S.cs[CUO][s];
    primal_update_exact<double>(dvv, d0, d1, tu, tv, g, rh, uo, p0, p1, lam, alpha0, alpha1,
                                theta, u, v0, v1, ub, vb0, vb1);
  }

  const bool st = inner && m;
  const size_t n = A.n;
  const uint32_t i = st ? (uint32_t)gy * (uint32_t)W + (uint32_t)gx : 0u;
  const double uo = S.cs[CUO][s];
  double adu = 0.0, amax = 0.0;
  if (fin && st) {  // clip / accumulate (solver.py:356-360) on the interior
    const double du = fmin(fmax(u - uo, -A.du_max), A.du_max);
    u = uo + du;
    amax = fabs(du);
    const double2 dd = reinterpret_cast<const double2*>(A.dirs)[i];
    double2 wv = reinterpret_cast<double2*>(A.wv)[i];
    wv.x = wv.x + du * dd.x;
    wv.y = wv.y + du * dd.y;
    reinterpret_cast<double2*>(A.wv)[i] = wv;
    adu = fabs(du);
  }
  if (st) {
    if (first) A.uo[i] = uo;
    A.du[i] = u;
    A.dv[i] = v0; (A.dv + n)[i] = v1;
    A.dp[i] = p0; (A.dp + n)[i] = p1;
    A.dq[i] = q0; (A.dq + n)[i] = q1; (A.dq + 2 * n)[i] = q2; (A.dq + 3 * n)[i] = q3;
    if (!fin) {  // u_bar / v_bar are reset at the next warp's start: dead after its last cycle
      A.dub[i] = ub;
      A.dvb[i] = vb0; (A.dvb + n)[i] = vb1;
    }
  }
  if (DIAG && fin && (A.diag_du || A.diag_du64)) {
    const double mx = warp_max(amax), sm = warp_sum(adu);
    if (lane == 0) { S.red_sum[ty] = sm; S.red_max[ty] = mx; }
    __syncthreads();
    if (tid == 0) {
      double tsum = 0.0, mm = 0.0;
      for (int j = 0; j < kH; ++j) { tsum += S.red_sum[j]; mm = fmax(mm, S.red_max[j]); }
      A.partials[(size_t)r * NC + rank] = tsum;
      if (A.diag_du64) atomic_max_nonneg(A.diag_du64, mm);
      else atomic_max_nonneg(A.diag_du, (float)mm);
    }
  }
}

struct CtileCfg {
  int R, CX, CY, TH;
};

// FSB_CTILE="R,CX,CY[,TH]" (tuning): halo / cycles per launch, cluster shape,
// rows per CTA
CtileCfg ctile_cfg() {
  static const CtileCfg c = [] {
    CtileCfg d{5, 2, 8, 8};  // 2 x 8 CTAs of 32 x 8: 64 x 64 regions, 4 CTAs per SM
    const char* e = getenv("FSB_CTILE");
    if (e) {
      CtileCfg t{0, 0, 0, 16};
      const int k = sscanf(e, "%d,%d,%d,%d", &t.R, &t.CX, &t.CY, &t.TH);
      auto is = [&](int r, int cx, int cy, int th) {
        return t.R == r && t.CX == cx && t.CY == cy && t.TH == th;
      };
      if (k >= 3 && (is(5, 2, 4, 16) || is(5, 4, 4, 16) || is(10, 4, 4, 16) || is(4, 2, 4, 16) ||
                     is(5, 2, 8, 16) || is(5, 4, 2, 16) || is(5, 2, 8, 8) || is(5, 2, 4, 8) ||
                     is(5, 4, 4, 8) || is(5, 2, 8, 4)))
        d = t;
    }
    return d;
  }();
  return c;
}

template <int R, int CX, int CY, int TH, bool DIAG>
int launch_ctile(const B64& A, const Ctile64Maps& M, int src, cudaStream_t st) {
  constexpr int NC = CX * CY, IW = CX * kW - 2 * R, IH = CY * TH - 2 * R;
  const int nrx = (A.w + IW - 1) / IW, nry = (A.h + IH - 1) / IH;
  auto kern = k64_ctile<R, CX, CY, TH, DIAG>;
  constexpr size_t smem = smem_bytes<TH>();
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [&] {
    if (NC > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)(nrx * nry * NC));
  cfg.blockDim = dim3(kW, TH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = NC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const CUtensorMap& ld = M.ld[src][A.first ? 1 : 0];
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, A, ld, M.cst, nrx);
  if (e != cudaSuccess) return (int)e;
  return launch_status();
}

template <int R, int CX, int CY, int TH>
int launch_ctile_d(const B64& A, const Ctile64Maps& M, int src, cudaStream_t st) {
  const bool diag = A.diag_p || A.diag_du || A.diag_du64;
  return diag ? launch_ctile<R, CX, CY, TH, true>(A, M, src, st)
              : launch_ctile<R, CX, CY, TH, false>(A, M, src, st);
}

}  // namespace

int pd64_ctile_halo() { return ctile_cfg().R; }

bool pd64_ctile_usable(int w, int h) {
  const CtileCfg c = ctile_cfg();
  return w % 2 == 0 && w >= kBW && h >= c.TH && w >= c.CX * kW && h >= c.CY * c.TH &&
         tma_encoder() != nullptr;
}

bool pd64_ctile_maps(Ctile64Maps* M, const double* set0, const double* set1, const double* cst,
                     int w, int h) {
  if (!pd64_ctile_usable(w, h)) return false;
  const CtileCfg c = ctile_cfg();
  if (((uintptr_t)set0 | (uintptr_t)set1 | (uintptr_t)cst) & 15) return false;
  const double* sets[2] = {set0, set1};
  for (int k = 0; k < 2; ++k)
    if (!make_map64(&M->ld[k][0], sets[k], w, h, kSt, kBW, c.TH, kSt) ||
        !make_map64(&M->ld[k][1], sets[k], w, h, kSt, kBW, c.TH, kSt0))
      return false;
  return make_map64(&M->cst, cst, w, h, kCst, kBW, c.TH, kCst);
}

size_t pd64_ctile_partials(int w, int h) {
  const CtileCfg c = ctile_cfg();
  const int IW = c.CX * kW - 2 * c.R, IH = c.CY * c.TH - 2 * c.R;
  return (size_t)((w + IW - 1) / IW) * ((h + IH - 1) / IH) * c.CX * c.CY;
}

int pd64_ctile_list(const uint8_t* mask, int w, int h, int* tiles, cudaStream_t st) {
  const CtileCfg c = ctile_cfg();
  return tile_list_internal(mask, w, h, c.CX * kW - 2 * c.R, c.CY * c.TH - 2 * c.R, tiles, st);
}

int pd64_ctile_launch(const B64& A, const Ctile64Maps& M, int src_set, cudaStream_t st) {
  const CtileCfg c = ctile_cfg();
  if (A.iters < 1 || A.iters > c.R || !A.tiles || (src_set & ~1)) return FSB_EINVAL;
  if (c.TH == 4) return launch_ctile_d<5, 2, 8, 4>(A, M, src_set, st);
  if (c.TH == 8) {
    if (c.CX == 4) return launch_ctile_d<5, 4, 4, 8>(A, M, src_set, st);
    if (c.CY == 8) return launch_ctile_d<5, 2, 8, 8>(A, M, src_set, st);
    return launch_ctile_d<5, 2, 4, 8>(A, M, src_set, st);
  }
  if (c.R == 5 && c.CX == 4 && c.CY == 4) return launch_ctile_d<5, 4, 4, 16>(A, M, src_set, st);
  if (c.R == 5 && c.CX == 4 && c.CY == 2) return launch_ctile_d<5, 4, 2, 16>(A, M, src_set, st);
  if (c.R == 5 && c.CY == 8) return launch_ctile_d<5, 2, 8, 16>(A, M, src_set, st);
  if (c.R == 10) return launch_ctile_d<10, 4, 4, 16>(A, M, src_set, st);
  if (c.R == 4) return launch_ctile_d<4, 2, 4, 16>(A, M, src_set, st);
  return launch_ctile_d<5, 2, 4, 16>(A, M, src_set, st);
}

}  // namespace fsb
