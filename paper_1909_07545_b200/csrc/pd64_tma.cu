// k64_tma: k64_tile fed and drained by TMA (FSB_PD64K=tma; not the default).
//
// Same cycle, tile shape (32 x 16, halo 2, one pixel per thread, x-neighbours
// by shuffle, y-neighbours through shared memory, 2 barriers per cycle) and
// arithmetic as k64_tile (pd64_tile.cu). The memory side differs: two CTAs per
// SM walk the level's work list (phase-staggered as in k64_tile); one thread
// loads a tile as two 3-D TMA boxes — the 12 (first launch of a warp: 9) state
// planes and the 10 constant planes (edge codes included), zero outside the
// image — under an mbarrier; the state moves into registers and the state box
// then serves as the y-exchange buffers and, after the cycles, as the interior
// box of one TMA store (12 planes; the warp's last launch 9). Pixels outside
// the solve mask store 0 (their state is 0 in both sets).
//
// Measured on the C3 1024^2 level: 57 us per 2-cycle launch, the same as
// k64_tile (and a one-CTA-per-SM variant prefetching the next tile: 61 us).
// 20% fewer instructions, but the launch stays bound by the ~190 MB it moves,
// which k64_ctile (pd64_ctile.cu) cuts by running 5 cycles per launch.
//
// Reference: solver.py:279-303 (primal_dual_iterate), 344-360 (warp-start
// reset, clip / accumulate epilogue), rasters.py:144-182.

#include <stdlib.h>

#include "pd64_block.cuh"
#include "pd_math.cuh"
#include "tma.cuh"

namespace fsb {

EncodeTiled tma_encoder() {
  // resolved once; a function-local static is initialised thread-safely
  static const EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiled>(p);
    return static_cast<EncodeTiled>(nullptr);
  }();
  return fn;
}

// planes x h x w float64 block (plane stride h*w) with a bw x bh x bp box
bool make_map64(CUtensorMap* m, const double* base, int w, int h, int planes, int bw, int bh,
                int bp) {
  EncodeTiled enc = tma_encoder();
  if (!enc) return false;
  const size_t n = (size_t)w * h;
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)w * sizeof(double), (cuuint64_t)n * sizeof(double)};
  cuuint32_t boxd[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bp};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
             boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int tile_list_internal(const uint8_t* mask, int w, int h, int TW, int TH, int* tiles,
                       cudaStream_t st);

namespace {

constexpr int kR = 2, kW = 32, kH = 16, kOW = kW - 2 * kR, kOH = kH - 2 * kR;
constexpr int kPl = kW * kH;     // doubles per plane of the load box
constexpr int kOPl = kOW * kOH;  // doubles per plane of the store box
constexpr int kSt = 12, kSt0 = 9, kCst = 10;

// state plane order inside a set / the boxes
enum { PU, PV0, PV1, PP0, PP1, PQ0, PQ1, PQ2, PQ3, PUB, PVB0, PVB1 };
// constant planes
enum { CA, CB, CC, CSP, CTU, CTV, CIU, CRH, CUO, CCODE };

// The state box is dead once the tile is in registers: it then holds the
// y-exchange buffers during the cycles and the interior (store) box after them.
struct Xch {
  double ub[kH][kW], vb0[kH][kW], vb1[kH][kW];  // y-exchange of the dual step
  double fy[3][kH][kW];                         // y-exchange of the primal step
};
struct Smem64T {
  double st[kSt][kPl];   // state box (TMA load) | Xch | interior box [12][kOH][kOW] (TMA store)
  double cs[kCst][kPl];  // constant box (TMA load), read through the cycles
  double red_sum[kH], red_max[kH];
  uint64_t bar;
};
static_assert(sizeof(Xch) <= sizeof(double) * kSt * kPl && kSt * kOPl <= kSt * kPl,
              "exchange and store boxes alias the state box");
static_assert(sizeof(double) * kSt * kPl % 128 == 0, "TMA boxes must stay 128-byte aligned");
constexpr size_t kSmemBytes = sizeof(Smem64T) + 128;

FSB_INLINE double shfl_dn(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
FSB_INLINE double shfl_up(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }

template <bool DIAG>
__global__ void __launch_bounds__(kW * kH, 2)
    k64_tma(const B64 A, const __grid_constant__ CUtensorMap m_ld,
            const __grid_constant__ CUtensorMap m_cst, const __grid_constant__ CUtensorMap m_st,
            int ntx) {
  extern __shared__ unsigned char smem_raw[];
  poison_dynamic_smem(smem_raw);  // checked build only (before the mbarrier lives there)
  // 128-B aligned base, formed as an offset from the shared array (keeps LDS / STS)
  Smem64T& S = *reinterpret_cast<Smem64T*>(smem_raw +
                                           ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
  Xch& X = *reinterpret_cast<Xch*>(&S.st[0][0]);
  double* out = &S.st[0][0];
  const int lane = threadIdx.x, ty = threadIdx.y, s = ty * kW + lane;
  const bool first = A.first, fin = A.fin;
  const uint32_t tx_bytes = (uint32_t)(((first ? kSt0 : kSt) + kCst) * kPl * sizeof(double));
  const int cnt = A.tiles[0];
  if (s == 0) {
    mbar_init(&S.bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  // Persistent: 2 CTAs per SM stride over the work list; with A.persist the
  // second half starts that many ns late so an SM's two CTAs keep opposite
  // phases (one loading while the other cycles), as in k64_tile.
  if (A.persist && blockIdx.x >= gridDim.x / 2) __nanosleep((unsigned)A.persist);

  const int W = A.w, H = A.h;
  const double alpha1 = A.alpha1, sq = A.sigma_q * A.alpha0, heps = A.heps;
  const double lam = A.lam, alpha0 = A.alpha0, theta = A.theta;
  const int tyd = ty + 1 < kH ? ty + 1 : ty;
  const bool box = lane >= kR && lane < kW - kR && ty >= kR && ty < kH - kR;
  uint32_t parity = 0;
  for (int k = blockIdx.x; k < cnt; k += gridDim.x) {
    const int t = A.tiles[1 + k];
    const int bx = t % ntx, by = t / ntx;
    if (s == 0) {  // one thread loads the tile (after the last store has read its box out)
      bulk_wait_read0();
      fence_proxy_async();
      mbar_expect_tx(&S.bar, tx_bytes);
      tma_load_3d(&S.st[0][0], &m_ld, bx * kOW - kR, by * kOH - kR, 0, &S.bar);
      tma_load_3d(&S.cs[0][0], &m_cst, bx * kOW - kR, by * kOH - kR, 0, &S.bar);
    }
    const int gx = bx * kOW - kR + lane, gy = by * kOH - kR + ty;
    const bool in = (unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H;
    const bool inner = box && in;
    mbar_wait(&S.bar, parity);
    parity ^= 1;
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
      X.ub[ty][lane] = ub;
      X.vb0[ty][lane] = vb0;
      X.vb1[ty][lane] = vb1;
      __syncthreads();
      const double a = S.cs[CA][s], b = S.cs[CB][s], c = S.cs[CC][s];
      // forward differences (rasters.py:144-155), zero where the edge leaves the mask
      const double ubx = shfl_dn(ub), vbx0 = shfl_dn(vb0), vbx1 = shfl_dn(vb1);
      const double uby = X.ub[tyd][lane], vby0 = X.vb0[tyd][lane], vby1 = X.vb1[tyd][lane];
      const double gxx = ex ? ubx - ub : 0.0, gyy = ey ? uby - ub : 0.0;
      const double g00 = ex ? vbx0 - vb0 : 0.0, g01 = ey ? vby0 - vb0 : 0.0;
      const double g10 = ex ? vbx1 - vb1 : 0.0, g11 = ey ? vby1 - vb1 : 0.0;
      dual_update_exact<double>(a, b, c, sp, sq, gxx, gyy, g00, g01, g10, g11, vb0, vb1, p0, p1,
                                q0, q1, q2, q3, heps);
      const double fx0 = ex ? a * p0 + b * p1 : 0.0;
      const double fy0 = ey ? b * p0 + c * p1 : 0.0;
      const double fx1 = ex ? q0 : 0.0, fy1 = ey ? q1 : 0.0;
      const double fx2 = ex ? q2 : 0.0, fy2 = ey ? q3 : 0.0;
      X.fy[0][ty][lane] = fy0;
      X.fy[1][ty][lane] = fy1;
      X.fy[2][ty][lane] = fy2;
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
      // backward divergence (rasters.py:158-172); the column left of / row above
      // the tile feed only halo pixels
      const double lx0 = shfl_up(fx0), lx1 = shfl_up(fx1), lx2 = shfl_up(fx2);
      double uy0 = 0.0, uy1 = 0.0, uy2 = 0.0;
      if (ty > 0) {
        uy0 = X.fy[0][ty - 1][lane]; uy1 = X.fy[1][ty - 1][lane]; uy2 = X.fy[2][ty - 1][lane];
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
    if (first && st) A.uo[i] = uo;
    if (DIAG && fin && (A.diag_du || A.diag_du64)) {
      const double mx = warp_max(amax), sm = warp_sum(adu);
      if (lane == 0) { S.red_sum[ty] = sm; S.red_max[ty] = mx; }
      __syncthreads();
      if (s == 0) {
        double tsum = 0.0, mm = 0.0;
        for (int r = 0; r < kH; ++r) { tsum += S.red_sum[r]; mm = fmax(mm, S.red_max[r]); }
        A.partials[t] = tsum;
        if (A.diag_du64) atomic_max_nonneg(A.diag_du64, mm);
        else atomic_max_nonneg(A.diag_du, (float)mm);
      }
    }
    __syncthreads();  // the exchange buffers are read: the interior box takes their place
    if (box) {
      double* o = out + (ty - kR) * kOW + (lane - kR);
      o[PU * kOPl] = m ? u : 0.0;
      o[PV0 * kOPl] = m ? v0 : 0.0; o[PV1 * kOPl] = m ? v1 : 0.0;
      o[PP0 * kOPl] = m ? p0 : 0.0; o[PP1 * kOPl] = m ? p1 : 0.0;
      o[PQ0 * kOPl] = m ? q0 : 0.0; o[PQ1 * kOPl] = m ? q1 : 0.0;
      o[PQ2 * kOPl] = m ? q2 : 0.0; o[PQ3 * kOPl] = m ? q3 : 0.0;
      if (!fin) {  // u_bar / v_bar are reset at the next warp's start: dead after its last cycle
        o[PUB * kOPl] = m ? ub : 0.0;
        o[PVB0 * kOPl] = m ? vb0 : 0.0; o[PVB1 * kOPl] = m ? vb1 : 0.0;
      }
    }
    fence_proxy_async();
    __syncthreads();  // the interior box is complete; the constant box is no longer read
    if (s == 0) {
      tma_store_3d(&m_st, out, bx * kOW, by * kOH, 0);
      bulk_commit();
    }
  }
  if (s == 0) bulk_wait0();
}

int num_sms64() {
  static const int v = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return v;
}

template <bool DIAG>
int launch64_tma(const B64& A, const CUtensorMap& ld, const CUtensorMap& cst,
                 const CUtensorMap& stm, cudaStream_t st) {
  const int ntx = (A.w + kOW - 1) / kOW;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k64_tma<DIAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
  });
  k64_tma<DIAG><<<2 * num_sms64(), dim3(kW, kH), kSmemBytes, st>>>(A, ld, cst, stm, ntx);
  return launch_status();
}

}  // namespace

bool pd64_tma_usable(int w, int h) {
  // row pitch and plane stride 16-B multiples with 16-B aligned box starts for
  // every plane (w % 4 == 0 also keeps x0 = 28 bx - 2 at an even column)
  return w % 4 == 0 && h >= kH && w >= kW && tma_encoder() != nullptr;
}

bool pd64_tma_level_maps(Tma64Level* M, const double* set0, const double* set1,
                         const double* cst, int w, int h) {
  if (!pd64_tma_usable(w, h)) return false;
  if (((uintptr_t)set0 | (uintptr_t)set1 | (uintptr_t)cst) & 15) return false;
  const double* sets[2] = {set0, set1};
  for (int k = 0; k < 2; ++k) {
    if (!make_map64(&M->ld[k][0], sets[k], w, h, kSt, kW, kH, kSt) ||
        !make_map64(&M->ld[k][1], sets[k], w, h, kSt, kW, kH, kSt0) ||
        !make_map64(&M->st[k][0], sets[k], w, h, kSt, kOW, kOH, kSt) ||
        !make_map64(&M->st[k][1], sets[k], w, h, kSt, kOW, kOH, kSt0))
      return false;
  }
  return make_map64(&M->cst, cst, w, h, kCst, kW, kH, kCst);
}

size_t pd64_tma_tile_count(int w, int h) {
  return (size_t)((w + kOW - 1) / kOW) * ((h + kOH - 1) / kOH);
}

int pd64_tma_tile_list(const uint8_t* mask, int w, int h, int* tiles, cudaStream_t st) {
  return tile_list_internal(mask, w, h, kOW, kOH, tiles, st);
}

int pd64_tma_launch(const B64& A, const Tma64Level& M, int src_set, cudaStream_t st) {
  if (A.iters < 1 || A.iters > kR || !A.tiles || (src_set & ~1)) return FSB_EINVAL;
  const CUtensorMap& ld = M.ld[src_set][A.first ? 1 : 0];
  const CUtensorMap& stm = M.st[src_set ^ 1][A.fin ? 1 : 0];
  const bool diag = A.diag_p || A.diag_du || A.diag_du64;
  return diag ? launch64_tma<true>(A, ld, M.cst, stm, st)
              : launch64_tma<false>(A, ld, M.cst, stm, st);
}

}  // namespace fsb
