// Whole-level solve for small pyramid levels on ONE thread-block cluster.
//
// Coarse levels (<= 16 rows per CTA x 16 CTAs, <= 32 warps per CTA) hold too
// few pixels to fill the GPU, so launch latency and per-tile halo work
// dominated their warp loops (three launches per warp). Here the entire
// solve_level warp loop (solver.py:331-365) — samples at x + w, I_u, K
// primal-dual cycles, clip / accumulate — runs in a single launch of a
// cluster of up to 16 CTAs. Each CTA owns a band of rows held in registers
// (one pixel pair per lane, packed fp32x2 math as in pd_tma.cu); neighbour
// rows of other CTAs are read from their shared memory through DSMEM, and a
// cluster barrier (release / acquire) separates the dual and primal halves of
// every cycle. No halo is recomputed and no state leaves the chip until the
// level ends.
//
// Arithmetic is identical to the pair / TMA kernels (same helpers, same
// order), so results agree with them to round-off.

#include <cooperative_groups.h>
#include <stdlib.h>
#include <string.h>

#include "pd_math.cuh"
#include "warp_math.cuh"

namespace cg = cooperative_groups;

namespace fsb {

struct ClusterArgs {
  int h, w, rpc, wr;  // level size, rows per CTA, warps per row
  size_t n;
  const uint8_t* mask;
  const float* T; const float* S;  // tensor a,b,c / steps sigma_p, tau_u, tau_v planes
  const float* i0;
  float* u; float* wv;             // in: initial WarpState; out: result
  float* v; float* p; float* q;   // out: final v (2), p (2), q (4) planes
  float* ub; float* vb;            // out: u_bar (= u after the clip), v_bar (2)
  float* i1w; uint8_t* i1w_ok;     // scratch planes (global, cluster-visible)
  SampleSrc src;                   // i1 / traj gather tables of the level
  float lam, alpha0, alpha1, theta, sigma_q, du_max;
  float huber_eps;  // > 0: Huber-TV dual step
  int N, K;
  float* diag_p; float* diag_q; float* diag_du; double* diag_mean;  // nullptr = off
};

namespace {

typedef float2 f2;
FSB_INLINE f2 mk2(float a, float b) { return make_float2(a, b); }
FSB_INLINE f2 add2(f2 a, f2 b) { return __fadd2_rn(a, b); }
FSB_INLINE f2 sub2(f2 a, f2 b) { return __fadd2_rn(a, mk2(-b.x, -b.y)); }
FSB_INLINE f2 mul2(f2 a, f2 b) { return __fmul2_rn(a, b); }
FSB_INLINE f2 fma2(f2 a, f2 b, f2 c) { return __ffma2_rn(a, b, c); }
FSB_INLINE f2 unit_scale2(f2 n2) {
  return mk2(n2.x > 1.f ? rsqrtf(n2.x) : 1.f, n2.y > 1.f ? rsqrtf(n2.y) : 1.f);
}
FSB_INLINE float shrink1(float uh, float rh, float g, float tl) {
  const float a = tl * g;
  const float th = a * g;
  const float q = g != 0.f ? __fdividef(rh, g) : 0.f;
  const float step = rh < -th ? a : (rh > th ? -a : -q);
  return g != 0.f ? uh + step : uh;
}

FSB_INLINE void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

constexpr int kMaxRows = 16, kMaxCols = 192;  // per CTA band: rows x padded columns
constexpr int kPlanes = 9;                     // ub vb0 vb1 | px py q0x q0y q1x q1y
constexpr int kMaxWarps = 64;                  // warp iterations with the in-kernel mean

// MAXT: block size bound. Bands of <= 256 threads (64^2 levels) get up to
// 255 registers instead of 128 (no spills in the sampling part).
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_level_cluster(const ClusterArgs A) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank(), ncta = (int)cluster.num_blocks();
  extern __shared__ float s_dyn[];  // kPlanes planes of rpc rows x (ncols + 2) columns
  __shared__ double s_red[32];
  __shared__ float s_redm[32];
  __shared__ double s_psum[kMaxWarps];  // this CTA's sum |du| per warp iteration
  __shared__ unsigned s_cnt;            // this CTA's mask pixels
  poison_dynamic_smem(s_dyn);           // checked build only (before any DSMEM reader)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rl = warp / A.wr;                    // row within the band
  const int c0 = (warp % A.wr) * 64 + 2 * lane;  // first column of this pair
  const int y = rank * A.rpc + rl;
  const bool row_ok = rl < A.rpc && y < A.h;
  const int W = A.w, H = A.h;
  const size_t n = A.n;
  const int ncols = A.wr * 64;
  const int RS = ncols + 2;        // row stride (+2: zero pad columns)
  const int PS = A.rpc * RS;       // plane stride
#define SP(pl, r, c) s_dyn[(pl) * PS + (r) * RS + (c)]

  // zero the pad columns once (column ncols and ncols + 1)
  for (int k = threadIdx.x; k < kPlanes * A.rpc; k += blockDim.x) {
    SP(k / A.rpc, k % A.rpc, ncols) = 0.f;
    SP(k / A.rpc, k % A.rpc, ncols + 1) = 0.f;
  }

  // ---- per-pixel constants and state of this pair
  float m[2], ex[2], ey[2];
  float u[2], wx[2], wy[2];
  float ta[2], tb[2], tc[2], sp[2], tu[2], tv[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int x = c0 + e;
    const bool in = row_ok && x < W;
    const size_t i = in ? (size_t)y * W + x : 0;
    const bool mk = in && A.mask[i];
    m[e] = mk ? 1.f : 0.f;
    ex[e] = (mk && x + 1 < W && A.mask[i + 1]) ? 1.f : 0.f;
    ey[e] = (mk && y + 1 < H && A.mask[i + W]) ? 1.f : 0.f;
    u[e] = in ? A.u[i] : 0.f;
    wx[e] = in ? A.wv[2 * i] : 0.f;
    wy[e] = in ? A.wv[2 * i + 1] : 0.f;
    ta[e] = in ? A.T[i] : 1.f; tb[e] = in ? A.T[n + i] : 0.f; tc[e] = in ? A.T[2 * n + i] : 1.f;
    sp[e] = in ? A.S[i] * A.alpha1 : 0.f;
    tu[e] = in ? A.S[n + i] : 0.f;
    tv[e] = in ? A.S[2 * n + i] : 0.f;
  }
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  {
    const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)(m[0] + m[1]));
    if (lane == 0 && c) atomicAdd(&s_cnt, c);
  }
  const f2 exf = mk2(ex[0], ex[1]), eyf = mk2(ey[0], ey[1]);
  const f2 ta2 = mk2(ta[0], ta[1]), tb2 = mk2(tb[0], tb[1]), tc2 = mk2(tc[0], tc[1]);
  const f2 sp2 = mk2(sp[0], sp[1]), tu2 = mk2(tu[0], tu[1]), tv2 = mk2(tv[0], tv[1]);
  const f2 sq2 = mk2(A.sigma_q * A.alpha0, A.sigma_q * A.alpha0);
  const f2 al0 = mk2(A.alpha0, A.alpha0), al1 = mk2(A.alpha1, A.alpha1);
  const f2 th2 = mk2(A.theta, A.theta), lam2 = mk2(A.lam, A.lam);
  // v, p, q start at zero (solver.py:323-327)
  f2 U = mk2(u[0], u[1]), V0 = mk2(0.f, 0.f), V1 = V0, P0 = V0, P1 = V0;
  f2 Q0 = V0, Q1 = V0, Q2 = V0, Q3 = V0;
  f2 UB = U, VB0 = V0, VB1 = V1;
  cluster_sync_all();

  // DSMEM views of the neighbour CTAs' planes (rows above / below the band)
  const float* s_up = rank > 0 ? cluster.map_shared_rank(s_dyn, rank - 1) : nullptr;
  const float* s_dn = rank + 1 < ncta ? cluster.map_shared_rank(s_dyn, rank + 1) : nullptr;

  for (int wi = 0; wi < A.N; ++wi) {
    // ---- samples at x + w (solver.py:332-337)
    float iw[2], dx[2], dy[2];
    bool iok[2], dok[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int x = c0 + e;
      iw[e] = dx[e] = dy[e] = 0.f;
      iok[e] = dok[e] = false;
      if (row_ok && x < W && m[e] != 0.f) {
        float2 d;
        bool a, b;
        warp_sample_nan_bits(A.src.packed, H, W, x, y, make_float2(wx[e], wy[e]), iw[e], a, d, b);
        iok[e] = a; dok[e] = b; dx[e] = d.x; dy[e] = d.y;
      }
      if (row_ok && x < W)  // NaN where invalid: the I_u gather reads validity from the value
        A.i1w[(size_t)y * W + x] = iok[e] ? iw[e] : __int_as_float(0x7fc00000);
    }
    cluster_sync_all();  // i1w of the whole level visible (release / acquire)
    // ---- I_u and rho0 (solver.py:339-343, image_derivative_along 192-202)
    float g[2], rh[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int x = c0 + e;
      g[e] = rh[e] = 0.f;
      if (iok[e] && dok[e]) {
        int ix, iy;
        float fx, fy, ahead[1];
        if (split_off(x, y, dx[e], dy[e], H, W, ix, iy, fx, fy)) {
          // plain (coherent) loads: other CTAs wrote i1w in this kernel
          float t[16];
          unsigned okb = 0;
          const bool inner = ix >= 1 && ix + 2 < W && iy >= 1 && iy + 2 < H;
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int r = iy + a - 1, c = ix + b - 1;
              const bool in = inner || ((unsigned)r < (unsigned)H && (unsigned)c < (unsigned)W);
              const float v = in ? A.i1w[(size_t)r * W + c] : __int_as_float(0x7fc00000);
              t[4 * a + b] = v;
              okb |= (isnan(v) ? 0u : 1u) << (4 * a + b);
            }
          if (bicubic_regs(t, okb, fx, fy, ahead[0])) {
            g[e] = ahead[0] - iw[e];
            rh[e] = iw[e] - A.i0[(size_t)y * W + x];
          }
        }
      }
    }
    const f2 G = mk2(g[0], g[1]), RH = mk2(rh[0], rh[1]);
    const f2 UO = U;  // u_omega = u; u_bar = u; v_bar = v (solver.py:344-346)
    UB = U; VB0 = V0; VB1 = V1;

    for (int it = 0; it < A.K; ++it) {
      // publish u_bar / v_bar
      if (row_ok) {
        *reinterpret_cast<f2*>(&SP(0, rl, c0)) = UB;
        *reinterpret_cast<f2*>(&SP(1, rl, c0)) = VB0;
        *reinterpret_cast<f2*>(&SP(2, rl, c0)) = VB1;
      }
      cluster_sync_all();
      float pmax = 0.f, qmax = 0.f;
      if (row_ok) {
        // right neighbour: own .y / next pair's .x (column c0 + 2, pad past the band)
        const f2 R0 = mk2(UB.y, SP(0, rl, c0 + 2));
        const f2 R1 = mk2(VB0.y, SP(1, rl, c0 + 2));
        const f2 R2 = mk2(VB1.y, SP(2, rl, c0 + 2));
        f2 D0, D1, D2;  // down neighbour
        if (y + 1 >= H) {
          D0 = D1 = D2 = mk2(0.f, 0.f);  // no row below (rows past H were never written)
        } else if (rl + 1 < A.rpc) {
          D0 = *reinterpret_cast<const f2*>(&SP(0, rl + 1, c0));
          D1 = *reinterpret_cast<const f2*>(&SP(1, rl + 1, c0));
          D2 = *reinterpret_cast<const f2*>(&SP(2, rl + 1, c0));
        } else if (s_dn) {
          D0 = *reinterpret_cast<const f2*>(&s_dn[(0) * PS + (0) * RS + (c0)]);
          D1 = *reinterpret_cast<const f2*>(&s_dn[(1) * PS + (0) * RS + (c0)]);
          D2 = *reinterpret_cast<const f2*>(&s_dn[(2) * PS + (0) * RS + (c0)]);
        } else {
          D0 = D1 = D2 = mk2(0.f, 0.f);
        }
        const f2 gx = mul2(exf, sub2(R0, UB)), gy = mul2(eyf, sub2(D0, UB));
        const f2 g00 = mul2(exf, sub2(R1, VB0)), g01 = mul2(eyf, sub2(D1, VB0));
        const f2 g10 = mul2(exf, sub2(R2, VB1)), g11 = mul2(eyf, sub2(D2, VB1));
        const f2 t0 = sub2(fma2(ta2, gx, mul2(tb2, gy)), VB0);
        const f2 t1 = sub2(fma2(tb2, gx, mul2(tc2, gy)), VB1);
        f2 pp0 = fma2(sp2, t0, P0), pp1 = fma2(sp2, t1, P1);
        if (A.huber_eps > 0.f) {  // Huber-TV: p / (1 + sp eps) before the projection
          const f2 kk = mk2(__frcp_rn(fmaf(sp2.x, A.huber_eps, 1.f)),
                            __frcp_rn(fmaf(sp2.y, A.huber_eps, 1.f)));
          pp0 = mul2(pp0, kk);
          pp1 = mul2(pp1, kk);
        }
        const f2 rp = unit_scale2(fma2(pp0, pp0, mul2(pp1, pp1)));
        P0 = mul2(pp0, rp);
        P1 = mul2(pp1, rp);
        const f2 qq0 = fma2(sq2, g00, Q0), qq1 = fma2(sq2, g01, Q1);
        const f2 qq2 = fma2(sq2, g10, Q2), qq3 = fma2(sq2, g11, Q3);
        const f2 rq = unit_scale2(add2(fma2(qq0, qq0, mul2(qq1, qq1)),
                                       fma2(qq2, qq2, mul2(qq3, qq3))));
        Q0 = mul2(qq0, rq); Q1 = mul2(qq1, rq); Q2 = mul2(qq2, rq); Q3 = mul2(qq3, rq);
        *reinterpret_cast<f2*>(&SP(3, rl, c0)) = mul2(exf, fma2(ta2, P0, mul2(tb2, P1)));
        *reinterpret_cast<f2*>(&SP(4, rl, c0)) = mul2(eyf, fma2(tb2, P0, mul2(tc2, P1)));
        *reinterpret_cast<f2*>(&SP(5, rl, c0)) = mul2(exf, Q0);
        *reinterpret_cast<f2*>(&SP(6, rl, c0)) = mul2(eyf, Q1);
        *reinterpret_cast<f2*>(&SP(7, rl, c0)) = mul2(exf, Q2);
        *reinterpret_cast<f2*>(&SP(8, rl, c0)) = mul2(eyf, Q3);
        if (A.diag_p) {
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (c0 + e < W) {
              const float a = e ? P0.y : P0.x, b = e ? P1.y : P1.x;
              const float c = e ? Q0.y : Q0.x, d = e ? Q1.y : Q1.x;
              const float f = e ? Q2.y : Q2.x, gg = e ? Q3.y : Q3.x;
              pmax = fmaxf(pmax, sqrtf(a * a + b * b));
              qmax = fmaxf(qmax, sqrtf((c * c + d * d) + (f * f + gg * gg)));
            }
        }
      }
      if (A.diag_p) {
        pmax = warp_max(pmax);
        qmax = warp_max(qmax);
        if (lane == 0) {
          atomic_max_nonneg(A.diag_p + wi * A.K + it, pmax);
          atomic_max_nonneg(A.diag_q + wi * A.K + it, qmax);
        }
      }
      cluster_sync_all();
      if (row_ok) {
        // left neighbour: previous pair's .y (column c0 - 1; column -1 reads as 0)
        const float lx = c0 > 0 ? SP(3, rl, c0 - 1) : 0.f;
        const float l0 = c0 > 0 ? SP(5, rl, c0 - 1) : 0.f;
        const float l1 = c0 > 0 ? SP(7, rl, c0 - 1) : 0.f;
        const f2 FX = *reinterpret_cast<const f2*>(&SP(3, rl, c0));
        const f2 FY = *reinterpret_cast<const f2*>(&SP(4, rl, c0));
        const f2 F0X = *reinterpret_cast<const f2*>(&SP(5, rl, c0));
        const f2 F0Y = *reinterpret_cast<const f2*>(&SP(6, rl, c0));
        const f2 F1X = *reinterpret_cast<const f2*>(&SP(7, rl, c0));
        const f2 F1Y = *reinterpret_cast<const f2*>(&SP(8, rl, c0));
        f2 UPY, UQ0, UQ1;  // up neighbour's y-fluxes
        if (rl > 0) {
          UPY = *reinterpret_cast<const f2*>(&SP(4, rl - 1, c0));
          UQ0 = *reinterpret_cast<const f2*>(&SP(6, rl - 1, c0));
          UQ1 = *reinterpret_cast<const f2*>(&SP(8, rl - 1, c0));
        } else if (s_up) {
          const int last = A.rpc - 1;
          UPY = *reinterpret_cast<const f2*>(&s_up[(4) * PS + (last) * RS + (c0)]);
          UQ0 = *reinterpret_cast<const f2*>(&s_up[(6) * PS + (last) * RS + (c0)]);
          UQ1 = *reinterpret_cast<const f2*>(&s_up[(8) * PS + (last) * RS + (c0)]);
        } else {
          UPY = UQ0 = UQ1 = mk2(0.f, 0.f);
        }
        const f2 dv = sub2(add2(sub2(FX, mk2(lx, FX.x)), FY), UPY);
        const f2 d0 = sub2(add2(sub2(F0X, mk2(l0, F0X.x)), F0Y), UQ0);
        const f2 d1 = sub2(add2(sub2(F1X, mk2(l1, F1X.x)), F1Y), UQ1);
        const f2 uhat = fma2(mul2(tu2, al1), dv, U);
        const f2 rhat = fma2(sub2(uhat, UO), G, RH);
        const f2 tl = mul2(tu2, lam2);
        const f2 un = mk2(shrink1(uhat.x, rhat.x, G.x, tl.x), shrink1(uhat.y, rhat.y, G.y, tl.y));
        const f2 v0n = fma2(tv2, fma2(al0, d0, mul2(al1, P0)), V0);
        const f2 v1n = fma2(tv2, fma2(al0, d1, mul2(al1, P1)), V1);
        UB = fma2(th2, sub2(un, U), un);
        VB0 = fma2(th2, sub2(v0n, V0), v0n);
        VB1 = fma2(th2, sub2(v1n, V1), v1n);
        U = un; V0 = v0n; V1 = v1n;
      }
    }
    // ---- clip and accumulate (solver.py:356-360)
    float dmax = 0.f;
    double dsum = 0.0;
    if (row_ok) {
      float du[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float un = e ? U.y : U.x, uo = e ? UO.y : UO.x;
        du[e] = fminf(fmaxf(un - uo, -A.du_max), A.du_max);
        if (m[e] == 0.f || c0 + e >= W) du[e] = 0.f;
        wx[e] = wx[e] + du[e] * dx[e];
        wy[e] = wy[e] + du[e] * dy[e];
        dmax = fmaxf(dmax, fabsf(du[e]));
        dsum += (double)fabsf(du[e]);
      }
      U = mk2(UO.x + du[0], UO.y + du[1]);
    }
    if (A.diag_du) {
      dmax = warp_max(dmax);
      dsum = warp_sum(dsum);
      if (lane == 0) { s_red[warp] = dsum; s_redm[warp] = dmax; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        float mm = 0.f;
        const int nw = blockDim.x >> 5;
        for (int k = 0; k < nw; ++k) { t += s_red[k]; mm = fmaxf(mm, s_redm[k]); }
        s_psum[wi] = t;
        atomic_max_nonneg(A.diag_du + wi, mm);
      }
      __syncthreads();
    }
    cluster_sync_all();  // next warp rewrites i1w: everyone finished reading it
  }

  // ---- level result
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int x = c0 + e;
    if (!row_ok || x >= W) continue;
    const size_t i = (size_t)y * W + x;
    A.u[i] = e ? U.y : U.x;
    A.wv[2 * i] = wx[e];
    A.wv[2 * i + 1] = wy[e];
    A.v[i] = e ? V0.y : V0.x;
    A.v[n + i] = e ? V1.y : V1.x;
    A.ub[i] = e ? U.y : U.x;
    A.vb[i] = e ? VB0.y : VB0.x;
    A.vb[n + i] = e ? VB1.y : VB1.x;
    A.p[i] = e ? P0.y : P0.x;
    A.p[n + i] = e ? P1.y : P1.x;
    A.q[i] = e ? Q0.y : Q0.x;
    A.q[n + i] = e ? Q1.y : Q1.x;
    A.q[2 * n + i] = e ? Q2.y : Q2.x;
    A.q[3 * n + i] = e ? Q3.y : Q3.x;
  }
  if (A.diag_mean) {  // mean |du|: rank-ordered sum of the CTA sums / mask count
    cluster_sync_all();
    if (rank == 0 && (int)threadIdx.x < A.N) {
      double t = 0.0;
      unsigned long long cnt = 0;
      for (int r = 0; r < ncta; ++r) {
        t += cluster.map_shared_rank(s_psum, r)[threadIdx.x];
        cnt += *cluster.map_shared_rank(&s_cnt, r);
      }
      A.diag_mean[threadIdx.x] = cnt ? t / (double)cnt : 0.0;
    }
  }
  cluster_sync_all();  // keep this CTA's shared memory alive for DSMEM readers
#undef SP
}

}  // namespace

// Geometry of the cluster for a level, or false when the level is too large.
bool cluster_shape(int h, int w, int* ncta, int* rpc, int* wr) {
  const int r = (w + 63) / 64;
  if (r * 64 > kMaxCols) return false;
  const int rows = (h + 15) / 16;  // rows per CTA over <= 16 CTAs
  if (rows > kMaxRows || r * rows > 16) return false;  // <= 512 threads: no spills
  *wr = r;
  *rpc = rows;
  *ncta = (h + rows - 1) / rows;
  return true;
}

bool level_cluster_fits(int h, int w, int warp_iters) {
  int a, b, c;
  static const int off = [] {
    const char* e = getenv("FSB_CLUSTER");
    return e && e[0] == '0';
  }();
  return !off && warp_iters <= kMaxWarps && cluster_shape(h, w, &a, &b, &c);
}

// The whole warp loop of one level (solver.py:331-365) in one cluster launch.
// Final u, w, v, p, q, u_bar, v_bar land in the level's primary planes.
int level_cluster_solve(const fsb_level* L, const fsb_params* prm, const fsb_diag* diag,
                        int64_t pd_off, int64_t warp_off, cudaStream_t st) {
  ClusterArgs A;
  memset(&A, 0, sizeof(A));
  int ncta;
  if (!cluster_shape(L->h, L->w, &ncta, &A.rpc, &A.wr) || prm->warp_iters > kMaxWarps)
    return FSB_EINVAL;
  A.h = L->h; A.w = L->w; A.n = (size_t)L->h * L->w;
  A.mask = L->mask; A.T = L->tensor; A.S = L->steps; A.i0 = L->i0;
  A.u = L->u; A.wv = L->wv; A.v = L->v; A.p = L->p; A.q = L->q; A.ub = L->u_bar; A.vb = L->v_bar;
  A.i1w = L->i1w; A.i1w_ok = L->i1w_ok;
  A.src = SampleSrc{L->i1, L->mask, L->traj, L->traj_ok,
                    reinterpret_cast<const float4*>(L->packed), L->full16, L->h, L->w};
  A.lam = (float)prm->lam; A.alpha0 = (float)prm->alpha0; A.alpha1 = (float)prm->alpha1;
  A.theta = (float)prm->theta; A.sigma_q = (float)sigma_q_of(prm);
  A.huber_eps = (float)huber_eps_of(prm);
  A.du_max = (float)prm->du_max;
  A.N = prm->warp_iters; A.K = prm->pd_iters;
  if (diag && diag->max_p_norm && diag->max_q_norm) {
    A.diag_p = diag->max_p_norm + pd_off;
    A.diag_q = diag->max_q_norm + pd_off;
  }
  if (diag && diag->max_du && diag->mean_abs_du) {
    A.diag_du = diag->max_du + warp_off;
    A.diag_mean = diag->mean_abs_du + warp_off;
  }
  const int nthreads = 32 * A.wr * A.rpc;
  void (*kern)(const ClusterArgs) =
      nthreads <= 256 ? k_level_cluster<256> : k_level_cluster<512>;
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [] {
    for (auto k : {k_level_cluster<256>, k_level_cluster<512>}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kPlanes * kMaxRows * (kMaxCols + 2) * (int)sizeof(float));
    }
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta, 1, 1);
  cfg.blockDim = dim3(nthreads, 1, 1);
  cfg.dynamicSmemBytes = (size_t)kPlanes * A.rpc * (A.wr * 64 + 2) * sizeof(float);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, A);
  if (e != cudaSuccess) return (int)e;
  return launch_status();
}

}  // namespace fsb
