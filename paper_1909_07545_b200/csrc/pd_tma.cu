// K6 (v4): persistent, TMA-fed pixel-pair primal-dual kernel.
//
// Same cycles as k_pd_pair (pd_pair.cu) — packed fp32x2 arithmetic on pixel
// pairs, shuffles for x-neighbours, strip-edge shared-memory exchange for
// y-neighbours, R-pixel halo, `iters` cycles per launch — but the per-tile
// load is issued by one thread as two 3-D TMA boxes (cp.async.bulk.tensor):
// the 12 state planes and the 10 constant planes (tensor a b c, steps,
// I_u, rho0, u_omega, mask) of a 64 x 32 tile (68-wide box, see kBoxW),
// zero-filled outside the image,
// landing in shared memory under an mbarrier. CTAs are persistent (one per
// SM) and prefetch tile t + gridDim while they iterate on tile t, so the
// 176 KB tile load overlaps the cycles instead of stalling them.
//
// Requirements (checked by the driver, else it uses k_pd_pair): both state
// sets and the constants are plane blocks of stride n = h*w, w % 4 == 0.

#include <cuda.h>
#include <stdlib.h>

#include "pd_args.cuh"
#include "pd_math.cuh"
#include "tma.cuh"

namespace fsb {
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
FSB_INLINE f2 shrink2(f2 uh, f2 rh, f2 g, f2 tl) {
  return mk2(shrink1(uh.x, rh.x, g.x, tl.x), shrink1(uh.y, rh.y, g.y, tl.y));
}

#ifndef FSB_ALIGNED_LOAD
#define FSB_ALIGNED_LOAD 0  // measured slower: the unpack shuffles cost more than the 2-way bank conflicts
#endif
#ifndef FSB_ALIGNED_STORE
#define FSB_ALIGNED_STORE 1
#endif
constexpr int kNW = 16, kPY = 2, kEW = 64, kEH = kNW * kPY;
constexpr int kStatePlanes = 12, kConstPlanes = 10;
// TMA needs the box's innermost start coordinate 16-byte aligned (measured on
// this B200 / driver: x0 % 4 != 0 faults). The box is therefore 4 columns wider
// than the 64-column tile and starts at floor4(ox); the kernel reads with the
// resulting 0..3 column shift.
constexpr int kBoxW = kEW + 4;
constexpr int kPlane = kBoxW * kEH;  // floats per plane in the staging tile
constexpr uint32_t kTileBytes = (kStatePlanes + kConstPlanes) * kPlane * sizeof(float);
constexpr size_t kSmemBytes = 1024 /*align slack*/ + kTileBytes +
                              2 * sizeof(f2) * kNW * 3 * 32 /*s_top, s_bot*/ + 64 /*mbarrier*/;

// staging plane indices
enum { SU, SUB, SV0, SV1, SVB0, SVB1, SP0, SP1, SQ0, SQ1, SQ2, SQ3 };
enum { CA, CB, CC, CSP, CTU, CTV, CIU, CRH, CUO, CM };

template <int R, bool LIN, bool FIN, bool DIAG>
__global__ void __launch_bounds__(kNW * 32, 1)
    k_pd_tma(const BlockArgs A, const __grid_constant__ CUtensorMap tm_src,
             const __grid_constant__ CUtensorMap tm_const, int ntx, int ntiles,
             const int* __restrict__ tlist) {
  constexpr int TW = kEW - 2 * R, TH = kEH - 2 * R, NW = kNW, PY = kPY, EH = kEH;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ unsigned char smem_raw[];
  // 1024-B aligned staging base, formed as an offset from the shared array
  // itself (not through a uintptr_t round trip) so the compiler keeps the
  // shared address space: LDS / STS instead of generic LD / ST.
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  poison_dynamic_smem(smem_raw);  // checked build only (before the mbarrier lives there)
  float* st = reinterpret_cast<float*>(base);  // [12 + 10][EH][64]
  const float* cs = st + kStatePlanes * kPlane;
  f2(*s_top)[3][32] = reinterpret_cast<f2(*)[3][32]>(base + kTileBytes);
  f2(*s_bot)[3][32] = s_top + NW;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_bot + NW);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = warp * PY, c0 = 2 * lane;
  const size_t n = A.n;

  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  // The tensor maps are used straight from the __grid_constant__ parameters
  // (never copied: TMA needs the descriptor in param/const/global space).
#define FSB_ISSUE_TILE(TILE)                                                              \
  do {                                                                                    \
    if (threadIdx.x == 0) {                                                               \
      const int tx_ = (TILE) % ntx, ty_ = (TILE) / ntx;                                   \
      const int bx_ = (tx_ * TW - R) & ~3; /* floor to a multiple of 4 */                 \
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");                        \
      mbar_expect_tx(bar, kTileBytes);                                                    \
      tma_load_3d(st, &tm_src, bx_, ty_ * TH - R, 0, bar);                                 \
      tma_load_3d(st + kStatePlanes * kPlane, &tm_const, bx_, ty_ * TH - R, 0, bar);       \
    }                                                                                     \
  } while (0)

  // Work list: all tiles, or the compacted list of tiles holding mask pixels
  // (tlist[0] = count, tlist[1 + k] = tile id; pd_tma_tile_list).
  const int cnt = tlist ? tlist[0] : ntiles;
  uint32_t parity = 0;
  int k = blockIdx.x;
  if (k < cnt) FSB_ISSUE_TILE(tlist ? tlist[1 + k] : k);
  for (; k < cnt; k += gridDim.x) {
    const int tile = tlist ? tlist[1 + k] : k;
    const int ox = (tile % ntx) * TW - R, oy = (tile / ntx) * TH - R;
    mbar_wait(bar, parity);
    parity ^= 1;

    f2 u[PY], v0[PY], v1[PY], p0[PY], p1[PY], q0[PY], q1[PY], q2[PY], q3[PY];
    f2 ub[PY], vb0[PY], vb1[PY];
    f2 ta[PY], tb[PY], tc[PY], sp[PY], tu[PY], tv[PY], g[PY], rh[PY], uo[PY];
    f2 exf[PY], eyf[PY];
    unsigned mbits = 0;  // mask of the two pixels of row j at bits 2j, 2j+1
    const f2 a1 = mk2(A.alpha1, A.alpha1);
    const int shift = ox - (ox & ~3);  // staging column of tile column 0 (parity of R)
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int r = r0 + j;
      const int o = r * kBoxW + c0 + shift;
      // Pixel pair (c0, c0+1) of a staged plane. Even R: 8-B aligned, one LDS.64.
      // Odd R: the aligned pair is (c0+1, c0+2); c0 comes from the lane below
      // by shuffle (lane 0 reads it directly) — conflict-free 64-bit loads
      // instead of two stride-2 scalar loads.
      auto pair = [&](const float* pl) -> f2 {
        if constexpr (!FSB_ALIGNED_LOAD) {
          return mk2(pl[o], pl[o + 1]);
        } else if constexpr ((R & 1) == 0) {
          return *reinterpret_cast<const f2*>(pl + o);
        } else {
          const f2 q = *reinterpret_cast<const f2*>(pl + o + 1);
          float left = __shfl_up_sync(FULL, q.y, 1);
          if (lane == 0) left = pl[o];
          return mk2(left, q.x);
        }
      };
      auto S2 = [&](int plane) { return pair(st + plane * kPlane); };
      auto C2 = [&](int plane) { return pair(cs + plane * kPlane); };
      u[j] = S2(SU); v0[j] = S2(SV0); v1[j] = S2(SV1);
      p0[j] = S2(SP0); p1[j] = S2(SP1);
      q0[j] = S2(SQ0); q1[j] = S2(SQ1); q2[j] = S2(SQ2); q3[j] = S2(SQ3);
      ta[j] = C2(CA); tb[j] = C2(CB); tc[j] = C2(CC);
      sp[j] = mul2(C2(CSP), a1); tu[j] = C2(CTU); tv[j] = C2(CTV);
      g[j] = C2(CIU); rh[j] = C2(CRH);
      if (LIN) {  // warp start (solver.py:344-346)
        uo[j] = u[j]; ub[j] = u[j]; vb0[j] = v0[j]; vb1[j] = v1[j];
      } else {
        uo[j] = C2(CUO); ub[j] = S2(SUB); vb0[j] = S2(SVB0); vb1[j] = S2(SVB1);
      }
      // mask (0/1 floats; zero outside the image and past the tile edge)
      const f2 m = C2(CM);
      const float mr = c0 + 2 < kEW ? cs[CM * kPlane + o + 2] : 0.f;
      const f2 md = r + 1 < EH ? mk2(cs[CM * kPlane + o + kBoxW], cs[CM * kPlane + o + kBoxW + 1])
                               : mk2(0.f, 0.f);
      exf[j] = mk2(m.x * m.y, m.y * mr);
      eyf[j] = mk2(m.x * md.x, m.y * md.y);
      mbits |= (m.x != 0.f ? 1u : 0u) << (2 * j);
      mbits |= (m.y != 0.f ? 1u : 0u) << (2 * j + 1);
    }
    __syncthreads();  // staging consumed: prefetch the next tile behind the cycles
    if (k + (int)gridDim.x < cnt) FSB_ISSUE_TILE(tlist ? tlist[1 + k + gridDim.x] : k + gridDim.x);

    const f2 sq2 = mk2(A.sigma_q * A.alpha0, A.sigma_q * A.alpha0);
    const f2 al0 = mk2(A.alpha0, A.alpha0), th2 = mk2(A.theta, A.theta);
    const f2 lam2 = mk2(A.lam, A.lam), zero = mk2(0.f, 0.f);

    // Rows whose cycle-`it` values reach the stored interior (dependency cone):
    // the primal half needs [lo, hi), the dual half one more row above (the
    // primal reads the flux of the row above). Warps entirely outside, or
    // entirely outside the image, skip the math but keep publishing and the
    // barriers; whatever they hold is never read by a needed row.
    for (int it = 1; it <= A.iters; ++it) {
      s_top[warp][0][lane] = ub[0];
      s_top[warp][1][lane] = vb0[0];
      s_top[warp][2][lane] = vb1[0];
      __syncthreads();
      float pmax = 0.f, qmax = 0.f;
      f2 fpx[PY], fpy[PY], fq0x[PY], fq0y[PY], fq1x[PY], fq1y[PY];
#pragma unroll
      for (int j = 0; j < PY; ++j) {
        const float nub = __shfl_down_sync(FULL, ub[j].x, 1);
        const float nvb0 = __shfl_down_sync(FULL, vb0[j].x, 1);
        const float nvb1 = __shfl_down_sync(FULL, vb1[j].x, 1);
        f2 dub, dvb0, dvb1;
        if (j + 1 < PY) {
          dub = ub[j + 1]; dvb0 = vb0[j + 1]; dvb1 = vb1[j + 1];
        } else if (warp + 1 < NW) {
          dub = s_top[warp + 1][0][lane]; dvb0 = s_top[warp + 1][1][lane];
          dvb1 = s_top[warp + 1][2][lane];
        } else {
          dub = dvb0 = dvb1 = zero;
        }
        const f2 gx = mul2(exf[j], sub2(mk2(ub[j].y, nub), ub[j]));
        const f2 gy = mul2(eyf[j], sub2(dub, ub[j]));
        const f2 g00 = mul2(exf[j], sub2(mk2(vb0[j].y, nvb0), vb0[j]));
        const f2 g01 = mul2(eyf[j], sub2(dvb0, vb0[j]));
        const f2 g10 = mul2(exf[j], sub2(mk2(vb1[j].y, nvb1), vb1[j]));
        const f2 g11 = mul2(eyf[j], sub2(dvb1, vb1[j]));
        const f2 t0 = sub2(fma2(ta[j], gx, mul2(tb[j], gy)), vb0[j]);
        const f2 t1 = sub2(fma2(tb[j], gx, mul2(tc[j], gy)), vb1[j]);
        f2 pp0 = fma2(sp[j], t0, p0[j]);
        f2 pp1 = fma2(sp[j], t1, p1[j]);
        if (A.huber_eps > 0.f) {  // Huber-TV: p / (1 + sp eps) before the projection
          const f2 kk = mk2(__frcp_rn(fmaf(sp[j].x, A.huber_eps, 1.f)),
                            __frcp_rn(fmaf(sp[j].y, A.huber_eps, 1.f)));
          pp0 = mul2(pp0, kk);
          pp1 = mul2(pp1, kk);
        }
        const f2 rp = unit_scale2(fma2(pp0, pp0, mul2(pp1, pp1)));
        p0[j] = mul2(pp0, rp);
        p1[j] = mul2(pp1, rp);
        const f2 qq0 = fma2(sq2, g00, q0[j]), qq1 = fma2(sq2, g01, q1[j]);
        const f2 qq2 = fma2(sq2, g10, q2[j]), qq3 = fma2(sq2, g11, q3[j]);
        const f2 rq = unit_scale2(add2(fma2(qq0, qq0, mul2(qq1, qq1)),
                                       fma2(qq2, qq2, mul2(qq3, qq3))));
        q0[j] = mul2(qq0, rq); q1[j] = mul2(qq1, rq);
        q2[j] = mul2(qq2, rq); q3[j] = mul2(qq3, rq);
        fpx[j] = mul2(exf[j], fma2(ta[j], p0[j], mul2(tb[j], p1[j])));
        fpy[j] = mul2(eyf[j], fma2(tb[j], p0[j], mul2(tc[j], p1[j])));
        fq0x[j] = mul2(exf[j], q0[j]); fq0y[j] = mul2(eyf[j], q1[j]);
        fq1x[j] = mul2(exf[j], q2[j]); fq1y[j] = mul2(eyf[j], q3[j]);
        if (DIAG) {
          const int r = r0 + j, gyy = oy + r;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = c0 + e, gxx = ox + c;
            if (r >= R && r < EH - R && c >= R && c < kEW - R &&
                (unsigned)gxx < (unsigned)A.w && (unsigned)gyy < (unsigned)A.h) {
              const float a0 = e ? p0[j].y : p0[j].x, a1_ = e ? p1[j].y : p1[j].x;
              const float b0 = e ? q0[j].y : q0[j].x, b1 = e ? q1[j].y : q1[j].x;
              const float b2 = e ? q2[j].y : q2[j].x, b3 = e ? q3[j].y : q3[j].x;
              pmax = fmaxf(pmax, sqrtf(a0 * a0 + a1_ * a1_));
              qmax = fmaxf(qmax, sqrtf((b0 * b0 + b1 * b1) + (b2 * b2 + b3 * b3)));
            }
          }
        }
      }
      if (DIAG) {
        pmax = warp_max(pmax);
        qmax = warp_max(qmax);
        if (lane == 0 && A.diag_p && A.diag_q) {
          atomic_max_nonneg(A.diag_p + it - 1, pmax);
          atomic_max_nonneg(A.diag_q + it - 1, qmax);
        }
      }
      s_bot[warp][0][lane] = fpy[PY - 1];
      s_bot[warp][1][lane] = fq0y[PY - 1];
      s_bot[warp][2][lane] = fq1y[PY - 1];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < PY; ++j) {
        const float lpx = __shfl_up_sync(FULL, fpx[j].y, 1);
        const float lq0 = __shfl_up_sync(FULL, fq0x[j].y, 1);
        const float lq1 = __shfl_up_sync(FULL, fq1x[j].y, 1);
        f2 upy, uq0, uq1;
        if (j > 0) {
          upy = fpy[j - 1]; uq0 = fq0y[j - 1]; uq1 = fq1y[j - 1];
        } else if (warp > 0) {
          upy = s_bot[warp - 1][0][lane]; uq0 = s_bot[warp - 1][1][lane];
          uq1 = s_bot[warp - 1][2][lane];
        } else {
          upy = uq0 = uq1 = zero;
        }
        const f2 dv = sub2(add2(sub2(fpx[j], mk2(lpx, fpx[j].x)), fpy[j]), upy);
        const f2 d0 = sub2(add2(sub2(fq0x[j], mk2(lq0, fq0x[j].x)), fq0y[j]), uq0);
        const f2 d1 = sub2(add2(sub2(fq1x[j], mk2(lq1, fq1x[j].x)), fq1y[j]), uq1);
        const f2 uhat = fma2(mul2(tu[j], a1), dv, u[j]);
        const f2 rhat = fma2(sub2(uhat, uo[j]), g[j], rh[j]);
        const f2 un = shrink2(uhat, rhat, g[j], mul2(tu[j], lam2));
        const f2 v0n = fma2(tv[j], fma2(al0, d0, mul2(a1, p0[j])), v0[j]);
        const f2 v1n = fma2(tv[j], fma2(al0, d1, mul2(a1, p1[j])), v1[j]);
        ub[j] = fma2(th2, sub2(un, u[j]), un);
        vb0[j] = fma2(th2, sub2(v0n, v0[j]), v0n);
        vb1[j] = fma2(th2, sub2(v1n, v1[j]), v1n);
        u[j] = un; v0[j] = v0n; v1[j] = v1n;
      }
    }

    // ---- epilogue + store of the interior. Per-pixel work (clip, w update,
    // diagnostics) in the lane's own pair; the stores go out as 8-B aligned
    // pairs: even R owns them, odd R pairs its .y with the next lane's .x.
    float dmax = 0.f;
    double dsum = 0.0;
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int r = r0 + j, gy = oy + r;
      const bool row_in = r >= R && r < EH - R && (unsigned)gy < (unsigned)A.h;
      f2 U2 = u[j], UB2 = ub[j];
      if (FIN) {  // solver.py:356-360
        float uu[2] = {u[j].x, u[j].y};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = c0 + e, gx = ox + c;
          if (!row_in || c < R || c >= kEW - R || (unsigned)gx >= (unsigned)A.w) continue;
          const size_t gi = (size_t)gy * A.w + gx;
          const float uom = e ? uo[j].y : uo[j].x;
          const bool mk = (mbits >> (2 * j + e)) & 1u;
          float du = fminf(fmaxf(uu[e] - uom, -A.du_max), A.du_max);
          if (!mk) du = 0.f;
          uu[e] = uom + du;
          const float2 d = reinterpret_cast<const float2*>(A.dirs)[gi];
          float2 wv = reinterpret_cast<float2*>(A.wv)[gi];
          wv.x = wv.x + du * d.x;
          wv.y = wv.y + du * d.y;
          reinterpret_cast<float2*>(A.wv)[gi] = wv;
          dmax = fmaxf(dmax, fabsf(du));
          dsum += (double)fabsf(du);
        }
        U2 = mk2(uu[0], uu[1]);
        UB2 = U2;  // u_bar = u after the clip
      }
      // aligned pair start (tile column) of this lane and its store predicate
      constexpr bool kOddPairs = FSB_ALIGNED_STORE && (R & 1);
      const int cs0 = kOddPairs ? c0 + 1 : c0;
      const int gxs = ox + cs0;
      // interior columns [R, kEW - R) split exactly into aligned pairs (gxs even,
      // w % 4 == 0, so gxs + 1 < w whenever gxs < w)
      const bool st_ok = row_in && cs0 >= R && cs0 + 1 < kEW - R && gxs < A.w;
      const size_t gs = (size_t)gy * A.w + gxs;
      auto put = [&](float* plane, f2 v) {
        if constexpr (kOddPairs) {
          const f2 o2 = mk2(v.y, __shfl_down_sync(FULL, v.x, 1));
          if (st_ok) *reinterpret_cast<f2*>(plane + gs) = o2;
        } else if constexpr (FSB_ALIGNED_STORE) {
          if (st_ok) *reinterpret_cast<f2*>(plane + gs) = v;
        } else {
          const size_t g0 = (size_t)gy * A.w + (ox + c0);
          if (row_in && c0 >= R && c0 < kEW - R && ox + c0 < A.w) plane[g0] = v.x;
          if (row_in && c0 + 1 >= R && c0 + 1 < kEW - R && ox + c0 + 1 < A.w) plane[g0 + 1] = v.y;
        }
      };
      if (LIN) put(A.u_omega, uo[j]);
      put(A.dst.u, U2);
      // after a warp's last cycle u_bar / v_bar are dead (the next warp start
      // resets them, solver.py:344-346) unless this is the level's last warp
      const bool bars = !FIN || A.store_bars;
      if (bars) put(A.dst.ub, UB2);
      put(A.dst.v, v0[j]);
      put(A.dst.v + n, v1[j]);
      if (bars) {
        put(A.dst.vb, vb0[j]);
        put(A.dst.vb + n, vb1[j]);
      }
      put(A.dst.p, p0[j]);
      put(A.dst.p + n, p1[j]);
      put(A.dst.q, q0[j]);
      put(A.dst.q + n, q1[j]);
      put(A.dst.q + 2 * n, q2[j]);
      put(A.dst.q + 3 * n, q3[j]);
    }
    if (FIN && DIAG && A.diag_du) {
      __shared__ double red_s[NW];
      __shared__ float red_m[NW];
      dmax = warp_max(dmax);
      dsum = warp_sum(dsum);
      if (lane == 0) { red_s[warp] = dsum; red_m[warp] = dmax; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        float m = 0.f;
        for (int k = 0; k < NW; ++k) { t += red_s[k]; m = fmaxf(m, red_m[k]); }
        A.partials[tile] = t;  // tiles off the list keep the zero of the level start
        atomic_max_nonneg(A.diag_du, m);
      }
      __syncthreads();
    }
  }
#undef FSB_ISSUE_TILE
}

EncodeTiled encoder() { return tma_encoder(); }

// planes x h x w fp32 block with plane stride n; box 64 x 32 x planes
bool make_map(CUtensorMap* m, const float* base, int w, int h, int planes, size_t n) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)w * sizeof(float), (cuuint64_t)n * sizeof(float)};
  cuuint32_t box[3] = {(cuuint32_t)kBoxW, (cuuint32_t)kEH, (cuuint32_t)planes};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int num_sms() {
  static const int sms = [] {  // one SKU per process (one B200 per rank)
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

template <int R, bool LIN, bool FIN, bool DIAG>
int launch_tma(const BlockArgs& A, const CUtensorMap& ms, const CUtensorMap& mc, cudaStream_t st,
               int* ntiles_out) {
  constexpr int TW = kEW - 2 * R, TH = kEH - 2 * R;
  const int ntx = (A.w + TW - 1) / TW, nty = (A.h + TH - 1) / TH, ntiles = ntx * nty;
  static std::atomic<unsigned long long> attr{0};
  auto kern = k_pd_tma<R, LIN, FIN, DIAG>;
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  });
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  if (ntiles_out) *ntiles_out = ntiles;
  kern<<<grid, kNW * 32, kSmemBytes, st>>>(A, ms, mc, ntx, ntiles, A.tile_list);
  return launch_status();
}

template <int R, bool LIN, bool FIN>
int launch_tma_d(const BlockArgs& A, const CUtensorMap& ms, const CUtensorMap& mc,
                 cudaStream_t st, int* nt) {
  if (A.diag_p || A.diag_du) return launch_tma<R, LIN, FIN, true>(A, ms, mc, st, nt);
  return launch_tma<R, LIN, FIN, false>(A, ms, mc, st, nt);
}

template <int R>
int launch_tma_r(const BlockArgs& A, const CUtensorMap& ms, const CUtensorMap& mc, bool lin,
                 bool fin, cudaStream_t st, int* nt) {
  if (lin && fin) return launch_tma_d<R, true, true>(A, ms, mc, st, nt);
  if (lin) return launch_tma_d<R, true, false>(A, ms, mc, st, nt);
  if (fin) return launch_tma_d<R, false, true>(A, ms, mc, st, nt);
  return launch_tma_d<R, false, false>(A, ms, mc, st, nt);
}

// One block per tile: does the interior [tx*TW, +TW) x [ty*TH, +TH) hold a
// mask pixel? The flag lands at tiles[1 + tile].
__global__ void k_tile_flags(const uint8_t* __restrict__ m, int w, int h, int TW, int TH, int ntx,
                             int* __restrict__ tiles) {
  const int t = blockIdx.x, x0 = (t % ntx) * TW, y0 = (t / ntx) * TH;
  int any = 0;
  for (int k = threadIdx.x; k < TW * TH; k += blockDim.x) {
    const int x = x0 + k % TW, y = y0 + k / TW;
    if (x < w && y < h && m[(size_t)y * w + x]) any = 1;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) tiles[1 + t] = any;
}

// In-place stream compaction of the flags into ascending tile ids (one block):
// tiles[0] = count, tiles[1 + k] = k-th active tile.
__global__ void k_tile_compact(int* tiles, int ntiles) {
  __shared__ int s_scan[1024];
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < ntiles; c0 += blockDim.x) {
    const int t = c0 + threadIdx.x;
    const int f = t < ntiles ? tiles[1 + t] : 0;
    s_scan[threadIdx.x] = f;
    __syncthreads();
    for (int d = 1; d < (int)blockDim.x; d <<= 1) {  // Hillis-Steele inclusive scan
      const int v = threadIdx.x >= (unsigned)d ? s_scan[threadIdx.x - d] : 0;
      __syncthreads();
      s_scan[threadIdx.x] += v;
      __syncthreads();
    }
    const int pos = s_base + s_scan[threadIdx.x] - f;
    __syncthreads();  // every flag of this chunk read before any write below
    if (f) tiles[1 + pos] = t;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_base += s_scan[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) tiles[0] = s_base;
}

}  // namespace

// Generic form: tiles of TW x TH interior pixels on a row-major tile grid.
int tile_list_internal(const uint8_t* mask, int w, int h, int TW, int TH, int* tiles,
                       cudaStream_t st) {
  const int ntx = (w + TW - 1) / TW, nty = (h + TH - 1) / TH;
  k_tile_flags<<<ntx * nty, 256, 0, st>>>(mask, w, h, TW, TH, ntx, tiles);
  k_tile_compact<<<1, 1024, 0, st>>>(tiles, ntx * nty);
  return launch_status();
}

int pd_tma_tile_list(const uint8_t* mask, int w, int h, int halo, int* tiles, cudaStream_t st) {
  return tile_list_internal(mask, w, h, kEW - 2 * halo, kEH - 2 * halo, tiles, st);
}

bool pd_tma_maps(TmaMaps* maps, const float* state_a, const float* state_b, const float* consts,
                 int w, int h) {
  const size_t n = (size_t)w * h;
  if (w % 4 != 0) return false;
  if (((uintptr_t)state_a | (uintptr_t)state_b | (uintptr_t)consts) & 15) return false;
  return make_map(&maps->state[0], state_a, w, h, kStatePlanes, n) &&
         make_map(&maps->state[1], state_b, w, h, kStatePlanes, n) &&
         make_map(&maps->consts, consts, w, h, kConstPlanes, n);
}

int pd_num_sms() { return num_sms(); }

size_t pd_tma_partials(int w, int h, int halo) {
  const int TW = kEW - 2 * halo, TH = kEH - 2 * halo;
  return (size_t)((w + TW - 1) / TW) * ((h + TH - 1) / TH);
}

int pd_tma_launch(const BlockArgs& A, const TmaMaps& maps, int src_set, int halo, bool lin,
                  bool fin, cudaStream_t st, int* nparts) {
  if (A.iters < 1 || A.iters > halo) return FSB_EINVAL;
  const CUtensorMap& ms = maps.state[src_set];
  switch (halo) {
    case 1: return launch_tma_r<1>(A, ms, maps.consts, lin, fin, st, nparts);
    case 2: return launch_tma_r<2>(A, ms, maps.consts, lin, fin, st, nparts);
    case 3: return launch_tma_r<3>(A, ms, maps.consts, lin, fin, st, nparts);
    case 4: return launch_tma_r<4>(A, ms, maps.consts, lin, fin, st, nparts);
    case 5: return launch_tma_r<5>(A, ms, maps.consts, lin, fin, st, nparts);
    case 10: return launch_tma_r<10>(A, ms, maps.consts, lin, fin, st, nparts);
    default: return FSB_EINVAL;
  }
}

}  // namespace fsb
