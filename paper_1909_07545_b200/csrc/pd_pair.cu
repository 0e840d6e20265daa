// K6 (v3): temporally blocked primal-dual kernel on PIXEL PAIRS with packed
// fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2, sm_100).
//
// Same algorithm and launch contract as k_pd_block (pd_block.cu): `iters` full
// primal-dual cycles (solver.py:279-303) per launch on a 64-pixel-wide tile with
// an R-pixel halo, optional fused warp-start resets (LIN) and epilogue (FIN,
// solver.py:356-360). The data movement is reorganised around the hardware:
//   - a warp owns a horizontal strip of PY rows, each lane a pair of adjacent
//     columns (2l, 2l+1) held as float2 registers, so every arithmetic step of
//     the cycle is one packed instruction for two pixels;
//   - x-neighbours come from the lane's own pair or a warp shuffle (no shared
//     memory), y-neighbours from the thread's own rows except at the strip
//     edges, where one row per warp is published through shared memory;
//   - two block barriers per cycle, as before, but ~1/6 of the shared-memory
//     traffic of the per-pixel tile kernel.
// Rounding follows the per-pixel kernels (same contraction pattern), so both
// agree to fp32 round-off (tests/test_gpu_blocked.py).

#include <stdlib.h>

#include "pd_args.cuh"
#include "pd_math.cuh"

namespace fsb {



namespace {

typedef float2 f2;

FSB_INLINE f2 mk2(float a, float b) { return make_float2(a, b); }
FSB_INLINE f2 add2(f2 a, f2 b) { return __fadd2_rn(a, b); }
FSB_INLINE f2 sub2(f2 a, f2 b) { return __fadd2_rn(a, mk2(-b.x, -b.y)); }
FSB_INLINE f2 neg2(f2 a) { return mk2(-a.x, -a.y); }
FSB_INLINE f2 mul2(f2 a, f2 b) { return __fmul2_rn(a, b); }
FSB_INLINE f2 fma2(f2 a, f2 b, f2 c) { return __ffma2_rn(a, b, c); }
// edge masks are kept as 0/1 floats: x * 1 == x exactly, x * 0 == +-0 (finite x),
// one FMUL2 per pixel pair instead of two selects on predicate bits
FSB_INLINE f2 sub2(f2 a, f2 b);

// x / max(1, |x|) on two pixels at once (see dual_update in pd_math.cuh)
FSB_INLINE f2 unit_scale2(f2 n2) {
  return mk2(n2.x > 1.f ? rsqrtf(n2.x) : 1.f, n2.y > 1.f ? rsqrtf(n2.y) : 1.f);
}

// thresholding_step (solver.py:205-218) on two pixels, branch-free;
// tl = tau_u * lam. The interior case divides with the approximate reciprocal
// (<= 2 ulp, fp32 path); iu == 0 passes through exactly.
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

template <int NW, int PY, int R>
struct PairTile {
  static constexpr int EW = 64, EH = NW * PY;
  static constexpr int TW = EW - 2 * R, TH = EH - 2 * R;
  static_assert(TW > 0 && TH > 0, "halo larger than tile");
  static_assert(6 * PY <= 32, "mask bits");
};

template <int NW, int PY, int R, bool LIN, bool FIN, bool DIAG>
__global__ void __launch_bounds__(NW * 32, 1) k_pd_pair(const BlockArgs A) {
  using TL = PairTile<NW, PY, R>;
  constexpr int EH = TL::EH;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ f2 s_top[NW][3][32];  // first row of each strip: u_bar, v_bar0, v_bar1
  __shared__ f2 s_bot[NW][3][32];  // last row of each strip: y-fluxes py, q0y, q1y
  __shared__ uint8_t s_m[EH + 1][66];  // mask tile (+1 row / column of zero pad)

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ox = (int)blockIdx.x * TL::TW - R, oy = (int)blockIdx.y * TL::TH - R;
  const int r0 = warp * PY;  // first tile row of this strip
  const int c0 = 2 * lane;   // first tile column of this pair
  const size_t n = A.n;

  // ---- mask tile, then per-pixel edge bits
  for (int k = threadIdx.x; k < (EH + 1) * 66; k += NW * 32) {
    const int r = k / 66, c = k - r * 66;
    const int gx = ox + c, gy = oy + r;
    const bool in = c < 64 && r < EH && (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
    s_m[r][c] = in ? A.mask[(size_t)gy * A.w + gx] : 0;
  }
  __syncthreads();

  f2 u[PY], v0[PY], v1[PY], p0[PY], p1[PY], q0[PY], q1[PY], q2[PY], q3[PY];
  f2 ub[PY], vb0[PY], vb1[PY];
  f2 ta[PY], tb[PY], tc[PY], sp[PY], tu[PY], tv[PY], g[PY], rh[PY], uo[PY];
  f2 exf[PY], eyf[PY];  // forward-edge indicators as 0/1 floats
  unsigned bits = 0;  // per row j: m.x m.y ex.x ex.y ey.x ey.y at bit 6j
  const float a1 = A.alpha1;

#pragma unroll
  for (int j = 0; j < PY; ++j) {
    const int r = r0 + j;
    const int gy = oy + r;
    unsigned b = 0;
    b |= (s_m[r][c0] ? 1u : 0u) | (s_m[r][c0 + 1] ? 2u : 0u);
    b |= (s_m[r][c0] && s_m[r][c0 + 1] ? 4u : 0u) | (s_m[r][c0 + 1] && s_m[r][c0 + 2] ? 8u : 0u);
    b |= (s_m[r][c0] && s_m[r + 1][c0] ? 16u : 0u) | (s_m[r][c0 + 1] && s_m[r + 1][c0 + 1] ? 32u : 0u);
    bits |= b << (6 * j);
    exf[j] = mk2(b & 4u ? 1.f : 0.f, b & 8u ? 1.f : 0.f);
    eyf[j] = mk2(b & 16u ? 1.f : 0.f, b & 32u ? 1.f : 0.f);
    float lu[2], lv0[2], lv1[2], lp0[2], lp1[2], lq0[2], lq1[2], lq2[2], lq3[2], lub[2], lvb0[2],
        lvb1[2], la[2], lb[2], lc[2], lsp[2], ltu[2], ltv[2], lg[2], lrh[2], luo[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int gx = ox + c0 + e;
      const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
      if (in) {
        const size_t gi = (size_t)gy * A.w + gx;
        lu[e] = A.src.u[gi];
        lv0[e] = A.src.v[gi]; lv1[e] = A.src.v[n + gi];
        lp0[e] = A.src.p[gi]; lp1[e] = A.src.p[n + gi];
        lq0[e] = A.src.q[gi]; lq1[e] = A.src.q[n + gi];
        lq2[e] = A.src.q[2 * n + gi]; lq3[e] = A.src.q[3 * n + gi];
        la[e] = A.T[gi]; lb[e] = A.T[n + gi]; lc[e] = A.T[2 * n + gi];
        lsp[e] = A.S[gi] * a1; ltu[e] = A.S[n + gi]; ltv[e] = A.S[2 * n + gi];
        lg[e] = A.iu[gi]; lrh[e] = A.rho0[gi];
        if (LIN) {  // warp start (solver.py:344-346)
          luo[e] = lu[e]; lub[e] = lu[e]; lvb0[e] = lv0[e]; lvb1[e] = lv1[e];
        } else {
          luo[e] = A.u_omega[gi];
          lub[e] = A.src.ub[gi]; lvb0[e] = A.src.vb[gi]; lvb1[e] = A.src.vb[n + gi];
        }
      } else {
        lu[e] = lv0[e] = lv1[e] = lp0[e] = lp1[e] = lq0[e] = lq1[e] = lq2[e] = lq3[e] = 0.f;
        lub[e] = lvb0[e] = lvb1[e] = 0.f;
        la[e] = 1.f; lb[e] = 0.f; lc[e] = 1.f;
        lsp[e] = ltu[e] = ltv[e] = lg[e] = lrh[e] = luo[e] = 0.f;
      }
    }
    u[j] = mk2(lu[0], lu[1]); v0[j] = mk2(lv0[0], lv0[1]); v1[j] = mk2(lv1[0], lv1[1]);
    p0[j] = mk2(lp0[0], lp0[1]); p1[j] = mk2(lp1[0], lp1[1]);
    q0[j] = mk2(lq0[0], lq0[1]); q1[j] = mk2(lq1[0], lq1[1]);
    q2[j] = mk2(lq2[0], lq2[1]); q3[j] = mk2(lq3[0], lq3[1]);
    ub[j] = mk2(lub[0], lub[1]); vb0[j] = mk2(lvb0[0], lvb0[1]); vb1[j] = mk2(lvb1[0], lvb1[1]);
    ta[j] = mk2(la[0], la[1]); tb[j] = mk2(lb[0], lb[1]); tc[j] = mk2(lc[0], lc[1]);
    sp[j] = mk2(lsp[0], lsp[1]); tu[j] = mk2(ltu[0], ltu[1]); tv[j] = mk2(ltv[0], ltv[1]);
    g[j] = mk2(lg[0], lg[1]); rh[j] = mk2(lrh[0], lrh[1]); uo[j] = mk2(luo[0], luo[1]);
  }

  const f2 sq2 = mk2(A.sigma_q * A.alpha0, A.sigma_q * A.alpha0);
  const f2 al0 = mk2(A.alpha0, A.alpha0), al1 = mk2(a1, a1), th2 = mk2(A.theta, A.theta);
  const f2 ta1 = al1;  // tau_u * alpha1 uses alpha1
  const f2 zero = mk2(0.f, 0.f);
  const f2 lam2 = mk2(A.lam, A.lam);

  for (int it = 1; it <= A.iters; ++it) {
    // publish this strip's first row of u_bar / v_bar for the strip above
    s_top[warp][0][lane] = ub[0];
    s_top[warp][1][lane] = vb0[0];
    s_top[warp][2][lane] = vb1[0];
    __syncthreads();

    float pmax = 0.f, qmax = 0.f;
    f2 fpx[PY], fpy[PY], fq0x[PY], fq0y[PY], fq1x[PY], fq1y[PY];
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      // right neighbours: own .y for .x, next lane's .x for .y. Lane 31's .y is
      // tile column 63, inside the halo and without an x-edge: any finite value.
      const float nub = __shfl_down_sync(FULL, ub[j].x, 1);
      const float nvb0 = __shfl_down_sync(FULL, vb0[j].x, 1);
      const float nvb1 = __shfl_down_sync(FULL, vb1[j].x, 1);
      // down neighbours: own next row, or the next strip's published first row
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
      // dual ascent (solver.py:290-293), two pixels per instruction
      f2 t0 = sub2(fma2(ta[j], gx, mul2(tb[j], gy)), vb0[j]);
      f2 t1 = sub2(fma2(tb[j], gx, mul2(tc[j], gy)), vb1[j]);
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
      f2 qq0 = fma2(sq2, g00, q0[j]), qq1 = fma2(sq2, g01, q1[j]);
      f2 qq2 = fma2(sq2, g10, q2[j]), qq3 = fma2(sq2, g11, q3[j]);
      const f2 qn2 = add2(fma2(qq0, qq0, mul2(qq1, qq1)), fma2(qq2, qq2, mul2(qq3, qq3)));
      const f2 rq = unit_scale2(qn2);
      q0[j] = mul2(qq0, rq); q1[j] = mul2(qq1, rq); q2[j] = mul2(qq2, rq); q3[j] = mul2(qq3, rq);
      // edge-masked fluxes
      fpx[j] = mul2(exf[j], fma2(ta[j], p0[j], mul2(tb[j], p1[j])));
      fpy[j] = mul2(eyf[j], fma2(tb[j], p0[j], mul2(tc[j], p1[j])));
      fq0x[j] = mul2(exf[j], q0[j]); fq0y[j] = mul2(eyf[j], q1[j]);
      fq1x[j] = mul2(exf[j], q2[j]); fq1y[j] = mul2(eyf[j], q3[j]);
      if (DIAG) {
        const int r = r0 + j, gyy = oy + r;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = c0 + e, gxx = ox + c;
          if (r >= R && r < EH - R && c >= R && c < 64 - R && (unsigned)gxx < (unsigned)A.w &&
              (unsigned)gyy < (unsigned)A.h) {
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
    // publish this strip's last row of y-fluxes for the strip below
    s_bot[warp][0][lane] = fpy[PY - 1];
    s_bot[warp][1][lane] = fq0y[PY - 1];
    s_bot[warp][2][lane] = fq1y[PY - 1];
    __syncthreads();

#pragma unroll
    for (int j = 0; j < PY; ++j) {
      // left neighbours: previous lane's .y for .x, own .x for .y. Lane 0's .x is
      // tile column 0, inside the halo: the value it reads only feeds halo pixels.
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
      // backward divergences ((f - f_left) + f_y) - f_up (rasters.py:168-171)
      const f2 dv = sub2(add2(sub2(fpx[j], mk2(lpx, fpx[j].x)), fpy[j]), upy);
      const f2 d0 = sub2(add2(sub2(fq0x[j], mk2(lq0, fq0x[j].x)), fq0y[j]), uq0);
      const f2 d1 = sub2(add2(sub2(fq1x[j], mk2(lq1, fq1x[j].x)), fq1y[j]), uq1);
      // primal descent + shrinkage + relaxation (solver.py:295-302)
      const f2 uhat = fma2(mul2(tu[j], ta1), dv, u[j]);
      const f2 rhat = fma2(sub2(uhat, uo[j]), g[j], rh[j]);
      const f2 un = shrink2(uhat, rhat, g[j], mul2(tu[j], lam2));
      const f2 v0n = fma2(tv[j], fma2(al0, d0, mul2(al1, p0[j])), v0[j]);
      const f2 v1n = fma2(tv[j], fma2(al0, d1, mul2(al1, p1[j])), v1[j]);
      ub[j] = fma2(th2, sub2(un, u[j]), un);
      vb0[j] = fma2(th2, sub2(v0n, v0[j]), v0n);
      vb1[j] = fma2(th2, sub2(v1n, v1[j]), v1n);
      u[j] = un; v0[j] = v0n; v1[j] = v1n;
    }
  }

  // ---- epilogue + store of the interior
  float dmax = 0.f;
  double dsum = 0.0;
#pragma unroll
  for (int j = 0; j < PY; ++j) {
    const int r = r0 + j, gy = oy + r;
    if (r < R || r >= EH - R || (unsigned)gy >= (unsigned)A.h) continue;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = c0 + e, gx = ox + c;
      if (c < R || c >= 64 - R || (unsigned)gx >= (unsigned)A.w) continue;
      const size_t gi = (size_t)gy * A.w + gx;
      float uu = e ? u[j].y : u[j].x, ubb = e ? ub[j].y : ub[j].x;
      if (FIN) {  // solver.py:356-360
        const float uom = e ? uo[j].y : uo[j].x;
        const bool mk = (bits >> (6 * j + e)) & 1u;
        float du = fminf(fmaxf(uu - uom, -A.du_max), A.du_max);
        if (!mk) du = 0.f;
        uu = uom + du;
        ubb = uu;
        const float2 d = reinterpret_cast<const float2*>(A.dirs)[gi];
        float2 wv = reinterpret_cast<float2*>(A.wv)[gi];
        wv.x = wv.x + du * d.x;
        wv.y = wv.y + du * d.y;
        reinterpret_cast<float2*>(A.wv)[gi] = wv;
        dmax = fmaxf(dmax, fabsf(du));
        dsum += (double)fabsf(du);
      }
      if (LIN) A.u_omega[gi] = e ? uo[j].y : uo[j].x;
      A.dst.u[gi] = uu;
      A.dst.ub[gi] = ubb;
      A.dst.v[gi] = e ? v0[j].y : v0[j].x;
      A.dst.v[n + gi] = e ? v1[j].y : v1[j].x;
      A.dst.vb[gi] = e ? vb0[j].y : vb0[j].x;
      A.dst.vb[n + gi] = e ? vb1[j].y : vb1[j].x;
      A.dst.p[gi] = e ? p0[j].y : p0[j].x;
      A.dst.p[n + gi] = e ? p1[j].y : p1[j].x;
      A.dst.q[gi] = e ? q0[j].y : q0[j].x;
      A.dst.q[n + gi] = e ? q1[j].y : q1[j].x;
      A.dst.q[2 * n + gi] = e ? q2[j].y : q2[j].x;
      A.dst.q[3 * n + gi] = e ? q3[j].y : q3[j].x;
    }
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
      A.partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
      atomic_max_nonneg(A.diag_du, m);
    }
  }
}

template <int NW, int PY, int R, bool LIN, bool FIN>
int launch_pair_shape(const BlockArgs& A, cudaStream_t st, int* nblocks) {
  using TL = PairTile<NW, PY, R>;
  dim3 grd((A.w + TL::TW - 1) / TL::TW, (A.h + TL::TH - 1) / TL::TH);
  if (nblocks) *nblocks = (int)(grd.x * grd.y);
  if (A.diag_p || A.diag_du)
    k_pd_pair<NW, PY, R, LIN, FIN, true><<<grd, NW * 32, 0, st>>>(A);
  else
    k_pd_pair<NW, PY, R, LIN, FIN, false><<<grd, NW * 32, 0, st>>>(A);
  return launch_status();
}

int pair_shape() {
  static const int t = [] {
    const char* e = getenv("FSB_PAIR_SHAPE");
    return e ? atoi(e) : 0;
  }();
  return t;
}

template <int R, bool LIN, bool FIN>
int launch_pair(const BlockArgs& A, cudaStream_t st, int* nblocks) {
  switch (pair_shape()) {  // 0: 16 warps x 2 rows, 1: 8 warps x 4 rows (64 x 32 tiles)
    case 1: return launch_pair_shape<8, 4, R, LIN, FIN>(A, st, nblocks);
    default: return launch_pair_shape<16, 2, R, LIN, FIN>(A, st, nblocks);
  }
}

template <int R>
int launch_pair_r(const BlockArgs& A, bool lin, bool fin, cudaStream_t st, int* nb) {
  if (lin && fin) return launch_pair<R, true, true>(A, st, nb);
  if (lin) return launch_pair<R, true, false>(A, st, nb);
  if (fin) return launch_pair<R, false, true>(A, st, nb);
  return launch_pair<R, false, false>(A, st, nb);
}

}  // namespace

int pd_pair_launch(const BlockArgs& A, int halo, bool lin, bool fin, cudaStream_t st,
                   int* nblocks) {
  if (A.iters < 1 || A.iters > halo) return FSB_EINVAL;
  switch (halo) {
    case 1: return launch_pair_r<1>(A, lin, fin, st, nblocks);
    case 2: return launch_pair_r<2>(A, lin, fin, st, nblocks);
    case 3: return launch_pair_r<3>(A, lin, fin, st, nblocks);
    case 5: return launch_pair_r<5>(A, lin, fin, st, nblocks);
    default: return FSB_EINVAL;
  }
}

}  // namespace fsb
