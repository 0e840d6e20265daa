// Temporally blocked primal-dual cycles for the float64 path (round-1 kernel,
// FSB_PD64K=block; the default is k64_tile, pd64_tile.cu).
//
// k64_dual + k64_primal (pd64.cu) run one cycle per launch pair and move the
// whole fp64 state through HBM twice per cycle. This kernel keeps a 32 x 16
// tile (one pixel per thread, state in registers) on chip for `iters` <= R
// cycles with an R-pixel halo, exchanging u_bar / v_bar and the edge-masked
// fluxes through shared memory. The arithmetic is the same helpers in the
// same order (dual_update_exact, make_flux_exact, the divergence expression
// of k64_primal, primal_update_exact), compiled with -fmad=false, so the
// interior results are bit-identical to the one-cycle kernels.
//
// Reference: solver.py:279-303 (primal_dual_iterate), rasters.py:144-182.

#include "pd64_block.cuh"
#include "pd_math.cuh"

#include <stddef.h>
#include <stdlib.h>
#include <string.h>

namespace fsb {



namespace {

constexpr int kTX = 32, kTY = 16;

// Shared-memory image of one tile (dynamic): the u_bar / v_bar exchange, the
// six edge-masked fluxes and (CS) the nine per-pixel constants.
template <int TY>
struct Tile64 {
  double ub[TY][kTX + 1], vb0[TY][kTX + 1], vb1[TY][kTX + 1];
  double f[6][TY][kTX + 1];  // px py q0x q0y q1x q1y
  double c[9][TY][kTX];
};

// Per-pixel constants kept in shared memory (CS) instead of registers: the 9
// level / warp constants are re-read each cycle with ld.shared (volatile, so
// they are not hoisted back into registers), which removes the register
// spills of the 64-register (2 CTAs / SM) build.
FSB_INLINE double lds64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

template <int R, int TY, bool DIAG, bool CS, int MINB>
__global__ void __launch_bounds__(kTX * TY, MINB) k64_block(const B64 A) {
  constexpr int TW = kTX - 2 * R, TH = TY - 2 * R;
  extern __shared__ double s_dyn[];
  Tile64<TY>& S = *reinterpret_cast<Tile64<TY>*>(s_dyn);
  auto& s_ub = S.ub;
  auto& s_vb0 = S.vb0;
  auto& s_vb1 = S.vb1;
  auto& s_f = S.f;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int gx = (int)blockIdx.x * TW - R + tx, gy = (int)blockIdx.y * TH - R + ty;
  const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
  const size_t n = A.n;
  const size_t i = in ? (size_t)gy * A.w + gx : 0;
  // edge indicators (ex_at / ey_at of pd64.cu); zero outside the image
  const bool m = in && A.mask[i];
  const bool ex = m && gx + 1 < A.w && A.mask[i + 1];
  const bool ey = m && gy + 1 < A.h && A.mask[i + A.w];
  // Outside the solve mask the whole state is exactly zero for the level
  // (upsample_state zeroes u there, v / p / q start at 0, and with both edge
  // indicators false every update maps 0 to 0), and no masked pixel feeds an
  // unmasked one (its fluxes and the differences towards it are masked out).
  // So masked pixels neither load nor store; both state sets are zeroed at
  // the level start.
  double u = 0, ub = 0, v0 = 0, v1 = 0, vb0 = 0, vb1 = 0, p0 = 0, p1 = 0;
  double q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  double a = 0, b = 0, c = 0, sp = 0, tu = 0, tv = 0, g = 0, rh = 0, uo = 0;
  if (m) {
    u = A.su[i];
    v0 = A.sv[i]; v1 = A.sv[n + i];
    if (A.first) {
      ub = u; vb0 = v0; vb1 = v1; uo = u;
    } else {
      ub = A.sub[i]; vb0 = A.svb[i]; vb1 = A.svb[n + i]; uo = A.uo[i];
    }
    p0 = A.sp[i]; p1 = A.sp[n + i];
    q0 = A.sq[i]; q1 = A.sq[n + i]; q2 = A.sq[2 * n + i]; q3 = A.sq[3 * n + i];
    a = A.T[i]; b = A.T[n + i]; c = A.T[2 * n + i];
    sp = A.S[i] * A.alpha1; tu = A.S[n + i]; tv = A.S[2 * n + i];
    g = A.iu[i]; rh = A.rho0[i];
  }
  double* const sc = &S.c[0][ty][tx];
  constexpr int PL = kTX * TY;
  if (CS) {
    sc[0] = a; sc[PL] = b; sc[2 * PL] = c; sc[3 * PL] = sp; sc[4 * PL] = tu;
    sc[5 * PL] = tv; sc[6 * PL] = g; sc[7 * PL] = rh; sc[8 * PL] = uo;
  }
  const double sq = A.sigma_q * A.alpha0;
  const bool interior = tx >= R && tx < kTX - R && ty >= R && ty < TY - R && in;
  const int txr = tx + 1 < kTX ? tx + 1 : tx, tyd = ty + 1 < TY ? ty + 1 : ty;
  for (int it = 0; it < A.iters; ++it) {
    if (CS) { a = lds64(sc); b = lds64(sc + PL); c = lds64(sc + 2 * PL); sp = lds64(sc + 3 * PL); }
    s_ub[ty][tx] = ub;
    s_vb0[ty][tx] = vb0;
    s_vb1[ty][tx] = vb1;
    __syncthreads();
    // dual ascent (k64_dual): forward differences where the edge is in the mask
    double gxx = 0, gyy = 0, g00 = 0, g01 = 0, g10 = 0, g11 = 0;
    if (ex) { gxx = s_ub[ty][txr] - ub; g00 = s_vb0[ty][txr] - vb0; g10 = s_vb1[ty][txr] - vb1; }
    if (ey) { gyy = s_ub[tyd][tx] - ub; g01 = s_vb0[tyd][tx] - vb0; g11 = s_vb1[tyd][tx] - vb1; }
    dual_update_exact<double>(a, b, c, sp, sq, gxx, gyy, g00, g01, g10, g11, vb0, vb1, p0, p1,
                              q0, q1, q2, q3, A.heps);
    const FluxT<double> f = make_flux_exact<double>(a, b, c, ex, ey, p0, p1, q0, q1, q2, q3);
    s_f[0][ty][tx] = f.px; s_f[1][ty][tx] = f.py;
    s_f[2][ty][tx] = f.q0x; s_f[3][ty][tx] = f.q0y;
    s_f[4][ty][tx] = f.q1x; s_f[5][ty][tx] = f.q1y;
    if (DIAG) {
      double pn = 0, qn = 0;
      if (interior) {
        pn = sqrt(p0 * p0 + p1 * p1);
        qn = sqrt(((q0 * q0 + q1 * q1) + q2 * q2) + q3 * q3);
      }
      pn = warp_max(pn);
      qn = warp_max(qn);
      if (tx == 0 && A.diag_p) {  // one warp per tile row
        atomic_max_nonneg(A.diag_p + it, (float)pn);
        atomic_max_nonneg(A.diag_q + it, (float)qn);
      }
    }
    __syncthreads();
    // primal descent (k64_primal): backward divergence of the fluxes. The row
    // above / column left of the tile feed only halo pixels; outside the image
    // the fluxes are zero (mask 0), as the reference's zero padding.
    double flx = 0, flq0 = 0, flq1 = 0, fuy = 0, fuq0 = 0, fuq1 = 0;
    if (tx > 0) { flx = s_f[0][ty][tx - 1]; flq0 = s_f[2][ty][tx - 1]; flq1 = s_f[4][ty][tx - 1]; }
    if (ty > 0) { fuy = s_f[1][ty - 1][tx]; fuq0 = s_f[3][ty - 1][tx]; fuq1 = s_f[5][ty - 1][tx]; }
    const double dvv = ((f.px - flx) + f.py) - fuy;
    const double d0 = ((f.q0x - flq0) + f.q0y) - fuq0;
    const double d1 = ((f.q1x - flq1) + f.q1y) - fuq1;
    if (CS) {
      tu = lds64(sc + 4 * PL); tv = lds64(sc + 5 * PL); g = lds64(sc + 6 * PL);
      rh = lds64(sc + 7 * PL); uo = lds64(sc + 8 * PL);
    }
    primal_update_exact<double>(dvv, d0, d1, tu, tv, g, rh, uo, p0, p1, A.lam, A.alpha0,
                                A.alpha1, A.theta, u, v0, v1, ub, vb0, vb1);
  }
  if (A.fin) {  // k64_finish (solver.py:356-360) on the interior
    if (CS) uo = lds64(sc + 8 * PL);
    double adu = 0.0;
    if (interior && m) {  // masked pixels: du = 0, nothing changes
      double du = fmin(fmax(u - uo, -A.du_max), A.du_max);
      if (!m) du = 0.0;
      u = uo + du;
      ub = u;
      A.wv[2 * i] = A.wv[2 * i] + du * A.dirs[2 * i];
      A.wv[2 * i + 1] = A.wv[2 * i + 1] + du * A.dirs[2 * i + 1];
      adu = fabs(du);
    }
    if (DIAG && (A.diag_du || A.diag_du64)) {
      __shared__ double s_sum[TY], s_max[TY];
      const double mx = warp_max(adu), sm = warp_sum(adu);
      if (tx == 0) { s_sum[ty] = sm; s_max[ty] = mx; }
      __syncthreads();
      if (tx == 0 && ty == 0) {
        double t = 0.0, mm = 0.0;
        for (int k = 0; k < TY; ++k) { t += s_sum[k]; mm = fmax(mm, s_max[k]); }
        A.partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
        if (A.diag_du64) atomic_max_nonneg(A.diag_du64, mm);
        else atomic_max_nonneg(A.diag_du, (float)mm);
      }
    }
  }
  if (!interior || !m) return;
  if (A.first) A.uo[i] = CS ? lds64(sc + 8 * PL) : uo;
  A.du[i] = u; A.dub[i] = ub;
  A.dv[i] = v0; A.dv[n + i] = v1;
  A.dvb[i] = vb0; A.dvb[n + i] = vb1;
  A.dp[i] = p0; A.dp[n + i] = p1;
  A.dq[i] = q0; A.dq[n + i] = q1; A.dq[2 * n + i] = q2; A.dq[3 * n + i] = q3;
}

template <int R, int TY, bool DIAG, bool CS, int MINB>
int launch64v(const B64& A, cudaStream_t st) {
  constexpr int TW = kTX - 2 * R, TH = TY - 2 * R;
  const dim3 blk(kTX, TY), grd((A.w + TW - 1) / TW, (A.h + TH - 1) / TH);
  const size_t dyn = CS ? sizeof(Tile64<TY>) : offsetof(Tile64<TY>, c);
  static std::atomic<unsigned long long> attr{0};
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(k64_block<R, TY, DIAG, CS, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  });
  k64_block<R, TY, DIAG, CS, MINB><<<grd, blk, dyn, st>>>(A);
  return launch_status();
}

// Measured on C3 (fp64 frame): constants in shared memory 29.4 ms, in
// registers 31.2 ms; 32 x 32 tiles at one CTA / SM 32.0 ms; 32 x 16 tiles at
// one CTA / SM without spills 35.4 ms (occupancy matters more than spills).
bool pd64_const_regs() {
  static const bool v = [] {
    const char* e = getenv("FSB_PD64_CONST");
    return e && strcmp(e, "regs") == 0;
  }();
  return v;
}

template <int R>
int launch64(const B64& A, cudaStream_t st) {
  const bool diag = A.diag_p || A.diag_du || A.diag_du64;
  if (pd64_const_regs())  // FSB_PD64_CONST=regs: constants in registers (spills)
    return diag ? launch64v<R, kTY, true, false, 2>(A, st) : launch64v<R, kTY, false, false, 2>(A, st);
  return diag ? launch64v<R, kTY, true, true, 2>(A, st) : launch64v<R, kTY, false, true, 2>(A, st);
}

}  // namespace

size_t pd64_block_tiles(int w, int h, int halo) {
  const int TW = kTX - 2 * halo, TH = kTY - 2 * halo;
  return (size_t)((w + TW - 1) / TW) * ((h + TH - 1) / TH);
}

// `iters` (<= halo) cycles from the src set into the dst set.
int pd64_block_launch(const B64& A, int halo, cudaStream_t st) {
  if (A.iters < 1 || A.iters > halo) return FSB_EINVAL;
  switch (halo) {
    case 1: return launch64<1>(A, st);
    case 2: return launch64<2>(A, st);
    case 3: return launch64<3>(A, st);
    case 5: return launch64<5>(A, st);
    default: return FSB_EINVAL;
  }
}

}  // namespace fsb
