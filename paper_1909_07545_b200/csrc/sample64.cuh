// The float64 path's NaN-texel warp prologue for one pixel (levels <= 256^2):
// the level buffers (P64) and the per-pixel sampling / linearisation shared by
// the standalone kernels (sample64.cu, -fmad=false: NumPy's rounding) and the
// whole-level kernel k64_level (pd64_level.cu, FMA contraction on: ~1 ulp
// differences, far inside the parity gates; tests/test_gpu_variants.py).
//
// Reference: solver.py:332-346, solver.py:192-202, rasters.py:57-141.
#pragma once

#include <math.h>
#include <stdint.h>

#include "fsb_common.cuh"

namespace fsb {

struct P64 {  // one level's prologue buffers
  int h, w;
  const double* i0;
  const uint8_t* mask;
  const double4* tex;  // packed texels (k64_pack)
  const double* wv;    // (h, w, 2) warp
  double* i1wn;        // sampled image, NaN where invalid
  double* dirs;        // (h, w, 2) unit directions, 0 where invalid
  uint8_t* dir_ok;
  double* iu;
  double* rho0;
};


FSB_INLINE double4 ld256(const double4* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}

// Fallback of bicubic_bits from registers: bilinear over the valid inner 2x2
// (in4[k] = tap (1 + k/2, 1 + k%2)), renormalised; else the index of the
// nearest valid tap in *best (value read by the caller). okb != 0, != 0xFFFF.
template <int C>
FSB_INLINE bool fallback_bilinear(unsigned okb, const double in4[4][C], double fx, double fy,
                                  double out[C], int* best) {
  const double bx[2] = {1.0 - fx, fx};
  const double by[2] = {1.0 - fy, fy};
  double bil[C];
#pragma unroll
  for (int k = 0; k < C; ++k) bil[k] = 0.0;
  double bws = 0.0;
#pragma unroll
  for (int a = 1; a <= 2; ++a)
#pragma unroll
    for (int b = 1; b <= 2; ++b)
      if (okb >> (4 * a + b) & 1u) {
        const double bw = by[a - 1] * bx[b - 1];
#pragma unroll
        for (int k = 0; k < C; ++k) bil[k] = tap_acc(bil[k], bw, in4[2 * (a - 1) + (b - 1)][k]);
        bws += bw;
      }
  if (bws > 1e-12) {
#pragma unroll
    for (int k = 0; k < C; ++k) out[k] = bil[k] / bws;
    return true;
  }
  double nd2 = INFINITY;
  int bi = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (okb >> (4 * a + b) & 1u) {
        const double d2 = dist2(double(b - 1) - fx, double(a - 1) - fy);
        if (d2 < nd2) { nd2 = d2; bi = 4 * a + b; }
      }
  *best = bi;
  return false;
}

// solver.py:332-337 for one in-image mask pixel (w loaded by the caller): the
// NaN-encoded i1w value (NaN where invalid) and the unit direction with its flag.
FSB_INLINE void sample_nan_px(const P64& L, int x, int y, double2 wv, double& iwn, double& d0,
                              double& d1, bool& dok_out) {
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  double iv = 0.0;
  bool wok = false, dok = false;
  d0 = 0.0;
  d1 = 0.0;
  int ix, iy;
  double fx, fy;
  if (split_pos<double>((double)x + wv.x, (double)y + wv.y, L.h, L.w, ix, iy, fx, fy)) {
    const bool inner = ix >= 1 && ix + 2 < L.w && iy >= 1 && iy + 2 < L.h;
    double wx[4], wy[4];
    cubic_weights(fx, wx);
    cubic_weights(fy, wy);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    unsigned oki = 0, okt = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int r = iy + a - 1, c = ix + b - 1;
        double4 t = make_double4(nan, nan, nan, 0.0);
        if (inner || ((unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w))
          t = ld256(L.tex + (size_t)r * L.w + c);
        const double wt = wy[a] * wx[b];
        s0 = tap_acc(s0, wt, t.x);
        s1 = tap_acc(s1, wt, t.y);
        s2 = tap_acc(s2, wt, t.z);
        oki |= (isnan(t.x) ? 0u : 1u) << (4 * a + b);
        okt |= (isnan(t.y) ? 0u : 1u) << (4 * a + b);
      }
    // fallback (some tap invalid, rare): the inner 2x2 again (L1-resident)
    double in_i[4][1], in_t[4][2];
    if ((oki != 0xFFFFu && oki) || (okt != 0xFFFFu && okt)) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = iy + (k >> 1), c = ix + (k & 1);
        double4 t = make_double4(nan, nan, nan, 0.0);
        if ((unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w)
          t = ld256(L.tex + (size_t)r * L.w + c);
        in_i[k][0] = t.x;
        in_t[k][0] = t.y;
        in_t[k][1] = t.z;
      }
    }
    if (oki == 0xFFFFu) {
      iv = s0;
      wok = true;
    } else if (oki) {
      int best = 0;
      double o[1];
      wok = true;
      if (fallback_bilinear<1>(oki, in_i, fx, fy, o, &best)) {
        iv = o[0];
      } else {
        iv = ld256(L.tex + (size_t)(iy + (best >> 2) - 1) * L.w + (ix + (best & 3) - 1)).x;
      }
    }
    double dr[2] = {s1, s2};
    if (okt == 0xFFFFu) {
      dok = true;
    } else if (okt) {
      int best = 0;
      dok = true;
      if (!fallback_bilinear<2>(okt, in_t, fx, fy, dr, &best)) {
        const double4 t =
            ld256(L.tex + (size_t)(iy + (best >> 2) - 1) * L.w + (ix + (best & 3) - 1));
        dr[0] = t.y;
        dr[1] = t.z;
      }
    }
    if (dok) {
      const double nrm = sqrt(dr[0] * dr[0] + dr[1] * dr[1]);
      if (nrm > 0.5) {
        d0 = dr[0] / fmax(nrm, 1e-300);
        d1 = dr[1] / fmax(nrm, 1e-300);
      } else {
        dok = false;
      }
    }
  }
  iwn = wok ? iv : nan;
  dok_out = dok;
}

// solver.py:339-343 + image_derivative_along (solver.py:192-202) for one pixel
// from its own sampled value / direction and a tap source tap(r, c) -> the
// NaN-encoded i1w there (NaN outside the image): I_u = B(i1w, x + dirs; mask &
// i1w_ok) - i1w, rho0 = i1w - I0 where data_ok, else 0.
template <class Tap>
FSB_INLINE void linearize_nan_px(const P64& L, int x, int y, double i1w, double i0, double2 dv,
                                 bool dok, Tap tap, double& iu, double& rho0) {
  const bool ok0 = !isnan(i1w) && dok;
  bool data_ok = false;
  double ahead = 0.0;
  int ix, iy;
  double fx, fy;
  if (ok0 && split_pos<double>((double)x + dv.x, (double)y + dv.y, L.h, L.w, ix, iy, fx, fy)) {
    double wx[4], wy[4];
    cubic_weights(fx, wx);
    cubic_weights(fy, wy);
    double s = 0.0, in4[4][1];
    unsigned okb = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double t = tap(iy + a - 1, ix + b - 1);
        s = tap_acc(s, wy[a] * wx[b], t);
        okb |= (isnan(t) ? 0u : 1u) << (4 * a + b);
        if (a >= 1 && a <= 2 && b >= 1 && b <= 2) in4[2 * (a - 1) + (b - 1)][0] = t;
      }
    if (okb == 0xFFFFu) {
      ahead = s;
      data_ok = true;
    } else if (okb) {
      int best = 0;
      double o[1];
      data_ok = true;
      ahead = fallback_bilinear<1>(okb, in4, fx, fy, o, &best)
                  ? o[0]
                  : tap(iy + (best >> 2) - 1, ix + (best & 3) - 1);
    }
  }
  iu = data_ok ? ahead - i1w : 0.0;
  rho0 = data_ok ? i1w - i0 : 0.0;
}

}  // namespace fsb
