// Float64 warp prologue with NaN-encoded texels (the float64 path's
// solver.py:332-346 + image_derivative_along, solver.py:192-202).
//
// Per level, k64_pack folds the two gathered fields and their validity into
// one 32-byte texel per pixel: {mask ? I1 : NaN, traj_ok ? dx : NaN,
// traj_ok ? dy : NaN, 0}. A bicubic tap is then ONE 256-bit load
// (LDG.E.ENL2.256) that carries both fields and both validities, and the
// sampler needs no mask gathers and no all-16-valid flag array: the
// Catmull-Rom sums are formed unconditionally and a NaN sum means "some tap
// invalid" — exactly the reference's all-16-valid test (rasters.py:57-141),
// because the weights are finite. Only then does the fallback chain run
// (bilinear over the valid inner 2x2, renormalised; else the nearest valid tap,
// strict '<' in scan order), from the taps already in registers (the nearest
// tap is re-read in that rare case). The sampled image is written NaN-encoded
// (valid ? i1w : NaN), so the linearisation reads one double per tap and gets
// the validity of each tap (mask & i1w_ok) for free.
//
// Same operation order as the masked samplers (bicubic_bits): identical
// results. Compiled with -fmad=false like the other float64 samplers.
//
// Reference: solver.py:332-346, solver.py:192-202, rasters.py:57-141.

#include <math.h>
#include <stdint.h>
#include <stdlib.h>

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

namespace {

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

__global__ void k64_pack(const double* __restrict__ i1, const uint8_t* __restrict__ mask,
                         const double* __restrict__ traj, const uint8_t* __restrict__ tok,
                         size_t n, double4* __restrict__ tex) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const double2 t = reinterpret_cast<const double2*>(traj)[i];
  const bool ok = tok[i];
  tex[i] = make_double4(mask[i] ? i1[i] : nan, ok ? t.x : nan, ok ? t.y : nan, 0.0);
}

// solver.py:332-337: i1w = B(I1, x + w), dirs = B(traj, x + w) renormalised
// where valid and |dirs| > 0.5.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k64_sample_nan(P64 L) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const uint8_t mk = L.mask[i];
  const double2 wv = reinterpret_cast<const double2*>(L.wv)[i];
  if (!mk) {  // i1w_ok and dir_ok are false off the mask
    L.i1wn[i] = nan;
    reinterpret_cast<double2*>(L.dirs)[i] = make_double2(0.0, 0.0);
    L.dir_ok[i] = 0;
    return;
  }
  int ix, iy;
  double fx, fy;
  double iv = 0.0, d0 = 0.0, d1 = 0.0;
  bool wok = false, dok = false;
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
  L.i1wn[i] = wok ? iv : nan;
  reinterpret_cast<double2*>(L.dirs)[i] = make_double2(d0, d1);
  L.dir_ok[i] = dok;
}

// solver.py:339-343 + image_derivative_along (solver.py:192-202):
// I_u = B(i1w, x + dirs; mask & i1w_ok) - i1w, rho0 = i1w - I0 where data_ok.
__global__ void k64_linearize_nan(P64 L) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  const double i1w = L.i1wn[i], i0 = L.i0[i];
  const double2 dv = reinterpret_cast<const double2*>(L.dirs)[i];
  const bool ok0 = !isnan(i1w) && L.dir_ok[i];
  bool data_ok = false;
  double ahead = 0.0;
  int ix, iy;
  double fx, fy;
  if (ok0 && split_pos<double>((double)x + dv.x, (double)y + dv.y, L.h, L.w, ix, iy, fx, fy)) {
    const bool inner = ix >= 1 && ix + 2 < L.w && iy >= 1 && iy + 2 < L.h;
    double wx[4], wy[4];
    cubic_weights(fx, wx);
    cubic_weights(fy, wy);
    double s = 0.0, in4[4][1];
    unsigned okb = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int r = iy + a - 1, c = ix + b - 1;
        double t = __longlong_as_double(0x7ff8000000000000LL);
        if (inner || ((unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w))
          t = __ldg(L.i1wn + (size_t)r * L.w + c);
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
                  : L.i1wn[(size_t)(iy + (best >> 2) - 1) * L.w + (ix + (best & 3) - 1)];
    }
  }
  L.iu[i] = data_ok ? ahead - i1w : 0.0;
  L.rho0[i] = data_ok ? i1w - i0 : 0.0;
}

}  // namespace

int pack64_internal(const double* i1, const uint8_t* mask, const double* traj,
                    const uint8_t* tok, int h, int w, double4* tex, cudaStream_t st) {
  const size_t n = (size_t)h * w;
  k64_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(i1, mask, traj, tok, n, tex);
  return launch_status();
}

int sample_nan64_internal(const P64& L, int bx, int by, cudaStream_t st) {
  const dim3 b(bx, by), g((L.w + bx - 1) / bx, (L.h + by - 1) / by);
  static const int minb = [] {
    const char* e = getenv("FSB_S64_MINB");
    return e ? atoi(e) : 2;
  }();
  if (minb >= 4) k64_sample_nan<4><<<g, b, 0, st>>>(L);
  else if (minb == 3) k64_sample_nan<3><<<g, b, 0, st>>>(L);
  else k64_sample_nan<2><<<g, b, 0, st>>>(L);
  return launch_status();
}

int linearize_nan64_internal(const P64& L, int bx, int by, cudaStream_t st) {
  const dim3 b(bx, by), g((L.w + bx - 1) / bx, (L.h + by - 1) / by);
  k64_linearize_nan<<<g, b, 0, st>>>(L);
  return launch_status();
}

}  // namespace fsb
