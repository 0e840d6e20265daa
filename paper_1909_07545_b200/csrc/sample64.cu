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

#include "sample64.cuh"

namespace fsb {

namespace {

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
  double iwn, d0, d1;
  bool dok;
  sample_nan_px(L, x, y, wv, iwn, d0, d1, dok);
  L.i1wn[i] = iwn;
  reinterpret_cast<double2*>(L.dirs)[i] = make_double2(d0, d1);
  L.dir_ok[i] = dok;
}

// solver.py:339-343 + image_derivative_along (solver.py:192-202):
// I_u = B(i1w, x + dirs; mask & i1w_ok) - i1w, rho0 = i1w - I0 where data_ok.
__global__ void k64_linearize_nan(P64 L) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.w || y >= L.h) return;
  const size_t i = (size_t)y * L.w + x;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  auto tap = [&](int r, int c) {
    return ((unsigned)r < (unsigned)L.h && (unsigned)c < (unsigned)L.w)
               ? __ldg(L.i1wn + (size_t)r * L.w + c)
               : nan;
  };
  linearize_nan_px(L, x, y, L.i1wn[i], L.i0[i], reinterpret_cast<const double2*>(L.dirs)[i],
                   L.dir_ok[i], tap, L.iu[i], L.rho0[i]);
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
