// K4: per-level solver setup — normalised Gaussian smoothing, edge tensor T,
// diagonal preconditioner steps. Runs once per pyramid level; fp64 compute
// (compiled with -fmad=false), fp32 storage of T and the steps.
//
// Reference: rasters.py:185-191 (smooth_masked via scipy.ndimage.gaussian_filter),
// solver.py:122-161 (compute_tensor, _central_gradient), solver.py:246-276
// (precondition_steps).
//
// scipy.ndimage.gaussian_filter (SciPy >= 1.10, 1.18.1 in this image) is
// restated here: weights exp(-x^2 / (2 sigma^2)) / sum over x in [-r, r],
// r = int(4 sigma + 0.5) (truncate=4); separable correlation along axis 0 then
// axis 1; mode 'reflect' = half-sample symmetric extension; per output the
// symmetric-kernel accumulation of ni_filters.c: c*w0 then (a[-j]+a[j])*w[j]
// for j = r..1.

#include <math.h>

#include "fsb_common.cuh"

namespace fsb {
namespace {

constexpr int kBX = 32, kBY = 8;
constexpr int kMaxRadius = 32;

struct Gauss {
  int radius;
  double w[kMaxRadius + 1];  // w[j] for |x| = j
};

// numpy pairwise sum for n < 128 (8 interleaved accumulators), as phi.sum().
double np_sum(const double* a, int n) {
  if (n < 8) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i];
    return s;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

bool make_gauss(double sigma, Gauss& g) {
  int radius = (int)(4.0 * sigma + 0.5);
  if (radius > kMaxRadius || radius < 0 || !(sigma > 0)) return false;
  double phi[2 * kMaxRadius + 1];
  double sigma2 = sigma * sigma;
  double a = -0.5 / sigma2;
  for (int i = 0; i < 2 * radius + 1; ++i) {
    double x = (double)(i - radius);
    phi[i] = exp(a * (x * x));
  }
  double s = np_sum(phi, 2 * radius + 1);
  g.radius = radius;
  for (int j = 0; j <= radius; ++j) g.w[j] = phi[radius + j] / s;
  return true;
}

__device__ __forceinline__ int reflect_idx(int i, int n) {
  if (n == 1) return 0;
  int period = 2 * n;
  i %= period;
  if (i < 0) i += period;
  return i < n ? i : period - 1 - i;
}

// axis-0 pass on (f*m, m): out[2*i] = num, out[2*i+1] = den
template <typename TI>
__global__ void k_gauss_rows(const TI* __restrict__ f, const uint8_t* __restrict__ m, int h,
                             int w, Gauss g, double* __restrict__ out) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  auto fm = [&](int yy) {
    size_t k = (size_t)yy * w + x;
    return (double)f[k] * (m[k] ? 1.0 : 0.0);
  };
  auto mm = [&](int yy) { return m[(size_t)yy * w + x] ? 1.0 : 0.0; };
  double num = fm(y) * g.w[0];
  double den = mm(y) * g.w[0];
  for (int j = g.radius; j >= 1; --j) {
    int a = reflect_idx(y - j, h), b = reflect_idx(y + j, h);
    num += (fm(a) + fm(b)) * g.w[j];
    den += (mm(a) + mm(b)) * g.w[j];
  }
  size_t i = (size_t)y * w + x;
  out[2 * i] = num;
  out[2 * i + 1] = den;
}

// axis-1 pass + normalisation (rasters.py:188-190) -> smoothed image (f64)
__global__ void k_gauss_cols(const double* __restrict__ nd, const uint8_t* __restrict__ m, int h,
                             int w, Gauss g, double* __restrict__ sm) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const double* row = nd + 2 * (size_t)y * w;
  double num = row[2 * x] * g.w[0];
  double den = row[2 * x + 1] * g.w[0];
  for (int j = g.radius; j >= 1; --j) {
    int a = reflect_idx(x - j, w), b = reflect_idx(x + j, w);
    num += (row[2 * a] + row[2 * b]) * g.w[j];
    den += (row[2 * a + 1] + row[2 * b + 1]) * g.w[j];
  }
  size_t i = (size_t)y * w + x;
  sm[i] = m[i] ? num / fmax(den, 1e-12) : 0.0;
}

__device__ __forceinline__ bool edge_x(const uint8_t* m, int w, int x, size_t i) {
  return x + 1 < w && m[i] && m[i + 1];
}
__device__ __forceinline__ bool edge_y(const uint8_t* m, int h, int y, int w, size_t i) {
  return y + 1 < h && m[i] && m[i + w];
}

// compute_tensor (solver.py:122-161) on the smoothed image; tensor in f64
// scratch (3 per pixel) and f32 planes.
template <typename TO>
__global__ void k_tensor(const double* __restrict__ sm, const uint8_t* __restrict__ m, int h, int w,
                         double beta, double eta, double* __restrict__ t64,
                         TO* __restrict__ t32) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  size_t i = (size_t)y * w + x;
  size_t n = (size_t)h * w;
  double a = 1.0, b = 0.0, c = 1.0;
  if (m[i]) {
    // _central_gradient: average of the valid forward edges at x and x-1
    bool ex = edge_x(m, w, x, i), exl = x > 0 && edge_x(m, w, x - 1, i - 1);
    bool ey = edge_y(m, h, y, w, i), eyu = y > 0 && edge_y(m, h, y - 1, w, i - w);
    double dx = ex ? (sm[i + 1] - sm[i]) : 0.0;
    double dxl = exl ? (sm[i] - sm[i - 1]) : 0.0;
    double dy = ey ? (sm[i + w] - sm[i]) : 0.0;
    double dyu = eyu ? (sm[i] - sm[i - w]) : 0.0;
    double gx = dx, gy = dy, nx = ex ? 1.0 : 0.0, ny = ey ? 1.0 : 0.0;
    if (x > 0) { gx = gx + dxl; nx = nx + (exl ? 1.0 : 0.0); }
    if (y > 0) { gy = gy + dyu; ny = ny + (eyu ? 1.0 : 0.0); }
    gx = gx / fmax(nx, 1.0);
    gy = gy / fmax(ny, 1.0);
    double mag = hypot(gx, gy);
    double safe = fmax(mag, 1e-300);
    double ux = mag > 1e-12 ? gx / safe : 1.0;
    double uy = mag > 1e-12 ? gy / safe : 0.0;
    double lam_n = exp(-beta * pow(mag, eta));
    a = (lam_n * ux) * ux + uy * uy;
    b = ((lam_n - 1.0) * ux) * uy;
    c = (lam_n * uy) * uy + ux * ux;
  }
  t64[3 * i] = a; t64[3 * i + 1] = b; t64[3 * i + 2] = c;
  t32[i] = (TO)a; t32[n + i] = (TO)b; t32[2 * n + i] = (TO)c;
}

// precondition_steps (solver.py:246-276)
template <typename TO>
__global__ void k_steps(const double* __restrict__ t64, const uint8_t* __restrict__ m, int h, int w,
                        double alpha0, double alpha1, bool tgv, TO* __restrict__ steps) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  size_t i = (size_t)y * w + x;
  size_t n = (size_t)h * w;
  double a = fabs(t64[3 * i]), b = fabs(t64[3 * i + 1]), c = fabs(t64[3 * i + 2]);
  double exf = edge_x(m, w, x, i) ? 1.0 : 0.0;
  double eyf = edge_y(m, h, y, w, i) ? 1.0 : 0.0;
  double row_px = ((2.0 * a) * exf + (2.0 * b) * eyf) + 1.0;
  double row_py = ((2.0 * b) * exf + (2.0 * c) * eyf) + 1.0;
  double sigma_p = 1.0 / (alpha1 * fmax(row_px, row_py));
  double col_u = (a + b) * exf + (b + c) * eyf;
  double ecount = exf + eyf;
  if (x > 0) {
    size_t l = i - 1;
    double al = fabs(t64[3 * l]), bl = fabs(t64[3 * l + 1]);
    double exl = edge_x(m, w, x - 1, l) ? 1.0 : 0.0;
    col_u = col_u + (al + bl) * exl;
    ecount = ecount + exl;
  }
  if (y > 0) {
    size_t u = i - w;
    double bu = fabs(t64[3 * u + 1]), cu = fabs(t64[3 * u + 2]);
    double eyu = edge_y(m, h, y - 1, w, u) ? 1.0 : 0.0;
    col_u = col_u + (bu + cu) * eyu;
    ecount = ecount + eyu;
  }
  double tau_u = 1.0 / fmax(alpha1 * col_u, 1e-12);
  double tau_v = tgv ? 1.0 / (alpha1 + alpha0 * ecount) : 0.0;  // TV / Huber: v held at 0
  steps[i] = (TO)sigma_p;
  steps[n + i] = (TO)tau_u;
  steps[2 * n + i] = (TO)tau_v;
}

__global__ void k_planes_to_t64(const float* __restrict__ t32, size_t n, double* __restrict__ t64) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    t64[3 * i] = t32[i];
    t64[3 * i + 1] = t32[n + i];
    t64[3 * i + 2] = t32[2 * n + i];
  }
}

__global__ void k_f32_to_f64(const float* __restrict__ a, size_t n, double* __restrict__ o) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = (double)a[i];
}

__global__ void k_to_f32(const double* __restrict__ a, size_t n, float* __restrict__ o) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = (float)a[i];
}

size_t smooth_bytes(int h, int w) {
  size_t n = (size_t)h * w;
  return align_up(n * 2 * sizeof(double)) + align_up(n * sizeof(double)) +
         align_up(n * 3 * sizeof(double));
}

}  // namespace

size_t level_setup_scratch_internal(int h, int w) { return smooth_bytes(h, w); }

template <typename T>
int level_setup_t(const T* i0, const uint8_t* mask, int h, int w, const fsb_params* prm,
                  T* tensor, T* steps, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (!prm || !scratch) return FSB_EINVAL;
  if (scratch_bytes < smooth_bytes(h, w)) return FSB_ENOSPC;
  Gauss g;
  if (!make_gauss(prm->tensor_sigma, g)) return FSB_EINVAL;
  size_t n = (size_t)h * w;
  char* p = static_cast<char*>(scratch);
  double* nd = reinterpret_cast<double*>(p); p += align_up(n * 2 * sizeof(double));
  double* sm = reinterpret_cast<double*>(p); p += align_up(n * sizeof(double));
  double* t64 = reinterpret_cast<double*>(p);
  dim3 blk(kBX, kBY), grd = grid2d(w, h, blk);
  k_gauss_rows<T><<<grd, blk, 0, st>>>(i0, mask, h, w, g, nd);
  k_gauss_cols<<<grd, blk, 0, st>>>(nd, mask, h, w, g, sm);
  k_tensor<T><<<grd, blk, 0, st>>>(sm, mask, h, w, prm->beta, prm->eta, t64, tensor);
  k_steps<T><<<grd, blk, 0, st>>>(t64, mask, h, w, prm->alpha0, prm->alpha1,
                                  prm->regularizer == FSB_REG_TGV, steps);
  return launch_status();
}

int level_setup_internal(const fsb_level* lv, const fsb_params* prm, void* scratch,
                         size_t scratch_bytes, cudaStream_t st) {
  if (!lv) return FSB_EINVAL;
  return level_setup_t<float>(lv->i0, lv->mask, lv->h, lv->w, prm, lv->tensor, lv->steps, scratch,
                              scratch_bytes, st);
}

int level_setup64_internal(const double* i0, const uint8_t* mask, int h, int w,
                           const fsb_params* prm, double* tensor, double* steps, void* scratch,
                           size_t scratch_bytes, cudaStream_t st) {
  return level_setup_t<double>(i0, mask, h, w, prm, tensor, steps, scratch, scratch_bytes, st);
}

}  // namespace fsb

using namespace fsb;

extern "C" {

size_t fsb_smooth_scratch_bytes(int32_t h, int32_t w) { return smooth_bytes(h, w); }

int fsb_smooth_masked(const float* f, const uint8_t* mask, int32_t h, int32_t w, double sigma,
                      float* out, void* scratch, size_t scratch_bytes, void* stream) {
  if (h < 1 || w < 1 || !f || !mask || !out || !scratch) return FSB_EINVAL;
  if (scratch_bytes < smooth_bytes(h, w)) return FSB_ENOSPC;
  Gauss g;
  if (!make_gauss(sigma, g)) return FSB_EINVAL;
  cudaStream_t st = as_stream(stream);
  size_t n = (size_t)h * w;
  char* p = static_cast<char*>(scratch);
  double* nd = reinterpret_cast<double*>(p); p += align_up(n * 2 * sizeof(double));
  double* sm = reinterpret_cast<double*>(p);
  dim3 blk(kBX, kBY), grd = grid2d(w, h, blk);
  k_gauss_rows<float><<<grd, blk, 0, st>>>(f, mask, h, w, g, nd);
  k_gauss_cols<<<grd, blk, 0, st>>>(nd, mask, h, w, g, sm);
  k_to_f32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sm, n, out);
  return launch_status();
}

int fsb_compute_tensor(const float* smoothed, const uint8_t* mask, int32_t h, int32_t w,
                       double beta, double eta, float* tensor, void* scratch,
                       size_t scratch_bytes, void* stream) {
  if (h < 1 || w < 1 || !smoothed || !mask || !tensor || !scratch) return FSB_EINVAL;
  size_t n = (size_t)h * w;
  if (scratch_bytes < align_up(n * sizeof(double)) + align_up(n * 3 * sizeof(double)))
    return FSB_ENOSPC;
  cudaStream_t st = as_stream(stream);
  double* sm = static_cast<double*>(scratch);
  double* t64 = reinterpret_cast<double*>(static_cast<char*>(scratch) + align_up(n * sizeof(double)));
  k_f32_to_f64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(smoothed, n, sm);
  dim3 blk(kBX, kBY), grd = grid2d(w, h, blk);
  k_tensor<float><<<grd, blk, 0, st>>>(sm, mask, h, w, beta, eta, t64, tensor);
  return launch_status();
}

int fsb_precondition_steps(const float* tensor, const uint8_t* mask, int32_t h, int32_t w,
                           const fsb_params* prm, float* steps, void* scratch,
                           size_t scratch_bytes, void* stream) {
  if (h < 1 || w < 1 || !tensor || !mask || !steps || !scratch || !prm) return FSB_EINVAL;
  size_t n = (size_t)h * w;
  if (scratch_bytes < n * 3 * sizeof(double)) return FSB_ENOSPC;
  cudaStream_t st = as_stream(stream);
  double* t64 = static_cast<double*>(scratch);
  k_planes_to_t64<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(tensor, n, t64);
  dim3 blk(kBX, kBY), grd = grid2d(w, h, blk);
  k_steps<<<grd, blk, 0, st>>>(t64, mask, h, w, prm->alpha0, prm->alpha1,
                               prm->regularizer == FSB_REG_TGV, steps);
  return launch_status();
}


}  // extern "C"
