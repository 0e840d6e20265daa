// K3 / K7 and the raster primitives: generic masked bicubic sampling, forward
// gradient / backward divergence, pyramid shapes, masked area downsampling,
// state upsampling. Compiled with -fmad=false (fp64 accumulation where the
// reference's order matters).
//
// Reference: rasters.py:57-297.

#include "fsb_common.cuh"

namespace fsb {
namespace {

constexpr int kBX = 32, kBY = 8;

template <int C>
__global__ void k_sample_pts(const float* __restrict__ field, int h, int w,
                             const uint8_t* __restrict__ mask, const double* __restrict__ pos,
                             int64_t n, float* __restrict__ out, uint8_t* __restrict__ valid,
                             bool acc64) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = pos[2 * i], y = pos[2 * i + 1];
  bool ok;
  float r[C];
  if (acc64) {
    double v[C];
    ok = bicubic_sample<C, double>(field, mask, h, w, x, y, v);
#pragma unroll
    for (int k = 0; k < C; ++k) r[k] = (float)v[k];
  } else {
    float v[C];
    ok = bicubic_sample<C, float>(field, mask, h, w, x, y, v);
#pragma unroll
    for (int k = 0; k < C; ++k) r[k] = v[k];
  }
#pragma unroll
  for (int k = 0; k < C; ++k) out[C * i + k] = ok ? r[k] : NAN;
  valid[i] = ok;
}

// gradient (rasters.py:144-155)
__global__ void k_gradient(const float* __restrict__ u, const uint8_t* __restrict__ m, int h, int w,
                           float* __restrict__ g) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  size_t i = (size_t)y * w + x;
  bool ex = x + 1 < w && m[i] && m[i + 1];
  bool ey = y + 1 < h && m[i] && m[i + w];
  g[2 * i] = ex ? u[i + 1] - u[i] : 0.f;
  g[2 * i + 1] = ey ? u[i + w] - u[i] : 0.f;
}

// divergence (rasters.py:158-172)
__global__ void k_divergence(const float* __restrict__ p, const uint8_t* __restrict__ m, int h,
                             int w, float* __restrict__ d) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  size_t i = (size_t)y * w + x;
  auto ex = [&](int xx, size_t j) { return xx + 1 < w && m[j] && m[j + 1]; };
  auto ey = [&](int yy, size_t j) { return yy + 1 < h && m[j] && m[j + w]; };
  float px = ex(x, i) ? p[2 * i] : 0.f;
  float py = ey(y, i) ? p[2 * i + 1] : 0.f;
  float pxl = (x > 0 && ex(x - 1, i - 1)) ? p[2 * (i - 1)] : 0.f;
  float pyu = (y > 0 && ey(y - 1, i - w)) ? p[2 * (i - w) + 1] : 0.f;
  float dv = px;
  if (x > 0) dv = dv - pxl;
  dv = dv + py;
  if (y > 0) dv = dv - pyu;
  d[i] = dv;
}

// downsample_area (rasters.py:224-260): fine pixels binned by (i*nc)//nf,
// summed in fine raster order (np.bincount), mask from the nearest fine sample.
template <typename T>
__global__ void k_downsample(const T* __restrict__ src, const uint8_t* __restrict__ mask,
                             int fh, int fw, T* __restrict__ dst, uint8_t* __restrict__ dmask,
                             int ch, int cw) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (j >= cw || i >= ch) return;
  int r0 = (int)(((int64_t)i * fh + ch - 1) / ch), r1 = (int)(((int64_t)(i + 1) * fh + ch - 1) / ch);
  int c0 = (int)(((int64_t)j * fw + cw - 1) / cw), c1 = (int)(((int64_t)(j + 1) * fw + cw - 1) / cw);
  double s = 0.0, cnt = 0.0;
  for (int r = r0; r < r1; ++r)
    for (int c = c0; c < c1; ++c) {
      size_t k = (size_t)r * fw + c;
      double mk = mask[k] ? 1.0 : 0.0;
      s += (double)src[k] * mk;
      cnt += mk;
    }
  double avg = s / fmax(cnt, 1.0);
  int rr = (int)rint(((i + 0.5) * fh) / ch - 0.5);
  int cc = (int)rint(((j + 0.5) * fw) / cw - 0.5);
  rr = min(max(rr, 0), fh - 1);
  cc = min(max(cc, 0), fw - 1);
  bool cm = mask[(size_t)rr * fw + cc] && cnt > 0.0;
  size_t o = (size_t)i * cw + j;
  dst[o] = cm ? (T)avg : T(0);
  dmask[o] = cm;
}

// upsample_state (rasters.py:276-297), f64 taps/accumulation.
template <typename T>
__global__ void k_upsample(const T* __restrict__ u, const T* __restrict__ wv,
                           const uint8_t* __restrict__ mask, int sh, int sw,
                           const uint8_t* __restrict__ dmask, int dh, int dw, double sx, double sy,
                           T* __restrict__ uo, T* __restrict__ wo) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= dw || y >= dh) return;
  double px = (x + 0.5) / sx - 0.5, py = (y + 0.5) / sy - 0.5;
  double us[1], ws[2];
  bool ok = bicubic_sample<1, double, T>(u, mask, sh, sw, px, py, us);
  ok = bicubic_sample<2, double, T>(wv, mask, sh, sw, px, py, ws) && ok;
  size_t i = (size_t)y * dw + x;
  bool keep = ok && dmask[i];
  uo[i] = (T)((keep ? us[0] : 0.0) * (0.5 * (sx + sy)));
  wo[2 * i] = (T)((keep ? ws[0] : 0.0) * sx);
  wo[2 * i + 1] = (T)((keep ? ws[1] : 0.0) * sy);
}

}  // namespace

int pyramid_shapes_internal(int h, int w, int levels, double scale, int min_width, int* shapes,
                            int max_levels) {
  if (levels < 1 || !(scale > 1.0) || h < 1 || w < 1) return FSB_EINVAL;
  int n = 0;
  int ch = h, cw = w;
  if (n < max_levels) { shapes[2 * n] = ch; shapes[2 * n + 1] = cw; }
  n = 1;
  while (n < levels) {
    int nh = (int)ceil((double)ch / scale), nw = (int)ceil((double)cw / scale);
    if (nw < min_width) break;
    ch = nh; cw = nw;
    if (n < max_levels) { shapes[2 * n] = ch; shapes[2 * n + 1] = cw; }
    ++n;
  }
  return n;
}

template <typename T>
int downsample_t(const T* src, const uint8_t* mask, int fh, int fw, T* dst, uint8_t* dmask, int ch,
                 int cw, cudaStream_t st) {
  dim3 blk(kBX, kBY);
  k_downsample<T><<<grid2d(cw, ch, blk), blk, 0, st>>>(src, mask, fh, fw, dst, dmask, ch, cw);
  return launch_status();
}

template <typename T>
int upsample_t(const T* u, const T* wv, const uint8_t* mask, int sh, int sw, const uint8_t* dmask,
               int dh, int dw, T* uo, T* wo, cudaStream_t st) {
  double sx = (double)dw / (double)sw, sy = (double)dh / (double)sh;
  dim3 blk(kBX, kBY);
  k_upsample<T><<<grid2d(dw, dh, blk), blk, 0, st>>>(u, wv, mask, sh, sw, dmask, dh, dw, sx, sy,
                                                     uo, wo);
  return launch_status();
}

int downsample_internal(const float* src, const uint8_t* mask, int fh, int fw, float* dst,
                        uint8_t* dmask, int ch, int cw, cudaStream_t st) {
  return downsample_t<float>(src, mask, fh, fw, dst, dmask, ch, cw, st);
}
int downsample64_internal(const double* src, const uint8_t* mask, int fh, int fw, double* dst,
                          uint8_t* dmask, int ch, int cw, cudaStream_t st) {
  return downsample_t<double>(src, mask, fh, fw, dst, dmask, ch, cw, st);
}
int upsample_internal(const float* u, const float* wv, const uint8_t* mask, int sh, int sw,
                      const uint8_t* dmask, int dh, int dw, float* uo, float* wo, cudaStream_t st) {
  return upsample_t<float>(u, wv, mask, sh, sw, dmask, dh, dw, uo, wo, st);
}
int upsample64_internal(const double* u, const double* wv, const uint8_t* mask, int sh, int sw,
                        const uint8_t* dmask, int dh, int dw, double* uo, double* wo,
                        cudaStream_t st) {
  return upsample_t<double>(u, wv, mask, sh, sw, dmask, dh, dw, uo, wo, st);
}

}  // namespace fsb

using namespace fsb;

extern "C" {

int fsb_sample_bicubic(const float* field, int32_t h, int32_t w, int32_t c, const uint8_t* mask,
                       const double* pos, int64_t n, float* out, uint8_t* valid, int32_t acc64,
                       void* stream) {
  if (h < 1 || w < 1 || (c != 1 && c != 2) || n < 0) return FSB_EINVAL;
  if (n == 0) return FSB_OK;
  if (!field || !mask || !pos || !out || !valid) return FSB_EINVAL;
  int threads = 128;
  unsigned blocks = (unsigned)((n + threads - 1) / threads);
  cudaStream_t st = as_stream(stream);
  if (c == 1)
    k_sample_pts<1><<<blocks, threads, 0, st>>>(field, h, w, mask, pos, n, out, valid, acc64 != 0);
  else
    k_sample_pts<2><<<blocks, threads, 0, st>>>(field, h, w, mask, pos, n, out, valid, acc64 != 0);
  return launch_status();
}

int fsb_gradient(const float* u, const uint8_t* mask, int32_t h, int32_t w, float* g,
                 void* stream) {
  if (h < 1 || w < 1 || !u || !mask || !g) return FSB_EINVAL;
  dim3 blk(kBX, kBY);
  k_gradient<<<grid2d(w, h, blk), blk, 0, as_stream(stream)>>>(u, mask, h, w, g);
  return launch_status();
}

int fsb_divergence(const float* p, const uint8_t* mask, int32_t h, int32_t w, float* div,
                   void* stream) {
  if (h < 1 || w < 1 || !p || !mask || !div) return FSB_EINVAL;
  dim3 blk(kBX, kBY);
  k_divergence<<<grid2d(w, h, blk), blk, 0, as_stream(stream)>>>(p, mask, h, w, div);
  return launch_status();
}

int fsb_pyramid_shapes(int32_t h, int32_t w, int32_t levels, double scale, int32_t min_width,
                       int32_t* shapes, int32_t max_levels) {
  if (!shapes || max_levels < 1) return FSB_EINVAL;
  return pyramid_shapes_internal(h, w, levels, scale, min_width, shapes, max_levels);
}

int fsb_downsample_area(const float* src, const uint8_t* mask, int32_t fh, int32_t fw, float* dst,
                        uint8_t* dmask, int32_t ch, int32_t cw, void* stream) {
  if (fh < 1 || fw < 1 || ch < 1 || cw < 1 || !src || !mask || !dst || !dmask) return FSB_EINVAL;
  return downsample_internal(src, mask, fh, fw, dst, dmask, ch, cw, as_stream(stream));
}

int fsb_upsample_state(const float* u, const float* wv, const uint8_t* mask, int32_t sh,
                       int32_t sw, const uint8_t* dmask, int32_t dh, int32_t dw, float* u_out,
                       float* w_out, void* stream) {
  if (sh < 1 || sw < 1 || dh < 1 || dw < 1 || !u || !wv || !mask || !dmask || !u_out || !w_out)
    return FSB_EINVAL;
  return upsample_internal(u, wv, mask, sh, sw, dmask, dh, dw, u_out, w_out, as_stream(stream));
}

}  // extern "C"
