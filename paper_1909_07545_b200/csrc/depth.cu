// Post-solve depth: the solver's warp w (calibrated frame)
// -> camera-1 correspondence -> depth along camera-0 rays.
//
// Reference: fields.py:170-182 (compose_with_calibration), evaluate.py:101-114
// (depth_from_correspondence), camera.py:317-343 (triangulate_midpoint),
// camera.py:267-270 (camera1_center). fp64 throughout, compiled with
// -fmad=false so the rounding sequence follows NumPy's elementwise order.

#include "fsb_common.cuh"

namespace fsb {
namespace {

bool camera_valid(const fsb_camera& c) {
  return c.width > 0 && c.height > 0 &&
         (c.model == FSB_CAM_PINHOLE || c.model == FSB_CAM_UNIFIED ||
          c.model == FSB_CAM_POLYNOMIAL);
}

// compose_with_calibration: probe = x + w; cal sampled (f64 bicubic) under
// cal_ok; full = w + cal(probe) where valid, else 0.
__global__ void k_compose(const double* __restrict__ wv, const double* __restrict__ cal,
                          const uint8_t* __restrict__ cal_ok, int h, int w,
                          double* __restrict__ full, uint8_t* __restrict__ ok) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const size_t i = (size_t)y * w + x;
  const double w0 = wv[2 * i], w1 = wv[2 * i + 1];
  double c[2];
  const bool v = bicubic_sample<2, double, double>(cal, cal_ok, h, w, (double)x + w0,
                                                   (double)y + w1, c);
  full[2 * i] = v ? w0 + c[0] : 0.0;
  full[2 * i + 1] = v ? w1 + c[1] : 0.0;
  ok[i] = v;
}

// Point pairs: explicit arrays, or the pixel grid of a (h, w) correspondence
// field (x0 = pixel centre, x1 = x0 + corr).
struct Pairs {
  const double* x0;
  const double* x1;
  const double* corr;
  int w;
  FSB_INLINE void get(int64_t i, double& ax, double& ay, double& bx, double& by) const {
    if (corr) {
      ax = (double)(i % w);
      ay = (double)(i / w);
      bx = ax + corr[2 * i];
      by = ay + corr[2 * i + 1];
    } else {
      ax = x0[2 * i]; ay = x0[2 * i + 1];
      bx = x1[2 * i]; by = x1[2 * i + 1];
    }
  }
};

// Polynomial models: Newton iteration count of the whole call, per camera
// (camera.py:177-185 iterate until every point of the call converged).
__global__ void k_pair_iters(Cam c0, Cam c1, Pairs P, int64_t n, int* iters) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int k0 = 0, k1 = 0;
  if (i < n) {
    double ax, ay, bx, by;
    P.get(i, ax, ay, bx, by);
    if (c0.model == FSB_CAM_POLYNOMIAL) k0 = poly_conv_iters(c0, ax, ay);
    if (c1.model == FSB_CAM_POLYNOMIAL) k1 = poly_conv_iters(c1, bx, by);
  }
  for (int o = 16; o > 0; o >>= 1) {
    k0 = max(k0, __shfl_xor_sync(0xffffffffu, k0, o));
    k1 = max(k1, __shfl_xor_sync(0xffffffffu, k1, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(iters, k0);
    atomicMax(iters + 1, k1);
  }
}

struct RigGeom {
  double R[9];   // row-major rotation
  double c1[3];  // camera-1 centre in camera-0 coordinates
};

// triangulate_midpoint for one pair, then the depth_from_correspondence
// post-step when `valid` is given (ok &= valid; depth = min(depth, cap), 0 off).
__global__ void k_triangulate(Cam c0, Cam c1, RigGeom G, Pairs P, int64_t n, double min_angle,
                              const int* iters, const uint8_t* __restrict__ valid,
                              double depth_cap, double* __restrict__ depth,
                              uint8_t* __restrict__ okv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ax, ay, bx, by;
  P.get(i, ax, ay, bx, by);
  const int it0 = c0.model == FSB_CAM_POLYNOMIAL ? iters[0] : 0;
  const int it1 = c1.model == FSB_CAM_POLYNOMIAL ? iters[1] : 0;
  double r0[3], r1[3];
  const bool v0 = cam_unproject(c0, ax, ay, it0, r0[0], r0[1], r0[2]);
  const bool v1 = cam_unproject(c1, bx, by, it1, r1[0], r1[1], r1[2]);
  // d1 = r1 @ R (R^T r1), invalid rays zeroed (camera.py:330-332)
  double d1[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) d1[j] = (r1[0] * G.R[j] + r1[1] * G.R[3 + j]) + r1[2] * G.R[6 + j];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    if (!v0) r0[j] = 0.0;
    if (!v1) d1[j] = 0.0;
  }
  const double b = (r0[0] * d1[0] + r0[1] * d1[1]) + r0[2] * d1[2];
  const double cx = r0[1] * d1[2] - r0[2] * d1[1];
  const double cy = r0[2] * d1[0] - r0[0] * d1[2];
  const double cz = r0[0] * d1[1] - r0[1] * d1[0];
  const double sin_angle = sqrt((cx * cx + cy * cy) + cz * cz);
  const double p = (r0[0] * G.c1[0] + r0[1] * G.c1[1]) + r0[2] * G.c1[2];
  const double q = (d1[0] * G.c1[0] + d1[1] * G.c1[1]) + d1[2] * G.c1[2];
  bool ok = v0 && v1 && sin_angle >= min_angle;
  const double denom = ok ? 1.0 - b * b : 1.0;
  const double s0 = (p - b * q) / denom;
  ok = ok && s0 > 0.0;
  if (valid) {  // depth_from_correspondence (evaluate.py:110-113)
    ok = ok && valid[i];
    depth[i] = ok ? fmin(s0, depth_cap) : 0.0;
  } else {
    depth[i] = ok ? s0 : NAN;
  }
  okv[i] = ok;
}

// trace_epipolar_curves (fields.py:111-139): Euler steps of length `step`
// (a shorter last one) along the bicubic-sampled direction field, one thread
// per start; a trace dies where the sample is invalid or its norm <= 0.5.
__global__ void k_trace(const double* __restrict__ dirs, const uint8_t* __restrict__ valid, int h,
                        int w, const double* __restrict__ starts, int64_t n, int n_steps,
                        double length, double step, double* __restrict__ verts,
                        uint8_t* __restrict__ alive) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double px = starts[2 * s], py = starts[2 * s + 1];
  double* v = verts + (size_t)s * (n_steps + 1) * 2;
  uint8_t* al = alive + (size_t)s * (n_steps + 1);
  v[0] = px; v[1] = py;
  al[0] = 1;
  bool live = true;
  for (int i = 0; i < n_steps; ++i) {
    const double seg = fmin(step, length - (double)i * step);
    double d[2] = {0.0, 0.0};
    bool ok = bicubic_sample<2, double, double>(dirs, valid, h, w, px, py, d);
    const double d0 = ok ? d[0] : 0.0, d1 = ok ? d[1] : 0.0;
    const double nrm = sqrt(d0 * d0 + d1 * d1);
    ok = ok && nrm > 0.5;
    live = live && ok;
    const double den = fmax(nrm, 1e-300);
    const double ux = live ? d0 / den : 0.0, uy = live ? d1 / den : 0.0;
    px = px + seg * ux;
    py = py + seg * uy;
    v[2 * (i + 1)] = live ? px : NAN;
    v[2 * (i + 1) + 1] = live ? py : NAN;
    al[i + 1] = live;
  }
}

RigGeom rig_geom(const fsb_rig& r) {
  RigGeom G;
  for (int k = 0; k < 9; ++k) G.R[k] = r.rotation[k];
  // -R^T t, in the order of numpy's (3,3) @ (3,) product
  for (int j = 0; j < 3; ++j) {
    const double s = (r.rotation[j] * r.translation[0] + r.rotation[3 + j] * r.translation[1]) +
                     r.rotation[6 + j] * r.translation[2];
    G.c1[j] = -s;
  }
  return G;
}

int triangulate_t(const fsb_rig* rig, const Pairs& P, int64_t n, double min_angle,
                  const uint8_t* valid, double depth_cap, double* depth, uint8_t* ok,
                  void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (!rig || !camera_valid(rig->cam0) || !camera_valid(rig->cam1) || n < 0) return FSB_EINVAL;
  if (n > 0 && (!depth || !ok)) return FSB_EINVAL;
  if (!scratch || scratch_bytes < 2 * sizeof(int)) return FSB_EINVAL;
  if (n == 0) return FSB_OK;
  const Cam c0 = make_cam(rig->cam0), c1 = make_cam(rig->cam1);
  int* iters = static_cast<int*>(scratch);
  const int threads = 128;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  cudaMemsetAsync(iters, 0, 2 * sizeof(int), st);
  if (c0.model == FSB_CAM_POLYNOMIAL || c1.model == FSB_CAM_POLYNOMIAL)
    k_pair_iters<<<blocks, threads, 0, st>>>(c0, c1, P, n, iters);
  k_triangulate<<<blocks, threads, 0, st>>>(c0, c1, rig_geom(*rig), P, n, min_angle, iters, valid,
                                            depth_cap, depth, ok);
  return launch_status();
}

}  // namespace
}  // namespace fsb

using namespace fsb;

extern "C" {

int fsb_compose_calibration(const double* wv, const double* cal, const uint8_t* cal_ok, int32_t h,
                            int32_t w, double* full, uint8_t* ok, void* stream) {
  if (h <= 0 || w <= 0 || !wv || !cal || !cal_ok || !full || !ok) return FSB_EINVAL;
  const dim3 blk(32, 8);
  k_compose<<<grid2d(w, h, blk), blk, 0, as_stream(stream)>>>(wv, cal, cal_ok, h, w, full, ok);
  return launch_status();
}

int fsb_trace_epipolar_curves(const double* dirs, const uint8_t* valid, int32_t h, int32_t w,
                              const double* starts, int64_t n, int32_t n_steps, double length,
                              double step, double* verts, uint8_t* alive, void* stream) {
  if (h <= 0 || w <= 0 || n < 0 || n_steps < 0 || !(step > 0) || !dirs || !valid ||
      (n > 0 && (!starts || !verts || !alive)))
    return FSB_EINVAL;
  if (n == 0) return FSB_OK;
  const int threads = 128;
  k_trace<<<(unsigned)((n + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
      dirs, valid, h, w, starts, n, n_steps, length, step, verts, alive);
  return launch_status();
}

size_t fsb_triangulate_scratch_bytes(void) { return 256; }

int fsb_triangulate_midpoint(const fsb_rig* rig, const double* x0, const double* x1, int64_t n,
                             double min_angle, double* depth, uint8_t* ok, void* scratch,
                             size_t scratch_bytes, void* stream) {
  if (n > 0 && (!x0 || !x1)) return FSB_EINVAL;
  const Pairs P{x0, x1, nullptr, 0};
  return triangulate_t(rig, P, n, min_angle, nullptr, 0.0, depth, ok, scratch, scratch_bytes,
                       as_stream(stream));
}

int fsb_depth_from_correspondence(const fsb_rig* rig, const double* corr, const uint8_t* valid,
                                  int32_t h, int32_t w, double depth_cap, double* depth,
                                  uint8_t* ok, void* scratch, size_t scratch_bytes,
                                  void* stream) {
  if (h <= 0 || w <= 0 || !corr || !valid) return FSB_EINVAL;
  const Pairs P{nullptr, nullptr, corr, w};
  return triangulate_t(rig, P, (int64_t)h * w, 1e-6, valid, depth_cap, depth, ok, scratch,
                       scratch_bytes, as_stream(stream));
}

}  // extern "C"
