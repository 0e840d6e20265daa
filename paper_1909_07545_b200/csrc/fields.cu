// K1 / K2: camera masks, calibration field + calibrated image, trajectory field.
// fp64 compute (compiled with -fmad=false), fp32 storage of directions.
//
// Reference: fields.py:28-108 and camera.py:79-190, solver.py:389-398.

#include "fsb_common.cuh"

namespace fsb {
namespace {

constexpr int kBX = 32, kBY = 8;

struct PolyScratch {
  int* iters;  // call-wide Newton iteration count
};

// Pass 0 of every polynomial unproject: per-pixel convergence count -> max.
__global__ void k_poly_iters_grid(Cam c, int* iters) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  int n = 0;
  if (x < c.width && y < c.height) n = poly_conv_iters(c, (double)x, (double)y);
  // block max then one atomic
  for (int o = 16; o > 0; o >>= 1) n = max(n, __shfl_xor_sync(0xffffffffu, n, o));
  if ((threadIdx.x & 31) == 0) atomicMax(iters, n);
}

__global__ void k_poly_iters_pts(Cam c, const double* __restrict__ pix, int64_t n, int* iters) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int k = 0;
  if (i < n) k = poly_conv_iters(c, pix[2 * i], pix[2 * i + 1]);
  for (int o = 16; o > 0; o >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, o));
  if ((threadIdx.x & 31) == 0) atomicMax(iters, k);
}

__device__ __forceinline__ int poly_iters_of(const Cam& c, const int* iters) {
  return c.model == FSB_CAM_POLYNOMIAL ? *iters : 0;
}

// fov_mask (camera.py:79-84)
__global__ void k_fov_mask(Cam c, const int* iters, uint8_t* __restrict__ mask) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= c.width || y >= c.height) return;
  double rx, ry, rz;
  mask[(size_t)y * c.width + x] =
      cam_unproject(c, (double)x, (double)y, poly_iters_of(c, iters), rx, ry, rz) ? 1 : 0;
}

__global__ void k_unproject_pts(Cam c, const int* iters, const double* __restrict__ pix, int64_t n,
                                double* __restrict__ rays, uint8_t* __restrict__ valid) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double rx, ry, rz;
  bool ok = cam_unproject(c, pix[2 * i], pix[2 * i + 1], poly_iters_of(c, iters), rx, ry, rz);
  if (!ok) rx = ry = rz = NAN;
  rays[3 * i] = rx; rays[3 * i + 1] = ry; rays[3 * i + 2] = rz;
  valid[i] = ok;
}

__global__ void k_project_pts(Cam c, const double* __restrict__ pts, int64_t n,
                              double* __restrict__ pix, uint8_t* __restrict__ valid) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double px, py;
  bool ok = cam_project(c, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], px, py);
  if (!ok) px = py = NAN;
  pix[2 * i] = px; pix[2 * i + 1] = py;
  valid[i] = ok;
}

struct Rot { double r[9]; };

// Calibration flow of one cam0 pixel (fields.py:34-45): rays of camera 0,
// rotated by R (rays @ R.T), projected by camera 1.
__device__ __forceinline__ bool calib_flow(const Cam& c0, const Cam& c1, const Rot& R, int it0,
                                           int x, int y, double& fx, double& fy) {
  double rx, ry, rz;
  bool v0 = cam_unproject(c0, (double)x, (double)y, it0, rx, ry, rz);
  if (!v0) rx = ry = rz = 0.0;  // _grid_rays zeroes invalid rays (fields.py:31)
  double X = __dadd_rn(__dadd_rn(__dmul_rn(rx, R.r[0]), __dmul_rn(ry, R.r[1])), __dmul_rn(rz, R.r[2]));
  double Y = __dadd_rn(__dadd_rn(__dmul_rn(rx, R.r[3]), __dmul_rn(ry, R.r[4])), __dmul_rn(rz, R.r[5]));
  double Z = __dadd_rn(__dadd_rn(__dmul_rn(rx, R.r[6]), __dmul_rn(ry, R.r[7])), __dmul_rn(rz, R.r[8]));
  double px, py;
  bool v1 = cam_project(c1, X, Y, Z, px, py);
  bool ok = v0 && v1;
  fx = ok ? px - (double)x : 0.0;
  fy = ok ? py - (double)y : 0.0;
  return ok;
}

__global__ void k_calibration_field(Cam c0, Cam c1, Rot R, const int* iters0,
                                    double* __restrict__ field, uint8_t* __restrict__ ok) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= c0.width || y >= c0.height) return;
  double fx, fy;
  bool v = calib_flow(c0, c1, R, poly_iters_of(c0, iters0), x, y, fx, fy);
  size_t i = (size_t)y * c0.width + x;
  field[2 * i] = fx; field[2 * i + 1] = fy;
  ok[i] = v;
}

// calibrate_second_image (solver.py:389-398): i1c = bicubic(i1, x + cal, mask1),
// ok = sample_ok & cal_ok, zero where invalid. f64 accumulation.
template <typename TI, typename TO>
__global__ void k_calibrate_image(Cam c0, Cam c1, Rot R, const int* iters0,
                                  const TI* __restrict__ i1, const uint8_t* __restrict__ mask1,
                                  TO* __restrict__ i1c, uint8_t* __restrict__ okout) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= c0.width || y >= c0.height) return;
  double fx, fy;
  bool cal_ok = calib_flow(c0, c1, R, poly_iters_of(c0, iters0), x, y, fx, fy);
  double v[1];
  bool s_ok = bicubic_sample<1, double, TI>(i1, mask1, c1.height, c1.width, (double)x + fx,
                                            (double)y + fy, v);
  bool ok = s_ok && cal_ok;
  size_t i = (size_t)y * c0.width + x;
  i1c[i] = ok ? (TO)v[0] : TO(0);
  okout[i] = ok;
}

// ---------------------------------------------------------------- trajectory
// generate_trajectory_field (fields.py:48-108), three passes:
//   A: rays (cached) + flow at eps0 = 1e-4*depth, grid max of |w| over valid;
//   B: flow at eps0*eps_scale/peak, unit directions, residue/degenerate flags;
//   C: global residue renormalisation and the epipole cross (fields.py:91-107).

struct TrajScratch {
  double* rays;      // 3 per pixel
  double* dirs;      // 2 per pixel
  uint8_t* valid0;   // per pixel
  uint8_t* state;    // per pixel: bit0 good, bit1 degenerate
  double* peak;      // 1
  int* flags;        // [0] any residue, [1] any degenerate, [2] poly iters
};

__device__ __forceinline__ bool traj_flow(const Cam& c, double eps, const double* th, double depth,
                                          double rx, double ry, double rz, bool v0, int x, int y,
                                          double& wx, double& wy) {
  double X = rx * depth + eps * th[0];
  double Y = ry * depth + eps * th[1];
  double Z = rz * depth + eps * th[2];
  double px, py;
  bool v1 = cam_project(c, X, Y, Z, px, py);
  bool ok = v0 && v1;
  wx = ok ? px - (double)x : 0.0;
  wy = ok ? py - (double)y : 0.0;
  return ok;
}

struct Vec3 { double v[3]; };

__global__ void k_traj_a(Cam c, Vec3 that, double depth, TrajScratch s) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  double mag = 0.0;
  if (x < c.width && y < c.height) {
    size_t i = (size_t)y * c.width + x;
    double rx, ry, rz;
    bool v0 = cam_unproject(c, (double)x, (double)y, poly_iters_of(c, s.flags + 2), rx, ry, rz);
    if (!v0) rx = ry = rz = 0.0;
    s.rays[3 * i] = rx; s.rays[3 * i + 1] = ry; s.rays[3 * i + 2] = rz;
    s.valid0[i] = v0;
    double wx, wy;
    bool ok = traj_flow(c, 1e-4 * depth, that.v, depth, rx, ry, rz, v0, x, y, wx, wy);
    if (ok) mag = sqrt(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)));
  }
  mag = warp_max(mag);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(s.peak, mag);
}

__global__ void k_traj_b(Cam c, Vec3 that, double depth, double eps_scale, TrajScratch s) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  bool residue = false, degen = false;
  if (x < c.width && y < c.height) {
    size_t i = (size_t)y * c.width + x;
    double peak = *s.peak;
    double eps = 1e-4 * depth;
    if (peak > 0.0) eps = ((1e-4 * depth) * eps_scale) / peak;
    double wx, wy;
    bool valid = traj_flow(c, eps, that.v, depth, s.rays[3 * i], s.rays[3 * i + 1],
                           s.rays[3 * i + 2], s.valid0[i] != 0, x, y, wx, wy);
    double mag = sqrt(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)));
    degen = valid && mag < 1e-12;
    bool good = valid && mag >= 1e-12;
    double dx = good ? wx / mag : 0.0;
    double dy = good ? wy / mag : 0.0;
    residue = (fabs(dx) < 1e-9 && dx != 0.0) || (fabs(dy) < 1e-9 && dy != 0.0);
    s.dirs[2 * i] = dx; s.dirs[2 * i + 1] = dy;
    s.state[i] = (good ? 1 : 0) | (degen ? 2 : 0);
  }
  if (__any_sync(0xffffffffu, residue) && (threadIdx.x & 31) == 0) atomicOr(s.flags + 0, 1);
  if (__any_sync(0xffffffffu, degen) && (threadIdx.x & 31) == 0) atomicOr(s.flags + 1, 1);
}

template <typename TO>
__global__ void k_traj_c(int w, int h, TrajScratch s, TO* __restrict__ dirs,
                         uint8_t* __restrict__ ok) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  size_t i = (size_t)y * w + x;
  double dx = s.dirs[2 * i], dy = s.dirs[2 * i + 1];
  bool good = s.state[i] & 1;
  if (s.flags[0]) {  // fields.py:91-96 (applied to every pixel when any residue exists)
    if (fabs(dx) < 1e-9 && dx != 0.0) dx = 0.0;
    if (fabs(dy) < 1e-9 && dy != 0.0) dy = 0.0;
    double n = sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    if (n > 0.5) { dx = dx / n; dy = dy / n; } else { dx = 0.0; dy = 0.0; }
  }
  if (s.flags[1]) {  // fields.py:100-107: drop the 4-neighbour cross around degenerate pixels
    bool blocked = (s.state[i] & 2) || (y > 0 && (s.state[i - w] & 2)) ||
                   (y + 1 < h && (s.state[i + w] & 2)) || (x > 0 && (s.state[i - 1] & 2)) ||
                   (x + 1 < w && (s.state[i + 1] & 2));
    good = good && !blocked;
    if (!good) { dx = 0.0; dy = 0.0; }
  }
  dirs[2 * i] = (TO)dx;
  dirs[2 * i + 1] = (TO)dy;
  ok[i] = good;
}

TrajScratch carve_traj(void* base, int w, int h) {
  size_t n = (size_t)w * h;
  char* p = static_cast<char*>(base);
  TrajScratch s;
  s.rays = reinterpret_cast<double*>(p); p += align_up(n * 3 * sizeof(double));
  s.dirs = reinterpret_cast<double*>(p); p += align_up(n * 2 * sizeof(double));
  s.valid0 = reinterpret_cast<uint8_t*>(p); p += align_up(n);
  s.state = reinterpret_cast<uint8_t*>(p); p += align_up(n);
  s.peak = reinterpret_cast<double*>(p); p += 256;
  s.flags = reinterpret_cast<int*>(p);
  return s;
}

size_t traj_bytes(int w, int h) {
  size_t n = (size_t)w * h;
  return align_up(n * 3 * sizeof(double)) + align_up(n * 2 * sizeof(double)) + 2 * align_up(n) +
         512;
}

bool cam_ok(const fsb_camera* c) {
  return c && c->width > 0 && c->height > 0 &&
         (c->model == FSB_CAM_PINHOLE || c->model == FSB_CAM_UNIFIED ||
          c->model == FSB_CAM_POLYNOMIAL);
}

// Enqueue the polynomial iteration-count pre-pass for the full grid of `c`.
int poly_prepass_grid(const Cam& c, int* iters, cudaStream_t st) {
  if (c.model != FSB_CAM_POLYNOMIAL) return FSB_OK;
  cudaMemsetAsync(iters, 0, sizeof(int), st);
  dim3 blk(kBX, kBY);
  k_poly_iters_grid<<<grid2d(c.width, c.height, blk), blk, 0, st>>>(c, iters);
  return launch_status();
}

}  // namespace

// ---------------------------------------------------------------- internal API
// (used by the pyramid driver in solver.cu)

size_t traj_scratch_bytes_internal(int w, int h) { return traj_bytes(w, h); }

template <typename TO>
int trajectory_field_t(const fsb_camera* cam, const double t[3], double eps_scale, double depth,
                       TO* dirs, uint8_t* ok, void* scratch, size_t scratch_bytes,
                       cudaStream_t st) {
  if (!cam_ok(cam) || !dirs || !ok || !scratch || !t) return FSB_EINVAL;
  if (scratch_bytes < traj_bytes(cam->width, cam->height)) return FSB_ENOSPC;
  // fields.py:63-67: t_hat = t / ||t||, zero baseline is an error.
  double tn = sqrt((t[0] * t[0] + t[1] * t[1]) + t[2] * t[2]);
  if (tn == 0.0) return FSB_EDOMAIN;
  Vec3 th;
  th.v[0] = t[0] / tn; th.v[1] = t[1] / tn; th.v[2] = t[2] / tn;
  Cam c = make_cam(*cam);
  TrajScratch s = carve_traj(scratch, c.width, c.height);
  cudaMemsetAsync(s.peak, 0, 256 + 3 * sizeof(int), st);
  int rc = poly_prepass_grid(c, s.flags + 2, st);
  if (rc) return rc;
  dim3 blk(kBX, kBY), grd = grid2d(c.width, c.height, blk);
  k_traj_a<<<grd, blk, 0, st>>>(c, th, depth, s);
  k_traj_b<<<grd, blk, 0, st>>>(c, th, depth, eps_scale, s);
  k_traj_c<TO><<<grd, blk, 0, st>>>(c.width, c.height, s, dirs, ok);
  return launch_status();
}

int trajectory_field_internal(const fsb_camera* cam, const double t[3], double eps_scale,
                              double depth, float* dirs, uint8_t* ok, void* scratch,
                              size_t scratch_bytes, cudaStream_t st) {
  return trajectory_field_t<float>(cam, t, eps_scale, depth, dirs, ok, scratch, scratch_bytes, st);
}

int trajectory_field64_internal(const fsb_camera* cam, const double t[3], double eps_scale,
                                double depth, double* dirs, uint8_t* ok, void* scratch,
                                size_t scratch_bytes, cudaStream_t st) {
  return trajectory_field_t<double>(cam, t, eps_scale, depth, dirs, ok, scratch, scratch_bytes,
                                    st);
}

int fov_mask_internal(const fsb_camera* cam, uint8_t* mask, int* iters, cudaStream_t st) {
  if (!cam_ok(cam) || !mask || !iters) return FSB_EINVAL;
  Cam c = make_cam(*cam);
  int rc = poly_prepass_grid(c, iters, st);
  if (rc) return rc;
  dim3 blk(kBX, kBY);
  k_fov_mask<<<grid2d(c.width, c.height, blk), blk, 0, st>>>(c, iters, mask);
  return launch_status();
}

// i1c/ok on the cam0 grid; mask1 must be the cam1 FOV mask; iters0 scratch int.
template <typename TI, typename TO>
int calibrate_t(const fsb_rig* rig, const TI* i1, const uint8_t* mask1, TO* i1c, uint8_t* ok,
                int* iters0, cudaStream_t st) {
  Cam c0 = make_cam(rig->cam0), c1 = make_cam(rig->cam1);
  Rot R;
  for (int k = 0; k < 9; ++k) R.r[k] = rig->rotation[k];
  int rc = poly_prepass_grid(c0, iters0, st);
  if (rc) return rc;
  dim3 blk(kBX, kBY);
  k_calibrate_image<TI, TO><<<grid2d(c0.width, c0.height, blk), blk, 0, st>>>(c0, c1, R, iters0,
                                                                              i1, mask1, i1c, ok);
  return launch_status();
}

int calibrate_internal(const fsb_rig* rig, const float* i1, const uint8_t* mask1, float* i1c,
                       uint8_t* ok, int* iters0, cudaStream_t st) {
  return calibrate_t<float, float>(rig, i1, mask1, i1c, ok, iters0, st);
}

int calibrate64_internal(const fsb_rig* rig, const double* i1, const uint8_t* mask1, double* i1c,
                         uint8_t* ok, int* iters0, cudaStream_t st) {
  return calibrate_t<double, double>(rig, i1, mask1, i1c, ok, iters0, st);
}

}  // namespace fsb

using namespace fsb;

extern "C" {

size_t fsb_fov_mask_scratch_bytes(const fsb_camera*) { return 256; }

int fsb_fov_mask(const fsb_camera* cam, uint8_t* mask, void* scratch, size_t scratch_bytes,
                 void* stream) {
  if (!scratch || scratch_bytes < sizeof(int)) return FSB_EINVAL;
  return fov_mask_internal(cam, mask, static_cast<int*>(scratch), as_stream(stream));
}

size_t fsb_unproject_scratch_bytes(void) { return 256; }

int fsb_unproject(const fsb_camera* cam, const double* pix, int64_t n, double* rays,
                  uint8_t* valid, void* scratch, size_t scratch_bytes, void* stream) {
  if (!cam_ok(cam) || n < 0 || (n > 0 && (!pix || !rays || !valid))) return FSB_EINVAL;
  if (!scratch || scratch_bytes < sizeof(int)) return FSB_EINVAL;
  if (n == 0) return FSB_OK;
  cudaStream_t st = as_stream(stream);
  Cam c = make_cam(*cam);
  int* iters = static_cast<int*>(scratch);
  int threads = 128;
  unsigned blocks = (unsigned)((n + threads - 1) / threads);
  if (c.model == FSB_CAM_POLYNOMIAL) {
    cudaMemsetAsync(iters, 0, sizeof(int), st);
    k_poly_iters_pts<<<blocks, threads, 0, st>>>(c, pix, n, iters);
  }
  k_unproject_pts<<<blocks, threads, 0, st>>>(c, iters, pix, n, rays, valid);
  return launch_status();
}

int fsb_project(const fsb_camera* cam, const double* pts, int64_t n, double* pix, uint8_t* valid,
                void* stream) {
  if (!cam_ok(cam) || n < 0 || (n > 0 && (!pix || !pts || !valid))) return FSB_EINVAL;
  if (n == 0) return FSB_OK;
  int threads = 128;
  unsigned blocks = (unsigned)((n + threads - 1) / threads);
  k_project_pts<<<blocks, threads, 0, as_stream(stream)>>>(make_cam(*cam), pts, n, pix, valid);
  return launch_status();
}

int fsb_calibration_field(const fsb_rig* rig, double* field, uint8_t* ok, void* scratch,
                          size_t scratch_bytes, void* stream) {
  if (!rig || !cam_ok(&rig->cam0) || !cam_ok(&rig->cam1) || !field || !ok) return FSB_EINVAL;
  if (!scratch || scratch_bytes < sizeof(int)) return FSB_EINVAL;
  cudaStream_t st = as_stream(stream);
  Cam c0 = make_cam(rig->cam0), c1 = make_cam(rig->cam1);
  Rot R;
  for (int k = 0; k < 9; ++k) R.r[k] = rig->rotation[k];
  int* iters = static_cast<int*>(scratch);
  int rc = poly_prepass_grid(c0, iters, st);
  if (rc) return rc;
  dim3 blk(kBX, kBY);
  k_calibration_field<<<grid2d(c0.width, c0.height, blk), blk, 0, st>>>(c0, c1, R, iters, field,
                                                                        ok);
  return launch_status();
}

size_t fsb_calibrate_scratch_bytes(const fsb_rig* rig) {
  if (!rig) return 0;
  return align_up((size_t)rig->cam1.width * rig->cam1.height) + 512;
}

int fsb_calibrate_second_image(const fsb_rig* rig, const float* i1, const uint8_t* mask1,
                               float* i1c, uint8_t* ok, void* scratch, size_t scratch_bytes,
                               void* stream) {
  if (!rig || !cam_ok(&rig->cam0) || !cam_ok(&rig->cam1) || !i1 || !i1c || !ok || !scratch)
    return FSB_EINVAL;
  if (scratch_bytes < fsb_calibrate_scratch_bytes(rig)) return FSB_ENOSPC;
  cudaStream_t st = as_stream(stream);
  char* p = static_cast<char*>(scratch);
  int* iters = reinterpret_cast<int*>(p);
  int* iters1 = reinterpret_cast<int*>(p + 256);
  uint8_t* m1 = reinterpret_cast<uint8_t*>(p + 512);
  if (!mask1) {
    int rc = fov_mask_internal(&rig->cam1, m1, iters1, st);
    if (rc) return rc;
    mask1 = m1;
  }
  return calibrate_internal(rig, i1, mask1, i1c, ok, iters, st);
}

size_t fsb_trajectory_scratch_bytes(const fsb_camera* cam) {
  if (!cam) return 0;
  return traj_bytes(cam->width, cam->height);
}

int fsb_trajectory_field(const fsb_camera* cam, const double t[3], double epsilon_scale,
                         double depth, float* dirs, uint8_t* ok, void* scratch,
                         size_t scratch_bytes, void* stream) {
  return trajectory_field_internal(cam, t, epsilon_scale, depth, dirs, ok, scratch, scratch_bytes,
                                   as_stream(stream));
}

int fsb_trajectory_field_f64(const fsb_camera* cam, const double t[3], double epsilon_scale,
                             double depth, double* dirs, uint8_t* ok, void* scratch,
                             size_t scratch_bytes, void* stream) {
  return trajectory_field64_internal(cam, t, epsilon_scale, depth, dirs, ok, scratch,
                                     scratch_bytes, as_stream(stream));
}

}  // extern "C"
