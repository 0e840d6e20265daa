// Synthetic input generator: per-pixel ray casting of analytic primitives with
// procedural textures (the reference's input generator and test-pair source,
// SURVEY §8f row 2). fp64 compute (-fmad=false), fp32 image out.
//
// Reference: synth.py:28-84 (lattice hash, value noise, fractal noise),
// synth.py:87-118 (checkerboard, sine grating), synth.py:124-190 (plane /
// sphere / box intersection), synth.py:193-205 (nearest-hit cast),
// synth.py:217-268 (render with s x s supersampling).
//
// Difference noted in DESIGN.md: the polynomial lens Newton runs to per-pixel
// convergence here (the reference iterates until every pixel of the call has
// converged); the resulting ray differs by < 1e-10 rad.

#include "fsb_common.cuh"

namespace fsb {
namespace {

constexpr double kEps = 1e-9;  // synth.py:23

__device__ __forceinline__ double hash01(long long ix, long long iy, long long iz,
                                         unsigned long long salt) {
  unsigned long long h = ((unsigned long long)ix * 0x9E3779B97F4A7C15ull) ^
                         ((unsigned long long)iy * 0xC2B2AE3D27D4EB4Full) ^
                         ((unsigned long long)iz * 0x165667B19E3779F9ull) ^ salt;
  h ^= h >> 33;
  h *= 0xFF51AFD7ED558CCDull;
  h ^= h >> 33;
  h *= 0xC4CEB9FE1A85EC53ull;
  h ^= h >> 33;
  return (double)(h >> 11) / 9007199254740992.0;  // 2^53
}

__device__ double value_noise(double px, double py, double pz, double scale,
                              unsigned long long salt) {
  double cx = px / scale, cy = py / scale, cz = pz / scale;
  double bx = floor(cx), by = floor(cy), bz = floor(cz);
  double fx = cx - bx, fy = cy - by, fz = cz - bz;
  fx = fx * fx * (3.0 - 2.0 * fx);
  fy = fy * fy * (3.0 - 2.0 * fy);
  fz = fz * fz * (3.0 - 2.0 * fz);
  long long ix = (long long)bx, iy = (long long)by, iz = (long long)bz;
  double acc = 0.0;
  for (int dz = 0; dz < 2; ++dz) {
    double wz = dz ? fz : 1.0 - fz;
    for (int dy = 0; dy < 2; ++dy) {
      double wy = dy ? fy : 1.0 - fy;
      for (int dx = 0; dx < 2; ++dx) {
        double wx = dx ? fx : 1.0 - fx;
        acc += ((wx * wy) * wz) * hash01(ix + dx, iy + dy, iz + dz, salt);
      }
    }
  }
  return acc;
}

__device__ double shade(const fsb_prim& p, double x, double y, double z) {
  if (p.tex_kind == FSB_TEX_NOISE) {
    double total = 0.0, amp_sum = 0.0, amp = 1.0;
    for (int o = 0; o < p.octaves; ++o) {
      unsigned long long salt =
          (unsigned long long)(p.seed + o) * 0x27D4EB2Full + 0x165667B1ull;
      total += amp * value_noise(x, y, z, p.tex[0] / (double)(1ll << o), salt);
      amp_sum += amp;
      amp *= p.tex[3];
    }
    double t = total / amp_sum;
    return p.tex[1] + (p.tex[2] - p.tex[1]) * t;
  }
  if (p.tex_kind == FSB_TEX_CHECKER) {
    long long qx = (long long)floor(x / p.tex[0]), qy = (long long)floor(y / p.tex[0]),
              qz = (long long)floor(z / p.tex[0]);
    return ((qx + qy + qz) & 1) == 0 ? p.tex[1] : p.tex[2];
  }
  // sine grating: tex = wavelength, lo, hi, unit direction (host-normalised)
  double dot = (x * p.tex[3] + y * p.tex[4]) + z * p.tex[5];
  double phase = 2.0 * kPi * dot / p.tex[0];
  double t = 0.5 + 0.5 * sin(phase);
  return p.tex[1] + (p.tex[2] - p.tex[1]) * t;
}

__device__ double intersect(const fsb_prim& p, const double o[3], const double d[3]) {
  const double* g = p.geom;
  if (p.kind == FSB_PRIM_PLANE) {  // normal pre-normalised on the host
    double denom = (d[0] * g[3] + d[1] * g[4]) + d[2] * g[5];
    double num = ((g[0] - o[0]) * g[3] + (g[1] - o[1]) * g[4]) + (g[2] - o[2]) * g[5];
    double t = fabs(denom) > kEps ? num / (denom == 0.0 ? 1.0 : denom) : INFINITY;
    return t > kEps ? t : INFINITY;
  }
  if (p.kind == FSB_PRIM_SPHERE) {
    double oc0 = o[0] - g[0], oc1 = o[1] - g[1], oc2 = o[2] - g[2];
    double b = (d[0] * oc0 + d[1] * oc1) + d[2] * oc2;
    double c = ((oc0 * oc0 + oc1 * oc1) + oc2 * oc2) - g[3] * g[3];
    double disc = b * b - c;
    bool hit = disc >= 0.0;
    double sq = sqrt(fmax(disc, 0.0));
    double tn = -b - sq, tf = -b + sq;
    double t = tn > kEps ? tn : tf;
    return (hit && t > kEps) ? t : INFINITY;
  }
  // axis-aligned box, slab test (nan -> -inf / +inf as np.nan_to_num)
  double tnear = -INFINITY, tfar = INFINITY;
  for (int k = 0; k < 3; ++k) {
    double inv = 1.0 / d[k];
    double t1 = (g[k] - o[k]) * inv, t2 = (g[3 + k] - o[k]) * inv;
    if (isnan(t1)) t1 = -INFINITY;
    if (isnan(t2)) t2 = INFINITY;
    tnear = fmax(tnear, fmin(t1, t2));
    tfar = fmin(tfar, fmax(t1, t2));
  }
  bool hit = (tnear <= tfar) && (tfar > kEps);
  double t = tnear > kEps ? tnear : tfar;
  return hit ? t : INFINITY;
}

struct RenderArgs {
  Cam cam;
  double R[9];      // world->camera rotation (identity for camera 0)
  double origin[3]; // camera centre in world coordinates
  const fsb_prim* prims;
  int nprims;
  int ss;
};

// One ray: returns hit distance (inf = miss / invalid ray) and shade.
__device__ bool cast_ray(const RenderArgs& a, double px, double py, double& t_out,
                         double& sh_out) {
  double rx, ry, rz;
  int iters = 0;
  if (a.cam.model == FSB_CAM_POLYNOMIAL) iters = poly_conv_iters(a.cam, px, py);
  bool valid = cam_unproject(a.cam, px, py, iters, rx, ry, rz);
  if (!valid) rx = ry = rz = 0.0;
  // dirs = rays @ R (R^T applied row-wise), synth.py:264-266
  double d[3];
  for (int i = 0; i < 3; ++i) d[i] = (rx * a.R[0 * 3 + i] + ry * a.R[1 * 3 + i]) + rz * a.R[2 * 3 + i];
  double best = INFINITY, sh = 0.0;
  for (int k = 0; k < a.nprims; ++k) {
    const fsb_prim p = a.prims[k];
    double t = intersect(p, a.origin, d);
    if (t < best) {
      best = t;
      sh = shade(p, a.origin[0] + d[0] * t, a.origin[1] + d[1] * t, a.origin[2] + d[2] * t);
    }
  }
  t_out = best;
  sh_out = sh;
  return valid;
}

__global__ void k_render(RenderArgs a, float* __restrict__ image, float* __restrict__ depth,
                         uint8_t* __restrict__ hitmask) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= a.cam.width || y >= a.cam.height) return;
  double t, sh;
  bool valid = cast_ray(a, (double)x, (double)y, t, sh);
  bool hit = isfinite(t) && valid;
  double img;
  if (a.ss == 1) {
    img = hit ? sh : 0.0;
  } else {
    double acc = 0.0, cnt = 0.0;
    for (int j = 0; j < a.ss; ++j) {
      double oy = (j + 0.5) / a.ss - 0.5;
      for (int i = 0; i < a.ss; ++i) {
        double ox = (i + 0.5) / a.ss - 0.5;
        double ts, ss;
        bool va = cast_ray(a, x + ox, y + oy, ts, ss);
        bool ok = isfinite(ts) && va;
        acc += ok ? ss : 0.0;
        cnt += ok ? 1.0 : 0.0;
      }
    }
    img = (hit && cnt > 0.0) ? acc / fmax(cnt, 1.0) : 0.0;
  }
  size_t o = (size_t)y * a.cam.width + x;
  image[o] = (float)img;
  if (depth) depth[o] = hit ? (float)t : 0.f;
  if (hitmask) hitmask[o] = hit;
}

// Nearest hit distance of a ray from `o` along `d` over the scene (Scene.cast
// without the shading, synth.py:193-205).
__device__ double first_hit(const fsb_prim* prims, int nprims, const double o[3],
                            const double d[3]) {
  double best = INFINITY;
  for (int k = 0; k < nprims; ++k) {
    const double t = intersect(prims[k], o, d);
    if (t < best) best = t;
  }
  return best;
}

struct TruthArgs {
  Cam c0, c1;
  double R[9], t[3], c1w[3];  // pose (world = camera 0) and camera-1 centre
  const fsb_prim* prims;
  int nprims;
  double tol;
};

// make_ground_truth (synth.py:271-303) for one camera-0 pixel: depth0 from a
// point-sampled camera-0 render, the exact correspondence through camera 1,
// and covisibility (unoccluded from camera 1, inside its FOV and image).
__global__ void k_ground_truth(TruthArgs a, const int* iters, double* __restrict__ depth0,
                               double* __restrict__ corr, uint8_t* __restrict__ covis) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= a.c0.width || y >= a.c0.height) return;
  const size_t i = (size_t)y * a.c0.width + x;
  double r[3];
  const bool valid = cam_unproject(a.c0, (double)x, (double)y,
                                   a.c0.model == FSB_CAM_POLYNOMIAL ? *iters : 0, r[0], r[1],
                                   r[2]);
  if (!valid) r[0] = r[1] = r[2] = 0.0;
  const double o0[3] = {0.0, 0.0, 0.0};
  const double t0 = first_hit(a.prims, a.nprims, o0, r);
  const bool hit = isfinite(t0) && valid;  // render()'s valid0
  const double dep = hit ? t0 : 0.0;
  depth0[i] = dep;
  double pt[3];
  for (int k = 0; k < 3; ++k) pt[k] = (hit ? r[k] : 0.0) * dep;
  // pose.transform: pts @ R.T + t
  double q[3];
  for (int k = 0; k < 3; ++k)
    q[k] = ((pt[0] * a.R[3 * k] + pt[1] * a.R[3 * k + 1]) + pt[2] * a.R[3 * k + 2]) + a.t[k];
  double px, py;
  const bool v1 = cam_project(a.c1, q[0], q[1], q[2], px, py);
  const bool both = hit && v1;
  corr[2 * i] = both ? px - (double)x : 0.0;
  corr[2 * i + 1] = both ? py - (double)y : 0.0;
  // occlusion: re-cast from camera 1 toward the surface point
  double seg[3];
  for (int k = 0; k < 3; ++k) seg[k] = pt[k] - a.c1w[k];
  const double dist1 = sqrt((seg[0] * seg[0] + seg[1] * seg[1]) + seg[2] * seg[2]);
  const double inv = fmax(dist1, 1e-300);
  double d1[3];
  for (int k = 0; k < 3; ++k) d1[k] = seg[k] / inv;
  const double th = first_hit(a.prims, a.nprims, a.c1w, d1);
  const bool unocc = fabs(th - dist1) <= a.tol * fmax(dist1, 1.0);
  const bool inb = px >= 0.0 && px <= (double)(a.c1.width - 1) && py >= 0.0 &&
                   py <= (double)(a.c1.height - 1) && isfinite(px) && isfinite(py);
  covis[i] = both && unocc && inb;
}

// Polynomial camera 0: call-wide Newton count of the grid (camera.py:177-185).
__global__ void k_grid_iters(Cam c, int* iters) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  int n = 0;
  if (x < c.width && y < c.height) n = poly_conv_iters(c, (double)x, (double)y);
  for (int o = 16; o > 0; o >>= 1) n = max(n, __shfl_xor_sync(0xffffffffu, n, o));
  if ((threadIdx.x & 31) == 0) atomicMax(iters, n);
}

}  // namespace
}  // namespace fsb

using namespace fsb;

extern "C" int fsb_ground_truth(const fsb_rig* rig, const fsb_prim* prims, int32_t nprims,
                                double occlusion_tol, double* depth0, double* corr,
                                uint8_t* covis, void* scratch, size_t scratch_bytes,
                                void* stream) {
  if (!rig || rig->cam0.width < 1 || rig->cam0.height < 1 || nprims < 0 ||
      (nprims > 0 && !prims) || !depth0 || !corr || !covis || !scratch ||
      scratch_bytes < sizeof(int))
    return FSB_EINVAL;
  cudaStream_t st = as_stream(stream);
  TruthArgs a;
  a.c0 = make_cam(rig->cam0);
  a.c1 = make_cam(rig->cam1);
  for (int k = 0; k < 9; ++k) a.R[k] = rig->rotation[k];
  for (int k = 0; k < 3; ++k) a.t[k] = rig->translation[k];
  for (int j = 0; j < 3; ++j)  // camera1_center = -R^T t
    a.c1w[j] = -((a.R[j] * a.t[0] + a.R[3 + j] * a.t[1]) + a.R[6 + j] * a.t[2]);
  a.prims = prims;
  a.nprims = nprims;
  a.tol = occlusion_tol;
  int* iters = static_cast<int*>(scratch);
  const dim3 blk(16, 16), grd = grid2d(a.c0.width, a.c0.height, blk);
  cudaMemsetAsync(iters, 0, sizeof(int), st);
  if (a.c0.model == FSB_CAM_POLYNOMIAL) k_grid_iters<<<grd, blk, 0, st>>>(a.c0, iters);
  k_ground_truth<<<grd, blk, 0, st>>>(a, iters, depth0, corr, covis);
  return launch_status();
}

extern "C" int fsb_render(const fsb_camera* cam, const double rotation[9], const double origin[3],
                          const fsb_prim* prims, int32_t nprims, int32_t supersample,
                          float* image, float* depth, uint8_t* hit, void* stream) {
  if (!cam || cam->width < 1 || cam->height < 1 || !image || nprims < 0 || supersample < 1 ||
      (nprims > 0 && !prims))
    return FSB_EINVAL;
  RenderArgs a;
  a.cam = make_cam(*cam);
  for (int k = 0; k < 9; ++k) a.R[k] = rotation ? rotation[k] : (k % 4 == 0 ? 1.0 : 0.0);
  for (int k = 0; k < 3; ++k) a.origin[k] = origin ? origin[k] : 0.0;
  a.prims = prims;
  a.nprims = nprims;
  a.ss = supersample;
  dim3 blk(16, 16);
  k_render<<<grid2d(cam->width, cam->height, blk), blk, 0, as_stream(stream)>>>(a, image, depth,
                                                                               hit);
  return launch_status();
}
