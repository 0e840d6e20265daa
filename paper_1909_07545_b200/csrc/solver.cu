// Native host driver: solve_level and solve_pyramid enqueue the whole frame on
// one stream (no host sync, no allocation), so a frame can be captured into a
// CUDA graph once and replayed. Workspace is caller-owned and carved here.
//
// Reference: solver.py:306-367 (solve_level), solver.py:401-452 (solve_pyramid),
// fields.py:159-167 (translation_only_rig), camera.py:66-77 (scaled_to).

#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "fsb_common.cuh"
#include "pd_args.cuh"

namespace fsb {
void set_early_output_event64(cudaEvent_t ev);  // pd64.cu
}  // namespace fsb

namespace fsb {

// defined in the other translation units
int trajectory_field_internal(const fsb_camera* cam, const double t[3], double eps_scale,
                              double depth, float* dirs, uint8_t* ok, void* scratch,
                              size_t scratch_bytes, cudaStream_t st);
size_t traj_scratch_bytes_internal(int w, int h);
int fov_mask_internal(const fsb_camera* cam, uint8_t* mask, int* iters, cudaStream_t st);
int calibrate_internal(const fsb_rig* rig, const float* i1, const uint8_t* mask1, float* i1c,
                       uint8_t* ok, int* iters0, cudaStream_t st);
int pyramid_shapes_internal(int h, int w, int levels, double scale, int min_width, int* shapes,
                            int max_levels);
int downsample_internal(const float* src, const uint8_t* mask, int fh, int fw, float* dst,
                        uint8_t* dmask, int ch, int cw, cudaStream_t st);
int upsample_internal(const float* u, const float* wv, const uint8_t* mask, int sh, int sw,
                      const uint8_t* dmask, int dh, int dw, float* uo, float* wo, cudaStream_t st);
size_t level_setup_scratch_internal(int h, int w);
int level_setup_internal(const fsb_level* lv, const fsb_params* prm, void* scratch,
                         size_t scratch_bytes, cudaStream_t st);
int pd_iterate_internal(const fsb_level* L, const fsb_params* prm, int iters, float* diag_p,
                        float* diag_q, cudaStream_t st);
int warp_linearize_internal(const fsb_level* L, cudaStream_t st);
int warp_finish_internal(const fsb_level* L, const fsb_params* prm, float* dmax, double* dmean,
                         cudaStream_t st);
size_t level_partials_internal(int h, int w);
int warp_sample_internal(const fsb_level* L, cudaStream_t st);
int pack_level_internal(const fsb_level* L, cudaStream_t st);
int mask_to_float_internal(const uint8_t* m, size_t n, float* f, cudaStream_t st);
int warp_prologue_internal(const fsb_level* L, cudaStream_t st);
int mean_finish_internal(const double* partials, int nparts, const uint8_t* mask, size_t n,
                         double* out, cudaStream_t st);


namespace {

constexpr int kMaxLevels = 32;

bool params_ok(const fsb_params* p) {
  // SolverParams.__post_init__ (solver.py:63-69) plus the pyramid checks of
  // pyramid_shapes (rasters.py:210-213).
  if (!p) return false;
  if (!(p->lam > 0 && p->alpha0 > 0 && p->alpha1 > 0 && p->beta > 0 && p->eta > 0)) return false;
  if (!(p->du_max > 0)) return false;
  if (p->warp_iters < 1 || p->pd_iters < 1) return false;
  if (p->pyramid_levels < 1 || !(p->pyramid_scale > 1.0)) return false;
  if (p->regularizer < FSB_REG_TGV || p->regularizer > FSB_REG_HUBER) return false;
  if (p->regularizer == FSB_REG_HUBER && !(p->huber_eps > 0)) return false;
  return true;
}

bool cam_valid(const fsb_camera& c) {
  return c.width > 0 && c.height > 0 && c.model >= FSB_CAM_PINHOLE &&
         c.model <= FSB_CAM_POLYNOMIAL;
}

fsb_camera scaled_to(const fsb_camera& c, int h, int w) {  // camera.py:66-77
  fsb_camera o = c;
  double sx = (double)w / (double)c.width, sy = (double)h / (double)c.height;
  o.width = w; o.height = h;
  o.fx = c.fx * sx; o.fy = c.fy * sy;
  o.cx = (c.cx + 0.5) * sx - 0.5;
  o.cy = (c.cy + 0.5) * sy - 0.5;
  return o;
}

// translation_only_rig (fields.py:159-167): t_res = R^T t
void residual_translation(const fsb_rig& r, double t[3]) {
  for (int i = 0; i < 3; ++i)
    t[i] = (r.rotation[0 * 3 + i] * r.translation[0] + r.rotation[1 * 3 + i] * r.translation[1]) +
           r.rotation[2 * 3 + i] * r.translation[2];
}

// Bump allocator over the caller's workspace (sizing pass when base == nullptr).
struct Carve {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    size_t bytes = align_up(count * sizeof(T));
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += bytes;
    return p;
  }
};

struct LevelState {  // state buffers sized for the finest level, reused per level
  float* state_a;  // 12 planes u, u_bar, v x2, v_bar x2, p x2, q x4 (plane stride = level n)
  float* state_b;  // ping-pong copy
  float* consts[kMaxLevels];    // per level: 10 planes T x3, steps x3, iu, rho0, u_omega, maskf
  float* carry_u;  // previous level's u for upsample_state
  float* wv[2];
  float *i1w, *dirs;
  uint8_t *i1w_ok, *dir_ok;
  double* partials;
  float* packed[kMaxLevels];    // per level gather tables (filled ahead on the side stream)
  uint8_t* full16[kMaxLevels];
  int* tiles;
};

struct Plan {
  int nlev;
  int shapes[2 * kMaxLevels];  // finest first
  size_t n0;                   // finest pixel count
  // frame buffers
  uint8_t *mask0, *mask1, *i1c_ok, *solve_mask;
  int* iters;  // 4 ints of Newton-count scratch
  float *lvl_i0[kMaxLevels], *lvl_i1[kMaxLevels];
  uint8_t* lvl_mask[kMaxLevels];
  float* traj[kMaxLevels];
  uint8_t* traj_ok[kMaxLevels];
  void* traj_scratch;
  size_t traj_scratch_bytes;
  void* setup_scratch;
  size_t setup_scratch_bytes;
  LevelState st;
  size_t bytes;
};

int make_plan(const fsb_rig* rig, const fsb_params* prm, void* base, Plan& P) {
  const int H = rig->cam0.height, W = rig->cam0.width;
  int n = pyramid_shapes_internal(H, W, prm->pyramid_levels, prm->pyramid_scale, prm->min_width,
                                  P.shapes, kMaxLevels);
  if (n < 1) return FSB_EINVAL;
  if (n > kMaxLevels) return FSB_EINVAL;
  P.nlev = n;
  P.n0 = (size_t)H * W;
  const size_t n0 = P.n0, n1 = (size_t)rig->cam1.height * rig->cam1.width;
  Carve c{static_cast<char*>(base)};
  P.mask0 = c.take<uint8_t>(n0);
  P.mask1 = c.take<uint8_t>(n1);
  P.i1c_ok = c.take<uint8_t>(n0);
  P.solve_mask = c.take<uint8_t>(n0);
  P.iters = c.take<int>(64);
  for (int l = 0; l < n; ++l) {
    size_t np = (size_t)P.shapes[2 * l] * P.shapes[2 * l + 1];
    P.lvl_i0[l] = l == 0 ? nullptr : c.take<float>(np);
    P.lvl_i1[l] = l == 0 ? nullptr : c.take<float>(np);
    P.lvl_mask[l] = l == 0 ? nullptr : c.take<uint8_t>(np);
    P.traj[l] = c.take<float>(2 * np);
    P.traj_ok[l] = c.take<uint8_t>(np);
  }
  P.traj_scratch_bytes = traj_scratch_bytes_internal(W, H);
  P.traj_scratch = c.take<char>(P.traj_scratch_bytes);
  P.setup_scratch_bytes = level_setup_scratch_internal(H, W);
  P.setup_scratch = c.take<char>(P.setup_scratch_bytes);
  LevelState& s = P.st;
  for (int k = 0; k < 2; ++k) s.wv[k] = c.take<float>(2 * n0);
  s.state_a = c.take<float>(12 * n0);
  for (int l = 0; l < n; ++l) {
    const size_t np = (size_t)P.shapes[2 * l] * P.shapes[2 * l + 1];
    s.consts[l] = c.take<float>(10 * np);
    s.packed[l] = c.take<float>(4 * np);
    s.full16[l] = c.take<uint8_t>(np);
  }
  s.carry_u = c.take<float>(n0);
  s.i1w = c.take<float>(n0);
  s.dirs = c.take<float>(2 * n0);
  s.i1w_ok = c.take<uint8_t>(n0);
  s.dir_ok = c.take<uint8_t>(n0);
  s.partials = c.take<double>(level_partials_internal(H, W) + 64);
  s.state_b = c.take<float>(12 * n0);
  s.tiles = c.take<int>(pd_tma_partials(W, H, 10) + 1);
  P.bytes = c.off;
  return FSB_OK;
}

__global__ void k_and_mask(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, size_t n,
                           uint8_t* __restrict__ o) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i] && b[i];
}

// Frame outputs of the finest level (solver.py:451-452): u, w copied, v from
// planes to the interleaved (H,W,2) layout, the solve mask.
__global__ void k_outputs(const float* __restrict__ u, const float2* __restrict__ wv,
                          const float* __restrict__ v0, const float* __restrict__ v1,
                          const uint8_t* __restrict__ m, size_t n, float* __restrict__ uo,
                          float2* __restrict__ wo, float2* __restrict__ vo,
                          uint8_t* __restrict__ mo) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uo[i] = u[i];
  wo[i] = wv[i];
  vo[i] = make_float2(v0[i], v1[i]);
  mo[i] = m[i];
}

}  // namespace

size_t level_partials_count(int h, int w) { return level_partials_internal(h, w) + 64; }

namespace {

// PD iterations per launch of the blocked kernel (= its halo). FSB_PD_HALO
// overrides for tuning experiments (1, 2, 3, 4, 5 or 10); FSB_PD_HALO_L =
// "w:R,w:R,..." overrides it per level width.
struct HaloEnv {
  int env = 0;
  int lw[16], lr[16], nl = 0;
};

// parsed once (thread-safe function-local static: concurrent solves on
// several streams never see a half-parsed per-level list)
const HaloEnv& halo_env() {
  static const HaloEnv cfg = [] {
    HaloEnv c;
    const char* e = getenv("FSB_PD_HALO");
    c.env = e ? atoi(e) : 0;
    const char* l = getenv("FSB_PD_HALO_L");
    while (l && *l && c.nl < 16) {
      int a, b, n = 0;
      if (sscanf(l, "%d:%d%n", &a, &b, &n) != 2) break;
      c.lw[c.nl] = a; c.lr[c.nl] = b; ++c.nl;
      l += n;
      if (*l == ',') ++l;
    }
    return c;
  }();
  return cfg;
}

int pd_halo(int K, int w = 0, int hgt = 0) {
  const HaloEnv& E = halo_env();
  const int env = E.env, nl = E.nl;
  const int* lw = E.lw;
  const int* lr = E.lr;
  int h = env > 0 ? env : 5;
  // A level whose 10-cycle tiles (44 x 12 interiors) fit in one wave runs each
  // warp's K = 10 cycles in one launch: at these sizes the per-launch cost
  // (exposed tile load, launch gap) outweighs the extra halo (C3 256^2: -10 %).
  if (env <= 0 && K >= 10 && w > 0 && (int)pd_tma_partials(w, hgt, 10) <= pd_num_sms()) h = 10;
  for (int i = 0; i < nl; ++i)
    if (lw[i] == w) h = lr[i];
  if (K < h) h = K <= 1 ? 1 : (K == 2 ? 2 : (K == 3 ? 3 : (K == 4 ? 4 : 5)));
  return h;
}

// Blocked PD kernel: packed pixel pairs (default) or the per-pixel tile kernel.
int pd_launch(const BlockArgs& A, int halo, bool lin, bool fin, cudaStream_t st, int* nblocks) {
  static const int which = [] {  // FSB_PD_KERNEL=block; otherwise the pixel-pair kernel
    const char* e = getenv("FSB_PD_KERNEL");
    return (e && strcmp(e, "block") == 0) ? 1 : 0;
  }();
  return which ? pd_block_launch(A, halo, lin, fin, st, nblocks)
               : pd_pair_launch(A, halo, lin, fin, st, nblocks);
}

// The persistent TMA kernel needs plane blocks (see fsb_level in fsb200.h).
bool tma_layout(const fsb_level* L) {
  const size_t n = (size_t)L->h * L->w;
  if (!L->state_b || !L->maskf || L->w % 4 != 0) return false;
  const float* u = L->u;
  if (L->u_bar != u + n || L->v != u + 2 * n || L->v_bar != u + 4 * n || L->p != u + 6 * n ||
      L->q != u + 8 * n)
    return false;
  const float* c = L->tensor;
  if (L->steps != c + 3 * n || L->iu != c + 6 * n || L->rho0 != c + 7 * n ||
      L->u_omega != c + 8 * n || L->maskf != c + 9 * n)
    return false;
  static const bool env = [] {  // FSB_PD_KERNEL=pair|block disables TMA
    const char* e = getenv("FSB_PD_KERNEL");
    return !(e && strcmp(e, "tma") != 0);
  }();
  return env;
}

StateSet set_a(const fsb_level* L) {
  return StateSet{L->u, L->u_bar, L->v, L->v_bar, L->p, L->q};
}
StateSet set_b(const fsb_level* L) {
  const size_t n = (size_t)L->h * L->w;
  float* B = L->state_b;
  return StateSet{B, B + n, B + 2 * n, B + 4 * n, B + 6 * n, B + 8 * n};
}

void copy_set(const StateSet& d, const StateSet& s, size_t n, cudaStream_t st) {
  cudaMemcpyAsync(d.u, s.u, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(d.ub, s.ub, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(d.v, s.v, 2 * n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(d.vb, s.vb, 2 * n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(d.p, s.p, 2 * n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(d.q, s.q, 4 * n * sizeof(float), cudaMemcpyDeviceToDevice, st);
}

// The warp loop with the temporally blocked kernel: per warp ceil(K / halo)
// launches, the first fusing the linearisation, the last the clip/accumulate
// epilogue and the next warp's samples (solver.py:331-365).
int warp_loop_blocked(const fsb_level* L, const fsb_params* prm, const fsb_diag* diag,
                      int64_t pd_off, int64_t warp_off, cudaStream_t st) {
  const size_t n = (size_t)L->h * L->w;
  const int N = prm->warp_iters, K = prm->pd_iters;
  StateSet sets[2] = {set_a(L), set_b(L)};
  TmaMaps maps;
  const bool tma = tma_layout(L) && pd_tma_maps(&maps, L->u, L->state_b, L->tensor, L->w, L->h);
  int halo = pd_halo(K, L->w, L->h);
  if (!tma && halo > 5) halo = 5;  // the fallback kernels stop at R = 5
  int cur = 0;
  BlockArgs A;
  memset(&A, 0, sizeof(A));
  A.h = L->h; A.w = L->w; A.n = n;
  A.mask = L->mask; A.T = L->tensor; A.S = L->steps;
  A.iu = L->iu; A.rho0 = L->rho0; A.u_omega = L->u_omega;
  A.lam = (float)prm->lam; A.alpha0 = (float)prm->alpha0; A.alpha1 = (float)prm->alpha1;
  A.theta = (float)prm->theta; A.sigma_q = (float)sigma_q_of(prm);
  A.huber_eps = (float)huber_eps_of(prm);
  A.du_max = (float)prm->du_max;
  A.wv = L->wv; A.dirs = L->dirs;
  A.partials = L->partials;
  const bool dpq = diag && diag->max_p_norm && diag->max_q_norm;
  const bool ddu = diag && diag->max_du && diag->mean_abs_du;
  int rc = FSB_OK;
  if (tma && L->tiles) {
    // Skip tiles without mask pixels. Their state is constant for the whole
    // level (v, p, q = 0 and u fixed outside the mask), so both ping-pong sets
    // and u_omega must hold it from the start; partial sums of skipped tiles
    // stay zero.
    rc = pd_tma_tile_list(L->mask, L->w, L->h, halo, L->tiles, st);
    if (rc) return rc;
    copy_set(sets[1], sets[0], n, st);
    cudaMemcpyAsync(L->u_omega, L->u, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
    if (ddu) cudaMemsetAsync(L->partials, 0, pd_tma_partials(L->w, L->h, halo) * sizeof(double), st);
    A.tile_list = L->tiles;
  }
  for (int wi = 0; wi < N; ++wi) {
    rc = warp_prologue_internal(L, st);  // samples at x + w, I_u, rho0 (solver.py:332-343)
    if (rc) return rc;
    int done = 0, nblocks = 0;
    while (done < K) {
      const int it = K - done < halo ? K - done : halo;
      const bool lin = done == 0, fin = done + it == K;
      A.src = sets[cur]; A.dst = sets[cur ^ 1];
      A.iters = it;
      A.diag_p = dpq ? diag->max_p_norm + pd_off + (int64_t)wi * K + done : nullptr;
      A.diag_q = dpq ? diag->max_q_norm + pd_off + (int64_t)wi * K + done : nullptr;
      A.diag_du = (fin && ddu) ? diag->max_du + warp_off + wi : nullptr;
      A.store_bars = wi == N - 1;
      rc = tma ? pd_tma_launch(A, maps, cur, halo, lin, fin, st, &nblocks)
               : pd_launch(A, halo, lin, fin, st, &nblocks);
      if (rc) return rc;
      cur ^= 1;
      done += it;
    }
    if (ddu) {
      rc = mean_finish_internal(L->partials, nblocks, L->mask, n,
                                diag->mean_abs_du + warp_off + wi, st);
      if (rc) return rc;
    }
  }
  if (cur != 0) copy_set(sets[0], sets[1], n, st);
  return launch_status();
}

// Level setup (tensor, steps) plus the gather tables when the level has them.
int level_prepare(const fsb_level* L, const fsb_params* prm, void* scratch, size_t scratch_bytes,
                  cudaStream_t st) {
  int rc = level_setup_internal(L, prm, scratch, scratch_bytes, st);
  if (rc) return rc;
  if (L->packed && L->full16) return pack_level_internal(L, st);
  return FSB_OK;
}

// `iters` plain PD cycles with the blocked kernel (no fused prologue/epilogue);
// the result ends in the primary state set.
int pd_iterate_blocked(const fsb_level* L, const fsb_params* prm, int iters, float* dp, float* dq,
                       cudaStream_t st) {
  const size_t n = (size_t)L->h * L->w;
  const int halo = pd_halo(iters);
  StateSet sets[2] = {set_a(L), set_b(L)};
  TmaMaps maps;
  const bool tma = tma_layout(L) && pd_tma_maps(&maps, L->u, L->state_b, L->tensor, L->w, L->h);
  BlockArgs A;
  memset(&A, 0, sizeof(A));
  A.h = L->h; A.w = L->w; A.n = n;
  A.mask = L->mask; A.T = L->tensor; A.S = L->steps;
  A.iu = L->iu; A.rho0 = L->rho0; A.u_omega = L->u_omega;
  A.lam = (float)prm->lam; A.alpha0 = (float)prm->alpha0; A.alpha1 = (float)prm->alpha1;
  A.theta = (float)prm->theta; A.sigma_q = (float)sigma_q_of(prm);
  A.huber_eps = (float)huber_eps_of(prm);
  A.du_max = (float)prm->du_max;
  if (tma) {  // per-stage entry: the level setup has not filled maskf
    int rc = mask_to_float_internal(L->mask, n, L->maskf, st);
    if (rc) return rc;
  }
  int cur = 0, done = 0;
  while (done < iters) {
    const int it = iters - done < halo ? iters - done : halo;
    A.src = sets[cur]; A.dst = sets[cur ^ 1];
    A.iters = it;
    A.diag_p = (dp && dq) ? dp + done : nullptr;
    A.diag_q = (dp && dq) ? dq + done : nullptr;
    int rc = tma ? pd_tma_launch(A, maps, cur, halo, false, false, st, nullptr)
                 : pd_launch(A, halo, false, false, st, nullptr);
    if (rc) return rc;
    cur ^= 1;
    done += it;
  }
  if (cur != 0) copy_set(sets[0], sets[1], n, st);
  return launch_status();
}

}  // namespace

int solve_level_internal(const fsb_level* L, const fsb_params* prm, const fsb_diag* diag,
                         int64_t pd_off, int64_t warp_off, void* scratch, size_t scratch_bytes,
                         cudaStream_t st, bool prepared = false) {
  const size_t n = (size_t)L->h * L->w;
  int rc = prepared ? FSB_OK : level_prepare(L, prm, scratch, scratch_bytes, st);
  if (rc) return rc;
  // solver.py:323-327: v, p, q, v_bar start at zero, u_bar = u
  cudaMemsetAsync(L->v, 0, 2 * n * sizeof(float), st);
  cudaMemsetAsync(L->v_bar, 0, 2 * n * sizeof(float), st);
  cudaMemsetAsync(L->p, 0, 2 * n * sizeof(float), st);
  cudaMemsetAsync(L->q, 0, 4 * n * sizeof(float), st);
  cudaMemcpyAsync(L->u_bar, L->u, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  if (L->state_b && L->packed && level_cluster_fits(L->h, L->w, prm->warp_iters))
    return level_cluster_solve(L, prm, diag, pd_off, warp_off, st);
  if (L->state_b)
    return warp_loop_blocked(L, prm, diag, pd_off, warp_off, st);
  const int N = prm->warp_iters, K = prm->pd_iters;
  for (int wi = 0; wi < N; ++wi) {
    rc = warp_linearize_internal(L, st);
    if (rc) return rc;
    float* dp = (diag && diag->max_p_norm) ? diag->max_p_norm + pd_off + (int64_t)wi * K : nullptr;
    float* dq = (diag && diag->max_q_norm) ? diag->max_q_norm + pd_off + (int64_t)wi * K : nullptr;
    rc = pd_iterate_internal(L, prm, K, dp && dq ? dp : nullptr, dp && dq ? dq : nullptr, st);
    if (rc) return rc;
    float* dm = (diag && diag->max_du) ? diag->max_du + warp_off + wi : nullptr;
    double* dmean = (diag && diag->mean_abs_du) ? diag->mean_abs_du + warp_off + wi : nullptr;
    rc = warp_finish_internal(L, prm, dm && dmean ? dm : nullptr, dm && dmean ? dmean : nullptr,
                              st);
    if (rc) return rc;
  }
  return FSB_OK;
}

namespace {

// Side stream of a caller stream (one per device and caller stream, created on
// first use and kept): the per-level setup of every level (trajectory field,
// tensor, steps, gather tables) runs there, ahead of and concurrently with the
// level solves on the caller's stream, which wait on one event per level. The
// coarse levels (64^2 - 256^2) leave most SMs idle, so the finer levels'
// setup fills them. Works eagerly and under stream capture (fork / join by
// events). FSB_OVERLAP=0 keeps everything on the caller's stream.
struct SideCtx {
  int dev;
  cudaStream_t main, side;
  cudaEvent_t ev[kMaxLevels + 2];
};

SideCtx* side_ctx(cudaStream_t main) {
  static const bool off = [] {
    const char* e = getenv("FSB_OVERLAP");
    return e && e[0] == '0';
  }();
  if (off) return nullptr;
  static std::mutex mu;
  static std::vector<SideCtx*> ctxs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  for (SideCtx* c : ctxs)
    if (c->dev == dev && c->main == main) return c;
  SideCtx* c = new SideCtx();
  c->dev = dev;
  c->main = main;
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    cudaGetLastError();
    return nullptr;
  }
  int made = 0;
  for (cudaEvent_t& e : c->ev) {
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      for (int k = 0; k < made; ++k) cudaEventDestroy(c->ev[k]);
      cudaStreamDestroy(c->side);
      delete c;
      return nullptr;  // callers fall back to the caller's stream
    }
    ++made;
  }
  ctxs.push_back(c);
  return c;
}

}  // namespace

// The caller stream's side stream and its events (kMaxLevels + 2), for the
// float64 driver (pd64.cu); false when FSB_OVERLAP=0 or on failure.
bool side_stream_for(cudaStream_t main, cudaStream_t* side, cudaEvent_t** ev) {
  SideCtx* c = side_ctx(main);
  if (!c) return false;
  *side = c->side;
  *ev = c->ev;
  return true;
}

int solve_pyramid_internal(const fsb_rig* rig, const fsb_params* prm, const float* i0,
                           const float* i1, const float* const* traj_dirs,
                           const uint8_t* const* traj_okv, void* ws, size_t ws_bytes, float* u_out,
                           float* w_out, float* v_out, uint8_t* mask_out, float* i1c,
                           const fsb_diag* diag, cudaStream_t st) {
  if (!rig || !params_ok(prm) || !cam_valid(rig->cam0) || !cam_valid(rig->cam1)) return FSB_EINVAL;
  if (!i0 || !i1 || !ws || !u_out || !w_out || !v_out || !mask_out || !i1c) return FSB_EINVAL;
  if ((traj_dirs == nullptr) != (traj_okv == nullptr)) return FSB_EINVAL;
  Plan P;
  int rc = make_plan(rig, prm, nullptr, P);
  if (rc) return rc;
  if (ws_bytes < P.bytes) return FSB_ENOSPC;
  make_plan(rig, prm, ws, P);
  double t_res[3];
  residual_translation(*rig, t_res);
  if (!traj_dirs && t_res[0] == 0.0 && t_res[1] == 0.0 && t_res[2] == 0.0)
    return FSB_EDOMAIN;  // fields.py:63-66, raised before any work

  const int H = rig->cam0.height, W = rig->cam0.width;
  const size_t n0 = P.n0;
  const int N = prm->warp_iters, K = prm->pd_iters;

  if (diag) {  // max slots start at 0 (atomicMax on non-negative bit patterns)
    int64_t npd = (int64_t)P.nlev * N * K, nw = (int64_t)P.nlev * N;
    if (diag->max_p_norm) cudaMemsetAsync(diag->max_p_norm, 0, npd * sizeof(float), st);
    if (diag->max_q_norm) cudaMemsetAsync(diag->max_q_norm, 0, npd * sizeof(float), st);
    if (diag->max_du) cudaMemsetAsync(diag->max_du, 0, nw * sizeof(float), st);
    if (diag->mean_abs_du) cudaMemsetAsync(diag->mean_abs_du, 0, nw * sizeof(double), st);
  }

  // fork: trajectory fields (rig only) start on the side stream right away
  SideCtx* sc = side_ctx(st);
  cudaStream_t ss = sc ? sc->side : st;
  if (sc) {
    cudaEventRecord(sc->ev[0], st);
    cudaStreamWaitEvent(ss, sc->ev[0], 0);
  }
  auto traj_level = [&](int l) -> int {
    const int h = P.shapes[2 * l], w = P.shapes[2 * l + 1];
    fsb_camera cl = scaled_to(rig->cam0, h, w);
    return trajectory_field_internal(&cl, t_res, prm->epsilon_scale, 1.0, P.traj[l],
                                     P.traj_ok[l], P.traj_scratch, P.traj_scratch_bytes, ss);
  };
  if (!traj_dirs)
    for (int l = P.nlev - 1; l >= 1; --l)
      if ((rc = traj_level(l))) return rc;

  // masks + calibration (solver.py:418-420)
  rc = fov_mask_internal(&rig->cam0, P.mask0, P.iters + 0, st);
  if (rc) return rc;
  rc = fov_mask_internal(&rig->cam1, P.mask1, P.iters + 1, st);
  if (rc) return rc;
  rc = calibrate_internal(rig, i1, P.mask1, i1c, P.i1c_ok, P.iters + 2, st);
  if (rc) return rc;
  k_and_mask<<<(unsigned)((n0 + 255) / 256), 256, 0, st>>>(P.mask0, P.i1c_ok, n0, P.solve_mask);

  // pyramids (solver.py:423-426), finest first in P.shapes
  P.lvl_i0[0] = const_cast<float*>(i0);
  P.lvl_i1[0] = i1c;
  P.lvl_mask[0] = P.solve_mask;
  for (int l = 1; l < P.nlev; ++l) {
    int fh = P.shapes[2 * (l - 1)], fw = P.shapes[2 * (l - 1) + 1];
    int ch = P.shapes[2 * l], cw = P.shapes[2 * l + 1];
    rc = downsample_internal(P.lvl_i0[l - 1], P.lvl_mask[l - 1], fh, fw, P.lvl_i0[l],
                             P.lvl_mask[l], ch, cw, st);
    if (rc) return rc;
    rc = downsample_internal(P.lvl_i1[l - 1], P.lvl_mask[l - 1], fh, fw, P.lvl_i1[l],
                             P.lvl_mask[l], ch, cw, st);
    if (rc) return rc;
  }

  // fsb_level views of every level (coarse -> fine index k)
  LevelState& S = P.st;
  std::vector<fsb_level> lv(P.nlev);
  for (int k = 0; k < P.nlev; ++k) {
    const int l = P.nlev - 1 - k;
    const int h = P.shapes[2 * l], w = P.shapes[2 * l + 1];
    const size_t np = (size_t)h * w;
    fsb_level& L = lv[k];
    memset(&L, 0, sizeof(L));
    float* u = S.state_a;  // plane 0 of the level's state block
    L.h = h; L.w = w;
    L.i0 = P.lvl_i0[l]; L.i1 = P.lvl_i1[l]; L.mask = P.lvl_mask[l];
    L.traj = traj_dirs ? traj_dirs[k] : P.traj[l];
    L.traj_ok = traj_dirs ? traj_okv[k] : P.traj_ok[l];
    L.u = u; L.u_bar = u + np; L.v = u + 2 * np; L.v_bar = u + 4 * np; L.p = u + 6 * np;
    L.q = u + 8 * np;
    L.tensor = S.consts[l]; L.steps = S.consts[l] + 3 * np; L.iu = S.consts[l] + 6 * np;
    L.rho0 = S.consts[l] + 7 * np; L.u_omega = S.consts[l] + 8 * np;
    L.maskf = S.consts[l] + 9 * np;
    L.i1w = S.i1w;
    L.i1w_ok = S.i1w_ok; L.dirs = S.dirs; L.dir_ok = S.dir_ok; L.partials = S.partials;
    L.tiles = S.tiles;
    L.state_b = S.state_b;
    L.packed = S.packed[l]; L.full16 = S.full16[l];
  }
  // side stream: after the pyramids, every level's setup, coarse first, one
  // event per level (the finest trajectory field goes after the coarse setups)
  if (sc) {
    cudaEventRecord(sc->ev[kMaxLevels + 1], st);
    cudaStreamWaitEvent(ss, sc->ev[kMaxLevels + 1], 0);
  }
  for (int k = 0; k < P.nlev; ++k) {
    if (!traj_dirs && k == P.nlev - 1 && (rc = traj_level(0))) return rc;
    rc = level_prepare(&lv[k], prm, P.setup_scratch, P.setup_scratch_bytes, ss);
    if (rc) return rc;
    if (sc) cudaEventRecord(sc->ev[1 + k], ss);
  }

  int64_t pd_off = 0, warp_off = 0;
  int cur = 0;
  int prev_h = 0, prev_w = 0;
  const uint8_t* prev_mask = nullptr;
  for (int k = 0; k < P.nlev; ++k) {
    const int l = P.nlev - 1 - k;  // coarse -> fine
    const int h = P.shapes[2 * l], w = P.shapes[2 * l + 1];
    const size_t np = (size_t)h * w;
    const LevelRange nvtx_range("fsb level %dx%d", w, h);  // NVTX range per level
    float* u = S.state_a;  // plane 0 of the level's state block
    float* wv = S.wv[cur];
    if (k == 0) {
      cudaMemsetAsync(u, 0, np * sizeof(float), st);
      cudaMemsetAsync(wv, 0, 2 * np * sizeof(float), st);
    } else {
      rc = upsample_internal(S.carry_u, S.wv[cur ^ 1], prev_mask, prev_h, prev_w, P.lvl_mask[l],
                             h, w, u, wv, st);
      if (rc) return rc;
    }
    fsb_level L = lv[k];
    L.wv = wv;
    if (sc) cudaStreamWaitEvent(st, sc->ev[1 + k], 0);  // join: this level's setup done
    rc = solve_level_internal(&L, prm, diag, pd_off, warp_off, P.setup_scratch,
                              P.setup_scratch_bytes, st, /*prepared=*/true);
    if (rc) return rc;
    pd_off += (int64_t)N * K;
    warp_off += N;
    prev_h = h; prev_w = w; prev_mask = P.lvl_mask[l];
    if (l > 0) cudaMemcpyAsync(S.carry_u, u, np * sizeof(float), cudaMemcpyDeviceToDevice, st);
    if (l == 0) {
      // one pass: u, w, the v planes interleaved to (H,W,2), mask (two 4-byte-wide
      // cudaMemcpy2DAsync copies for v alone measured 185 us per frame)
      k_outputs<<<(unsigned)((n0 + 255) / 256), 256, 0, st>>>(
          u, reinterpret_cast<const float2*>(wv), L.v, L.v + n0, P.solve_mask, n0, u_out,
          reinterpret_cast<float2*>(w_out), reinterpret_cast<float2*>(v_out), mask_out);
    }
    cur ^= 1;
  }
  (void)H; (void)W;
  return launch_status();
}

size_t solve_pyramid_bytes(const fsb_rig* rig, const fsb_params* prm) {
  if (!rig || !params_ok(prm) || !cam_valid(rig->cam0) || !cam_valid(rig->cam1)) return 0;
  Plan P;
  if (make_plan(rig, prm, nullptr, P)) return 0;
  return P.bytes;
}

}  // namespace fsb

using namespace fsb;

extern "C" {

size_t fsb_level_partials(int32_t h, int32_t w) { return level_partials_count(h, w); }
size_t fsb_level_tiles(int32_t h, int32_t w) { return pd_tma_partials(w, h, 10) + 1; }

int fsb_level_setup(const fsb_level* lv, const fsb_params* prm, void* scratch,
                    size_t scratch_bytes, void* stream) {
  if (!lv || !prm || lv->h < 1 || lv->w < 1) return FSB_EINVAL;
  return level_prepare(lv, prm, scratch, scratch_bytes, as_stream(stream));
}

int fsb_warp_linearize(const fsb_level* lv, void* stream) {
  if (!lv || lv->h < 1 || lv->w < 1) return FSB_EINVAL;
  return warp_linearize_internal(lv, as_stream(stream));
}

int fsb_pd_iterate(const fsb_level* lv, const fsb_params* prm, int32_t iters, float* diag_p,
                   float* diag_q, void* stream) {
  if (!lv || !prm || iters < 0 || lv->h < 1 || lv->w < 1) return FSB_EINVAL;
  if (lv->state_b) return pd_iterate_blocked(lv, prm, iters, diag_p, diag_q, as_stream(stream));
  return pd_iterate_internal(lv, prm, iters, diag_p, diag_q, as_stream(stream));
}

int fsb_warp_finish(const fsb_level* lv, const fsb_params* prm, float* diag_max_du,
                    double* diag_mean_du, void* stream) {
  if (!lv || !prm || lv->h < 1 || lv->w < 1) return FSB_EINVAL;
  return warp_finish_internal(lv, prm, diag_max_du, diag_mean_du, as_stream(stream));
}

int fsb_solve_level(const fsb_level* lv, const fsb_params* prm, const fsb_diag* diag,
                    int64_t diag_pd_offset, int64_t diag_warp_offset, void* scratch,
                    size_t scratch_bytes, void* stream) {
  if (!lv || !params_ok(prm) || lv->h < 1 || lv->w < 1) return FSB_EINVAL;
  return solve_level_internal(lv, prm, diag, diag_pd_offset, diag_warp_offset, scratch,
                              scratch_bytes, as_stream(stream));
}

int fsb_diag_counts(int32_t h, int32_t w, const fsb_params* prm, int64_t* n_pd, int64_t* n_warp) {
  if (!params_ok(prm) || h < 1 || w < 1) return FSB_EINVAL;
  int shapes[2 * 32];
  int n = pyramid_shapes_internal(h, w, prm->pyramid_levels, prm->pyramid_scale, prm->min_width,
                                  shapes, 32);
  if (n < 1) return FSB_EINVAL;
  if (n_pd) *n_pd = (int64_t)n * prm->warp_iters * prm->pd_iters;
  if (n_warp) *n_warp = (int64_t)n * prm->warp_iters;
  return n;
}

size_t fsb_solve_pyramid_workspace_bytes(const fsb_rig* rig, const fsb_params* prm) {
  return solve_pyramid_bytes(rig, prm);
}

int fsb_solve_pyramid(const fsb_rig* rig, const fsb_params* prm, const float* i0, const float* i1,
                      const float* const* traj_dirs, const uint8_t* const* traj_ok,
                      void* workspace, size_t workspace_bytes, float* u, float* w, float* v,
                      uint8_t* mask, float* i1c, const fsb_diag* diag, void* stream) {
  return solve_pyramid_internal(rig, prm, i0, i1, traj_dirs, traj_ok, workspace, workspace_bytes,
                                u, w, v, mask, i1c, diag, as_stream(stream));
}

struct fsb_graph {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  cudaEvent_t early;  // float64 graphs: recorded once mask / i1c are final
};

}  // extern "C"

namespace {
template <typename Enqueue>
int capture_graph(void* stream, fsb_graph** out, int64_t* n_kernels, Enqueue enqueue) {
  if (!out || !stream) return FSB_EINVAL;  // capture needs a non-default stream
  *out = nullptr;
  cudaStream_t st = as_stream(stream);
  side_ctx(st);  // create the side stream / events outside the capture
  cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return (int)e;
  int rc = enqueue(st);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(st, &g);
  if (rc) { if (g) cudaGraphDestroy(g); return rc; }
  if (e != cudaSuccess) return (int)e;
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) cudaGraphGetNodes(g, nodes.data(), &n);
  int64_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nodes[i], &t);
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiate(&ex, g, 0);
  if (e != cudaSuccess) { cudaGraphDestroy(g); return (int)e; }
  fsb_graph* G = new fsb_graph{g, ex, nullptr};
  *out = G;
  if (n_kernels) *n_kernels = k;
  return FSB_OK;
}
}  // namespace

extern "C" {

int fsb_graph_create(const fsb_rig* rig, const fsb_params* prm, const float* i0, const float* i1,
                     const float* const* traj_dirs, const uint8_t* const* traj_ok,
                     void* workspace, size_t workspace_bytes, float* u, float* w, float* v,
                     uint8_t* mask, float* i1c, const fsb_diag* diag, void* stream,
                     fsb_graph** out, int64_t* n_kernels) {
  return capture_graph(stream, out, n_kernels, [&](cudaStream_t st) {
    return solve_pyramid_internal(rig, prm, i0, i1, traj_dirs, traj_ok, workspace,
                                  workspace_bytes, u, w, v, mask, i1c, diag, st);
  });
}

int fsb_graph_create_f64(const fsb_rig* rig, const fsb_params* prm, const double* i0,
                         const double* i1, const double* const* traj_dirs,
                         const uint8_t* const* traj_ok, void* workspace, size_t workspace_bytes,
                         double* u, double* w, double* v, uint8_t* mask, double* i1c,
                         const fsb_diag* diag, void* stream, fsb_graph** out,
                         int64_t* n_kernels) {
  cudaEvent_t early = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&early, cudaEventDisableTiming);
  if (e != cudaSuccess) return (int)e;
  fsb::set_early_output_event64(early);  // recorded inside the capture (pd64.cu)
  const int rc = capture_graph(stream, out, n_kernels, [&](cudaStream_t st) {
    return fsb_solve_pyramid_f64(rig, prm, i0, i1, traj_dirs, traj_ok, workspace,
                                 workspace_bytes, u, w, v, mask, i1c, diag, st);
  });
  fsb::set_early_output_event64(nullptr);
  if (rc) {
    cudaEventDestroy(early);
    return rc;
  }
  (*out)->early = early;
  return FSB_OK;
}

int fsb_graph_launch(fsb_graph* G, void* stream) {
  if (!G) return FSB_EINVAL;
  cudaError_t e = cudaGraphLaunch(G->exec, as_stream(stream));
  return e == cudaSuccess ? FSB_OK : (int)e;
}

int fsb_graph_destroy(fsb_graph* G) {
  if (!G) return FSB_OK;
  cudaGraphExecDestroy(G->exec);
  cudaGraphDestroy(G->graph);
  if (G->early) cudaEventDestroy(G->early);
  delete G;
  return FSB_OK;
}

void* fsb_graph_early_event(fsb_graph* G) { return G ? (void*)G->early : nullptr; }

int fsb_stream_wait_event(void* stream, void* event) {
  if (!event) return FSB_EINVAL;
  const cudaError_t e = cudaStreamWaitEvent(as_stream(stream), (cudaEvent_t)event, 0);
  return e == cudaSuccess ? FSB_OK : (int)e;
}

const char* fsb_version(void) { return "fsb200 0.1 sm_100a"; }

}  // extern "C"
