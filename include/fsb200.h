/*
 * fsb200.h — C ABI of the B200-native dense-mapping hot path of arXiv 1909.07545
 * (non-rectified variational fisheye stereo, anisotropic TGV-L1 along epipolar
 * trajectory fields).
 *
 * The reference package (`fisheyestereo`, pure Python/NumPy) has no FFI layer:
 * its boundary for this path is the Python function
 *     fisheyestereo.solve_pyramid(i0, i1, rig, params, collect_diagnostics=False,
 *                                 traj_override=None) -> StereoResult
 * (reference pkg/src/fisheyestereo/solver.py:401-452) plus the per-stage functions
 * its tests call directly. Every entry point below replaces one of those
 * functions; the replaced reference interface is cited on each declaration.
 * The Python host mirror (paper_1909_07545_b200/) binds these through ctypes.
 *
 * Conventions (all entry points):
 *   - every array argument is a DEVICE pointer owned by the caller; nothing is
 *     allocated inside (scratch is caller-provided, sized by *_bytes helpers);
 *   - images / scalar fields are row-major float32 (H, W); vector fields are
 *     interleaved float32 (H, W, 2) with channel order (x, y); masks are uint8
 *     0/1 (H, W) — the layout of reference rasters.py:1-11;
 *   - work is enqueued asynchronously on `stream` (a cudaStream_t, may be 0);
 *   - the return value is 0 on success, a cudaError_t (> 0) if a launch failed,
 *     or FSB_EINVAL (-1) / FSB_ENOSPC (-2) / FSB_EDOMAIN (-3) for argument errors
 *     (the reference's ValueError cases);
 *   - entry points are stateless and re-entrant; one stream per concurrent solve.
 */
#ifndef FSB200_H_
#define FSB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSB_OK 0
#define FSB_EINVAL (-1)   /* bad shape / null pointer / bad parameter (ValueError) */
#define FSB_ENOSPC (-2)   /* caller-provided scratch/workspace too small          */
#define FSB_EDOMAIN (-3)  /* trajectory field on a rotated or zero-baseline rig   */

#define FSB_CAM_PINHOLE 0     /* reference camera.py:87-106  */
#define FSB_CAM_UNIFIED 1     /* reference camera.py:109-136 */
#define FSB_CAM_POLYNOMIAL 2  /* reference camera.py:139-190 */

/* Lens + image grid; mirrors CameraBase and its subclasses (camera.py:47-190).
 * Distances in pixels, fov = full field-of-view angle in radians. */
typedef struct fsb_camera {
  int32_t model;
  int32_t width;
  int32_t height;
  int32_t reserved;
  double fx, fy, cx, cy, fov;
  double xi;    /* unified model only */
  double k[4];  /* polynomial model only: r/f = k1 t + k2 t^3 + k3 t^5 + k4 t^7 */
} fsb_camera;

/* StereoRig(cam0, cam1, RelativePose(R, t)) with X1 = R X0 + t (camera.py:245-287). */
typedef struct fsb_rig {
  fsb_camera cam0;
  fsb_camera cam1;
  double rotation[9];  /* row-major */
  double translation[3];
} fsb_rig;

/* SolverParams (solver.py:36-69). */
typedef struct fsb_params {
  double lam, alpha0, alpha1, beta, eta;
  int32_t warp_iters, pd_iters;
  double du_max;
  int32_t pyramid_levels;
  int32_t min_width;
  double pyramid_scale;
  double epsilon_scale;
  double tensor_sigma;
  double theta;
  /* Regulariser (extension, parity-unpinned against the TGV-only reference):
   * FSB_REG_TGV alpha1|T grad u - v| + alpha0|grad v| (solver.py:279-303),
   * FSB_REG_TV alpha1|T grad u| (v, q held at 0: tau_v = sigma_q = 0),
   * FSB_REG_HUBER alpha1 Huber_eps(T grad u) (TV with the Huber dual step
   * p <- proj((p + sigma_p alpha1 T grad u_bar) / (1 + sigma_p alpha1 eps))). */
  int32_t regularizer;
  int32_t reserved;
  double huber_eps;
} fsb_params;

enum { FSB_REG_TGV = 0, FSB_REG_TV = 1, FSB_REG_HUBER = 2 };

/* Per-iteration invariants (Diagnostics, solver.py:104-119). Device arrays the
 * caller sizes with fsb_diag_counts(); any pointer may be NULL. */
typedef struct fsb_diag {
  float* max_p_norm;    /* one per primal-dual iteration, all levels  */
  float* max_q_norm;    /* one per primal-dual iteration, all levels  */
  float* max_du;        /* one per warp iteration, all levels         */
  double* mean_abs_du;  /* one per warp iteration, all levels         */
  double* max_du_f64;   /* float64 path: max |du| per warp in float64 (the reference's
                           du_max + 1e-15 bound, test_acceptance.py:249-258); NULL = max_du */
} fsb_diag;

/* ---------------------------------------------------------------- geometry */

/* CameraBase.fov_mask (camera.py:79-84). mask: (cam.height, cam.width) uint8. */
int fsb_fov_mask(const fsb_camera* cam, uint8_t* mask, void* scratch, size_t scratch_bytes,
                 void* stream);
size_t fsb_fov_mask_scratch_bytes(const fsb_camera* cam);

/* camera.unproject / camera.project on n points (camera.py:101,115,126,155,171).
 * pix: (n,2) f64, rays/points: (n,3) f64, valid: (n) u8. Invalid outputs are NaN.
 * The polynomial model iterates Newton until every point of the call converged
 * (camera.py:177-185); scratch holds that convergence count. */
int fsb_unproject(const fsb_camera* cam, const double* pix, int64_t n, double* rays,
                  uint8_t* valid, void* scratch, size_t scratch_bytes, void* stream);
int fsb_project(const fsb_camera* cam, const double* pts, int64_t n, double* pix,
                uint8_t* valid, void* stream);
size_t fsb_unproject_scratch_bytes(void);

/* generate_calibration_field (fields.py:34-45). field: (H,W,2) f64, ok: (H,W) u8. */
int fsb_calibration_field(const fsb_rig* rig, double* field, uint8_t* ok, void* scratch,
                          size_t scratch_bytes, void* stream);

/* calibrate_second_image (solver.py:389-398): i1c = masked bicubic of i1 at
 * x + calibration(x), mask1 = cam1 FOV mask (computed inside when mask1 == NULL).
 * i1: (cam1.height, cam1.width) f32; i1c, ok: cam0 grid. */
int fsb_calibrate_second_image(const fsb_rig* rig, const float* i1, const uint8_t* mask1,
                               float* i1c, uint8_t* ok, void* scratch, size_t scratch_bytes,
                               void* stream);
size_t fsb_calibrate_scratch_bytes(const fsb_rig* rig);

/* trace_epipolar_curves (fields.py:111-139): Euler integration of a (h,w,2)
 * f64 direction field (validity `valid`) from n starts (n,2) f64 for n_steps =
 * ceil(length / step) steps; verts (n, n_steps+1, 2) f64 (NaN after a trace
 * dies), alive (n, n_steps+1) u8. */
int fsb_trace_epipolar_curves(const double* dirs, const uint8_t* valid, int32_t h, int32_t w,
                              const double* starts, int64_t n, int32_t n_steps, double length,
                              double step, double* verts, uint8_t* alive, void* stream);

/* ------------------------------------------------------- post-solve depth */

/* compose_with_calibration (fields.py:170-182): full = w + cal(x + w) where the
 * f64 bicubic of the calibration field under cal_ok is valid, else 0.
 * wv, cal, full: (h,w,2) f64; cal_ok, ok: (h,w) u8. */
int fsb_compose_calibration(const double* wv, const double* cal, const uint8_t* cal_ok, int32_t h,
                            int32_t w, double* full, uint8_t* ok, void* stream);

/* triangulate_midpoint (camera.py:317-343) on n pixel pairs x0 (cam0), x1
 * (cam1), (n,2) f64: distance along the camera-0 ray of the midpoint of the
 * shortest segment between the rays; invalid (NaN, ok = 0) for invalid rays,
 * rays closer to parallel than min_angle, or a midpoint behind camera 0. */
int fsb_triangulate_midpoint(const fsb_rig* rig, const double* x0, const double* x1, int64_t n,
                             double min_angle, double* depth, uint8_t* ok, void* scratch,
                             size_t scratch_bytes, void* stream);
size_t fsb_triangulate_scratch_bytes(void);

/* depth_from_correspondence (evaluate.py:101-114): x1 = x + corr on the cam0
 * grid, triangulated (min_angle 1e-6), ok &= valid, depth = min(depth, cap)
 * where ok else 0. corr: (h,w,2) f64; valid, ok: (h,w) u8; depth (h,w) f64.
 * Scratch: fsb_triangulate_scratch_bytes(). */
int fsb_depth_from_correspondence(const fsb_rig* rig, const double* corr, const uint8_t* valid,
                                  int32_t h, int32_t w, double depth_cap, double* depth,
                                  uint8_t* ok, void* scratch, size_t scratch_bytes, void* stream);

/* generate_trajectory_field (fields.py:48-108) for the translation-only rig
 * (cam, cam, (I, t)); fp64 throughout, dirs stored f32 (H,W,2), ok u8 (H,W).
 * Returns FSB_EDOMAIN for a zero baseline (fields.py:63-66). */
int fsb_trajectory_field(const fsb_camera* cam, const double t[3], double epsilon_scale,
                         double depth, float* dirs, uint8_t* ok, void* scratch,
                         size_t scratch_bytes, void* stream);
size_t fsb_trajectory_scratch_bytes(const fsb_camera* cam);
/* The same with float64 directions (the reference's dtype; the fp64 path's own
 * per-level field). */
int fsb_trajectory_field_f64(const fsb_camera* cam, const double t[3], double epsilon_scale,
                             double depth, double* dirs, uint8_t* ok, void* scratch,
                             size_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------- rasters */

/* sample_bicubic (rasters.py:57-141) with its mask-aware fallback chain.
 * field: (h,w,c) f32 interleaved, c in {1,2}; pos: (n,2) f64 (x,y);
 * out: (n,c) f32 (NaN where invalid); valid: (n) u8. Accumulates in f64 when
 * acc64 != 0, else in f32 (the per-warp hot-path precision). */
int fsb_sample_bicubic(const float* field, int32_t h, int32_t w, int32_t c,
                       const uint8_t* mask, const double* pos, int64_t n, float* out,
                       uint8_t* valid, int32_t acc64, void* stream);

/* gradient / divergence (rasters.py:144-172). u: (h,w); g, p: (h,w,2). */
int fsb_gradient(const float* u, const uint8_t* mask, int32_t h, int32_t w, float* g,
                 void* stream);
int fsb_divergence(const float* p, const uint8_t* mask, int32_t h, int32_t w, float* div,
                   void* stream);

/* smooth_masked (rasters.py:185-191), Gaussian with SciPy's reflect/truncate=4. */
int fsb_smooth_masked(const float* f, const uint8_t* mask, int32_t h, int32_t w,
                      double sigma, float* out, void* scratch, size_t scratch_bytes,
                      void* stream);
size_t fsb_smooth_scratch_bytes(int32_t h, int32_t w);

/* pyramid_shapes (rasters.py:207-221): writes up to max_levels (h,w) pairs,
 * finest first; returns the level count or FSB_EINVAL. Host-only. */
int fsb_pyramid_shapes(int32_t h, int32_t w, int32_t levels, double scale, int32_t min_width,
                       int32_t* shapes, int32_t max_levels);

/* downsample_area (rasters.py:228-260). */
int fsb_downsample_area(const float* src, const uint8_t* mask, int32_t fh, int32_t fw,
                        float* dst, uint8_t* dmask, int32_t ch, int32_t cw, void* stream);

/* upsample_state (rasters.py:276-297). */
int fsb_upsample_state(const float* u, const float* wv, const uint8_t* mask, int32_t sh,
                       int32_t sw, const uint8_t* dmask, int32_t dh, int32_t dw,
                       float* u_out, float* w_out, void* stream);

/* ---------------------------------------------------------------- solver */

/* Device view of one pyramid level's solver buffers (all (h,w) f32 planes
 * unless noted; pitch == w). Filled by the caller (or fsb_level_bind). */
typedef struct fsb_level {
  int32_t h, w;
  const float* i0;       /* level image 0                                 */
  const float* i1;       /* level (calibrated) image 1                    */
  const uint8_t* mask;   /* level solve mask                              */
  const float* traj;     /* (h,w,2) trajectory directions                 */
  const uint8_t* traj_ok;
  float* tensor;         /* 3 planes a,b,c    (compute_tensor)            */
  float* steps;          /* 3 planes sigma_p, tau_u, tau_v                */
  float* u;  float* u_bar;
  float* v;  float* v_bar;  /* 2 planes each                              */
  float* p;              /* 2 planes                                       */
  float* q;              /* 4 planes                                       */
  float* wv;             /* (h,w,2) accumulated warp                       */
  float* u_omega;
  float* iu;  float* rho0;
  float* i1w;            /* warped image                                   */
  uint8_t* i1w_ok;       /* warp_ok & mask                                 */
  float* dirs;           /* (h,w,2) sampled unit directions                */
  uint8_t* dir_ok;
  double* partials;      /* reduction scratch (fsb_level_partials(h,w))    */
  /* Optional second state set of 12 planes (u, u_bar, v x2, v_bar x2, p x2,
   * q x4) for the ping-pong of the temporally blocked PD kernel; NULL selects
   * the one-iteration-per-launch kernels. */
  float* state_b;
  /* Optional gather fast path: (h,w,4) {i1, traj.x, traj.y, 0} and a byte map
   * whose bit0 / bit1 say all 16 bicubic taps around (x,y) are in bounds and in
   * mask / traj_ok (filled by fsb_level_setup when non-NULL). */
  float* packed;
  uint8_t* full16;
  /* Optional 0/1 float copy of `mask` (filled by fsb_level_setup when non-NULL).
   * When u, u_bar, v, v_bar, p, q form one block of 12 planes of stride h*w,
   * state_b likewise, tensor, steps, iu, rho0, u_omega, maskf one block of 10
   * planes, and w % 4 == 0, the PD iterations run in the persistent TMA kernel. */
  float* maskf;
  /* Optional int32 scratch of fsb_level_tiles(h,w) entries. When non-NULL,
   * solve_level's TMA path lists the PD tiles whose interior holds a solve-mask
   * pixel and skips the others: outside the mask the edges are zero and I_u is
   * zero, so v, p, q stay 0 and u stays constant there (solver.py:279-303), and
   * a skipped tile's result is its input. */
  int32_t* tiles;
} fsb_level;

size_t fsb_level_partials(int32_t h, int32_t w);
size_t fsb_level_tiles(int32_t h, int32_t w);

/* compute_tensor(smooth_masked(i0)) + precondition_steps (solver.py:319-321,
 * 122-161, 246-276). scratch >= fsb_smooth_scratch_bytes(h,w). */
int fsb_level_setup(const fsb_level* lv, const fsb_params* prm, void* scratch,
                    size_t scratch_bytes, void* stream);

/* compute_tensor (solver.py:122-141) on an already-smoothed image; tensor
 * out: 3 planes a,b,c. */
int fsb_compute_tensor(const float* smoothed, const uint8_t* mask, int32_t h, int32_t w,
                       double beta, double eta, float* tensor, void* scratch,
                       size_t scratch_bytes, void* stream);

/* precondition_steps (solver.py:246-276) from tensor planes; steps out: 3 planes
 * sigma_p, tau_u, tau_v (sigma_q = 1 / (2 alpha0) is a scalar). */
int fsb_precondition_steps(const float* tensor, const uint8_t* mask, int32_t h, int32_t w,
                           const fsb_params* prm, float* steps, void* scratch,
                           size_t scratch_bytes, void* stream);

/* Warp-loop prologue (solver.py:332-346 with image_derivative_along 192-202):
 * i1w, dirs, I_u, rho0, and the u_omega / u_bar / v_bar resets. */
int fsb_warp_linearize(const fsb_level* lv, void* stream);

/* `iters` calls of primal_dual_iterate (solver.py:279-303). diag_p/diag_q, if
 * non-NULL, receive one max-norm per iteration (solver.py:350-354). */
int fsb_pd_iterate(const fsb_level* lv, const fsb_params* prm, int32_t iters, float* diag_p,
                   float* diag_q, void* stream);

/* thresholding_step (solver.py:205-218), elementwise on n f64 values (the same
 * device function runs fused, in f32, inside the primal kernel). */
int fsb_thresholding_step(const double* u_hat, const double* rho_hat, const double* iu,
                          const double* tau_u, double lam, int64_t n, double* out, void* stream);

/* Warp-loop epilogue (solver.py:356-365): clip, accumulate u and w. */
int fsb_warp_finish(const fsb_level* lv, const fsb_params* prm, float* diag_max_du,
                    double* diag_mean_du, void* stream);

/* solve_level (solver.py:306-367): setup + N warps of (linearize, K PD, finish).
 * u and wv hold the initial WarpState on entry and the result on exit; v, p, q,
 * u_bar, v_bar are (re)initialised inside as the reference does. */
int fsb_solve_level(const fsb_level* lv, const fsb_params* prm, const fsb_diag* diag,
                    int64_t diag_pd_offset, int64_t diag_warp_offset, void* scratch,
                    size_t scratch_bytes, void* stream);

/* ---------------------------------------------------------------- pyramid */

/* Number of levels / diagnostic slots for a frame of the given size. */
int fsb_diag_counts(int32_t h, int32_t w, const fsb_params* prm, int64_t* n_pd,
                    int64_t* n_warp);

/* Workspace for fsb_solve_pyramid. */
size_t fsb_solve_pyramid_workspace_bytes(const fsb_rig* rig, const fsb_params* prm);

/* solve_pyramid (solver.py:401-452), whole frame on device.
 * i0: cam0 grid f32; i1: cam1 grid f32. Outputs on the cam0 grid:
 * u (H,W), w (H,W,2), v (H,W,2), mask (H,W) u8, i1c (H,W).
 * traj_dirs / traj_ok: optional per-level override arrays (coarsest first,
 * level sizes from fsb_pyramid_shapes), i.e. the reference's traj_override
 * (solver.py:437-438); pass NULL to generate trajectory fields on device.
 * diag may be NULL. */
int fsb_solve_pyramid(const fsb_rig* rig, const fsb_params* prm, const float* i0,
                      const float* i1, const float* const* traj_dirs,
                      const uint8_t* const* traj_ok, void* workspace, size_t workspace_bytes,
                      float* u, float* w, float* v, uint8_t* mask, float* i1c,
                      const fsb_diag* diag, void* stream);

/* float64 path of solve_pyramid (the default, credited path): float64 images
 * in, float64 fields out, float64 storage and arithmetic in the reference's
 * operation order (temporally blocked primal-dual tiles). Holds the north-star
 * disparity gate against the reference at every configuration including C3 at
 * N=50 (tests/test_gpu_c3_parity.py); the fp32 fsb_solve_pyramid is faster but
 * misses the p99 gate at N=50. */
size_t fsb_solve_pyramid_f64_workspace_bytes(const fsb_rig* rig, const fsb_params* prm);
int fsb_solve_pyramid_f64(const fsb_rig* rig, const fsb_params* prm, const double* i0,
                          const double* i1, const double* const* traj_dirs,
                          const uint8_t* const* traj_ok, void* workspace, size_t workspace_bytes,
                          double* u, double* w, double* v, uint8_t* mask, double* i1c,
                          const fsb_diag* diag, void* stream);

/* Warp prologue of the float64 path (solver.py:332-346 + image_derivative_along
 * 192-202) on one level, for the per-stage gate: i1w = B(I1, x + w), dirs =
 * B(traj, x + w) renormalised, I_u, rho0. All (h,w[,2]) f64 / u8 device arrays;
 * i1w and dirs are 0 where invalid (i1w_ok, dir_ok), i1w / dirs / iu / rho0 are 0
 * off the mask. kind 0: masked-gather kernels (k64_sample / k64_linearize, the
 * large levels); kind 1: NaN-encoded texel kernels (sample64.cu, levels up to
 * 256^2). scratch: fsb_warp_linearize_f64_scratch_bytes, 32-byte aligned. */
size_t fsb_warp_linearize_f64_scratch_bytes(int32_t h, int32_t w);
int fsb_warp_linearize_f64(int32_t h, int32_t w, const double* i0, const double* i1,
                           const uint8_t* mask, const double* traj, const uint8_t* traj_ok,
                           const double* wv, double* i1w, uint8_t* i1w_ok, double* dirs,
                           uint8_t* dir_ok, double* iu, double* rho0, void* scratch,
                           size_t scratch_bytes, int32_t kind, void* stream);

/* Live kernel timing for the roofline (bench.py): a phase timer records, on
 * the solve stream, three CUDA events per warp iteration of one pyramid level
 * (`level` 0 = finest, up to `max_warps` warps): before the warp's sampling
 * kernels (solver.py:332-346), between sampling and its primal-dual launches
 * (solver.py:347-360), and after the last primal-dual launch. After the
 * stream is synchronised, fsb_phase_timer_read returns the summed sampling and
 * primal-dual milliseconds, the warps recorded, the PD launches per warp and
 * the level shape. fsb_solve_pyramid_f64_timed is fsb_solve_pyramid_f64
 * (no override, no diagnostics) with the timer attached; not for capture. */
typedef struct fsb_phase_timer fsb_phase_timer;
int fsb_phase_timer_create(int32_t level, int32_t max_warps, fsb_phase_timer** out);
int fsb_phase_timer_read(fsb_phase_timer* timer, double* sample_ms, double* pd_ms,
                         int32_t* warps, int32_t* pd_launches_per_warp, int32_t* level_h,
                         int32_t* level_w);
int fsb_phase_timer_destroy(fsb_phase_timer* timer);
int fsb_solve_pyramid_f64_timed(const fsb_rig* rig, const fsb_params* prm, const double* i0,
                                const double* i1, void* workspace, size_t workspace_bytes,
                                double* u, double* w, double* v, uint8_t* mask, double* i1c,
                                fsb_phase_timer* timer, void* stream);

/* CUDA-graph form of fsb_solve_pyramid: captures one frame (same arguments,
 * fixed buffers) on `stream` into an executable graph; *n_kernels receives the
 * number of kernel nodes per frame. Replay with fsb_graph_launch. */
typedef struct fsb_graph fsb_graph;
int fsb_graph_create(const fsb_rig* rig, const fsb_params* prm, const float* i0, const float* i1,
                     const float* const* traj_dirs, const uint8_t* const* traj_ok,
                     void* workspace, size_t workspace_bytes, float* u, float* w, float* v,
                     uint8_t* mask, float* i1c, const fsb_diag* diag, void* stream,
                     fsb_graph** graph, int64_t* n_kernels);
/* The same for the float64 path (fsb_solve_pyramid_f64's arguments). */
int fsb_graph_create_f64(const fsb_rig* rig, const fsb_params* prm, const double* i0,
                         const double* i1, const double* const* traj_dirs,
                         const uint8_t* const* traj_ok, void* workspace, size_t workspace_bytes,
                         double* u, double* w, double* v, uint8_t* mask, double* i1c,
                         const fsb_diag* diag, void* stream, fsb_graph** out,
                         int64_t* n_kernels);
int fsb_graph_launch(fsb_graph* graph, void* stream);
int fsb_graph_destroy(fsb_graph* graph);
/* float64 graphs: an event (cudaEvent_t, owned by the graph; NULL for float32
 * graphs) that each replay records as soon as `mask` and `i1c` hold their final
 * values (after the calibration, long before u / w / v), so the host can copy
 * those two outputs out while the frame is still solving. No reference
 * counterpart: an API-level latency optimisation of solve_pyramid's outputs
 * (solver.py:451-452). */
void* fsb_graph_early_event(fsb_graph* graph);
/* cudaStreamWaitEvent(stream, event, 0) for callers without a CUDA binding. */
int fsb_stream_wait_event(void* stream, void* event);

/* ---------------------------------------------------------------- synthetic inputs */

#define FSB_PRIM_PLANE 0   /* synth.py:124-138 */
#define FSB_PRIM_SPHERE 1  /* synth.py:141-158 */
#define FSB_PRIM_BOX 2     /* synth.py:161-182 */
#define FSB_TEX_NOISE 0    /* ValueNoise   synth.py:28-84  */
#define FSB_TEX_CHECKER 1  /* Checkerboard synth.py:87-98  */
#define FSB_TEX_SINE 2     /* SineGrating  synth.py:101-115 */

/* One textured primitive of a Scene (synth.py:187-205).
 * geom: plane point[3] + unit normal[3]; sphere center[3] + radius; box lo[3] + hi[3].
 * tex:  noise (scale, lo, hi, persistence); checker (period, lo, hi);
 *       sine (wavelength, lo, hi, unit direction[3]). */
typedef struct fsb_prim {
  int32_t kind, tex_kind, octaves, reserved;
  int64_t seed;
  double geom[7];
  double tex[8];
} fsb_prim;

/* render (synth.py:217-254) without sensor noise: ray-cast `prims` (device
 * array) through `cam` placed at `origin` with world->camera `rotation`
 * (NULL = identity / origin 0, i.e. camera 0), s x s supersampling.
 * image (H,W) f32 in [0,1]; depth (H,W) f32 and hit (H,W) u8 may be NULL. */
int fsb_render(const fsb_camera* cam, const double rotation[9], const double origin[3],
               const fsb_prim* prims, int32_t nprims, int32_t supersample, float* image,
               float* depth, uint8_t* hit, void* stream);

/* evaluate.make_report (evaluate.py:62-98) reductions over n pixels:
 * err = |w_est - w_gt| (0 outside valid; written to err_map when non-NULL),
 * out[0] = #valid, out[1] = mean err, out[2] = median err (exact radix select),
 * out[3] = mean |depth_est - depth_gt| over valid & finite & > 0 (NaN if none;
 * depth pointers both NULL to skip), out[4] = that count, out[5 + k] =
 * 100 * #(err > taus[k]) / #valid. w_*: (n,2) f64, taus/out: device f64,
 * ntaus <= 16. Scratch: fsb_error_report_scratch_bytes(n). */
int fsb_error_report(const double* w_est, const double* w_gt, const uint8_t* valid, int64_t n,
                     const double* taus, int32_t ntaus, const double* depth_est,
                     const double* depth_gt, double* err_map, double* out, void* scratch,
                     size_t scratch_bytes, void* stream);
size_t fsb_error_report_scratch_bytes(int64_t n);

/* make_ground_truth (synth.py:271-303): exact depth0 (cam0 ray distance, 0 off
 * the scene / FOV), correspondence x1 - x0 (0 where cam0 misses or cam1 cannot
 * project) and covisibility (unoccluded from camera 1 within occlusion_tol,
 * inside camera 1's FOV and image). depth0 (H,W) f64, corr (H,W,2) f64, covis
 * (H,W) u8 on the cam0 grid; scratch >= 256 bytes. */
int fsb_ground_truth(const fsb_rig* rig, const fsb_prim* prims, int32_t nprims,
                     double occlusion_tol, double* depth0, double* corr, uint8_t* covis,
                     void* scratch, size_t scratch_bytes, void* stream);

/* Library build identification, e.g. "fsb200 sm_100a". */
const char* fsb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FSB200_H_ */
