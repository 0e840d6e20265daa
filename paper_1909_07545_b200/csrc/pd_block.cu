// K6: temporally blocked, fused primal-dual kernel (the hot kernel).
//
// One launch runs `iters` (<= R) full primal-dual cycles (solver.py:279-303)
// on a 2-D tile with an R-pixel halo: the state of every owned pixel lives in
// registers, and only the values neighbours need cross shared memory —
// u_bar / v_bar for the forward differences of the dual step and the
// edge-masked fluxes (T p, q) for the backward divergence of the primal step.
// Iteration n recomputes a region shrunk by n, so after `iters` cycles the
// interior is exact; the halo work is the price of reading and writing the
// state once per `iters` iterations instead of once per iteration.
//
// Fused into the same launch when requested:
//   LIN: the warp-start resets u_omega = u, u_bar = u, v_bar = v
//        (solver.py:344-346; I_u and rho0 come from k_warp_prologue);
//   FIN: the warp epilogue (solver.py:356-360: clip, accumulate u and w).
//
// State is ping-ponged between two plane sets (src -> dst) because halos read
// neighbours' old values while their owners write new ones.

#include <stdlib.h>

#include "pd_args.cuh"
#include "pd_math.cuh"

namespace fsb {



namespace {

template <int CX, int NW, int PY, int R>
struct Tile {
  static constexpr int EW = 32 * CX, EH = NW * PY;  // extended tile
  static constexpr int TW = EW - 2 * R, TH = EH - 2 * R;  // interior
  static constexpr int SW = EW + 2, SH = EH + 2;     // smem plane with 1-px pad
  static constexpr int PLANE = SW * SH;
  static constexpr int NPLANES = 9;                  // ub, vb0, vb1, px, py, q0x, q0y, q1x, q1y
  static constexpr size_t SMEM = sizeof(float) * NPLANES * PLANE + PLANE;
  static constexpr int NPX = CX * PY;
  static_assert(TW > 0 && TH > 0, "halo larger than tile");
};

// Skipping rows outside the shrinking valid region saves ~15% of the work but
// splits the unrolled pixel loop into per-row branches (less ILP).
#ifndef FSB_PD_SKIP_ROWS
#define FSB_PD_SKIP_ROWS 0
#endif
constexpr bool kSkipRows = FSB_PD_SKIP_ROWS != 0;

__device__ __forceinline__ int sidx(int r, int c, int SW) { return (r + 1) * SW + (c + 1); }

template <int CX, int NW, int PY, int R, bool LIN, bool FIN>
__global__ void __launch_bounds__(NW * 32, 1) k_pd_block(const BlockArgs A) {
  using TL = Tile<CX, NW, PY, R>;
  constexpr int EW = TL::EW, EH = TL::EH, SW = TL::SW, PL = TL::PLANE, NPX = TL::NPX;
  extern __shared__ __align__(16) float smem[];
  float* s_ub = smem;
  float* s_vb0 = s_ub + PL;
  float* s_vb1 = s_vb0 + PL;
  float* s_px = s_vb1 + PL;
  float* s_py = s_px + PL;
  float* s_q0x = s_py + PL;
  float* s_q0y = s_q0x + PL;
  float* s_q1x = s_q0y + PL;
  float* s_q1y = s_q1x + PL;
  uint8_t* s_m = reinterpret_cast<uint8_t*>(s_q1y + PL);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ox = (int)blockIdx.x * TL::TW - R, oy = (int)blockIdx.y * TL::TH - R;
  const size_t n = A.n;

  // zero the 1-px pad ring of every plane (interior cells are all written below)
  constexpr int RING = 2 * (EW + 2) + 2 * EH;
  for (int k = threadIdx.x; k < RING; k += NW * 32) {
    int idx;
    if (k < EW + 2) idx = k;                                   // top pad row
    else if (k < 2 * (EW + 2)) idx = (EH + 1) * SW + (k - (EW + 2));  // bottom pad row
    else if (k < 2 * (EW + 2) + EH) idx = (k - 2 * (EW + 2) + 1) * SW;  // left pad column
    else idx = (k - 2 * (EW + 2) - EH + 1) * SW + EW + 1;        // right pad column
#pragma unroll
    for (int pl = 0; pl < TL::NPLANES; ++pl) smem[pl * PL + idx] = 0.f;
    s_m[idx] = 0;
  }

  // per-pixel registers
  float u[NPX], v0[NPX], v1[NPX], p0[NPX], p1[NPX], q0[NPX], q1[NPX], q2[NPX], q3[NPX];
  float ta[NPX], tb[NPX], tc[NPX], sp[NPX], tu[NPX], tv[NPX], g[NPX], rh[NPX], uo[NPX];
  unsigned bits = 0;  // per pixel: bit0 in-image&mask, bit1 ex, bit2 ey  (3 bits x NPX <= 32)
  static_assert(3 * NPX <= 32, "too many pixels per thread for the mask bit field");

#pragma unroll
  for (int j = 0; j < PY; ++j)
#pragma unroll
    for (int cx = 0; cx < CX; ++cx) {
      const int r = warp + NW * j, c = lane + 32 * cx;
      const int gx = ox + c, gy = oy + r;
      const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
      s_m[sidx(r, c, SW)] = in ? A.mask[(size_t)gy * A.w + gx] : 0;
    }
  __syncthreads();

#pragma unroll
  for (int j = 0; j < PY; ++j)
#pragma unroll
    for (int cx = 0; cx < CX; ++cx) {
      const int k = j * CX + cx;
      const int r = warp + NW * j, c = lane + 32 * cx;
      const int gx = ox + c, gy = oy + r;
      const bool in = (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
      const size_t gi = in ? (size_t)gy * A.w + gx : 0;
      const bool mk = s_m[sidx(r, c, SW)] != 0;
      const bool ex = mk && s_m[sidx(r, c + 1, SW)];
      const bool ey = mk && s_m[sidx(r + 1, c, SW)];
      bits |= ((mk ? 1u : 0u) | (ex ? 2u : 0u) | (ey ? 4u : 0u)) << (3 * k);
      float ub = 0.f, vb0 = 0.f, vb1 = 0.f;
      if (in) {
        u[k] = A.src.u[gi];
        v0[k] = A.src.v[gi]; v1[k] = A.src.v[n + gi];
        p0[k] = A.src.p[gi]; p1[k] = A.src.p[n + gi];
        q0[k] = A.src.q[gi]; q1[k] = A.src.q[n + gi];
        q2[k] = A.src.q[2 * n + gi]; q3[k] = A.src.q[3 * n + gi];
        ta[k] = A.T[gi]; tb[k] = A.T[n + gi]; tc[k] = A.T[2 * n + gi];
        sp[k] = A.S[gi] * A.alpha1; tu[k] = A.S[n + gi]; tv[k] = A.S[2 * n + gi];
        if (LIN) {  // warp start: u_omega = u, u_bar = u, v_bar = v (solver.py:344-346)
          g[k] = A.iu[gi]; rh[k] = A.rho0[gi];
          uo[k] = u[k];
          ub = u[k]; vb0 = v0[k]; vb1 = v1[k];
        } else {
          g[k] = A.iu[gi]; rh[k] = A.rho0[gi]; uo[k] = A.u_omega[gi];
          ub = A.src.ub[gi]; vb0 = A.src.vb[gi]; vb1 = A.src.vb[n + gi];
        }
      } else {
        u[k] = v0[k] = v1[k] = p0[k] = p1[k] = q0[k] = q1[k] = q2[k] = q3[k] = 0.f;
        ta[k] = 1.f; tb[k] = 0.f; tc[k] = 1.f; sp[k] = tu[k] = tv[k] = 0.f;
        g[k] = rh[k] = uo[k] = 0.f;
      }
      s_ub[sidx(r, c, SW)] = ub;
      s_vb0[sidx(r, c, SW)] = vb0;
      s_vb1[sidx(r, c, SW)] = vb1;
    }
  __syncthreads();

  const float sq = A.sigma_q * A.alpha0;
  for (int it = 1; it <= A.iters; ++it) {
    float pmax = 0.f, qmax = 0.f;
    // ---- dual ascent on rows [it-1, EH-1-it]
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int r = warp + NW * j;
      if (kSkipRows && (r < it - 1 || r > EH - 1 - it)) continue;
#pragma unroll
      for (int cx = 0; cx < CX; ++cx) {
        const int k = j * CX + cx;
        const int c = lane + 32 * cx;
        const bool ex = (bits >> (3 * k + 1)) & 1u, ey = (bits >> (3 * k + 2)) & 1u;
        const int i = sidx(r, c, SW);
        const float ub = s_ub[i], vb0 = s_vb0[i], vb1 = s_vb1[i];
        const float gx = ex ? s_ub[i + 1] - ub : 0.f;
        const float gy = ey ? s_ub[i + SW] - ub : 0.f;
        const float g00 = ex ? s_vb0[i + 1] - vb0 : 0.f;
        const float g01 = ey ? s_vb0[i + SW] - vb0 : 0.f;
        const float g10 = ex ? s_vb1[i + 1] - vb1 : 0.f;
        const float g11 = ey ? s_vb1[i + SW] - vb1 : 0.f;
        dual_update(ta[k], tb[k], tc[k], sp[k], sq, gx, gy, g00, g01, g10, g11, vb0, vb1, p0[k],
                    p1[k], q0[k], q1[k], q2[k], q3[k], A.huber_eps);
        const Flux f = make_flux(ta[k], tb[k], tc[k], ex, ey, p0[k], p1[k], q0[k], q1[k], q2[k],
                                 q3[k]);
        s_px[i] = f.px; s_py[i] = f.py;
        s_q0x[i] = f.q0x; s_q0y[i] = f.q0y;
        s_q1x[i] = f.q1x; s_q1y[i] = f.q1y;
        if (A.diag_p) {
          const int gx_ = ox + c, gy_ = oy + r;
          const bool interior = r >= R && r < EH - R && c >= R && c < EW - R &&
                                (unsigned)gx_ < (unsigned)A.w && (unsigned)gy_ < (unsigned)A.h;
          if (interior) {
            pmax = fmaxf(pmax, sqrtf(p0[k] * p0[k] + p1[k] * p1[k]));
            qmax = fmaxf(qmax, sqrtf((q0[k] * q0[k] + q1[k] * q1[k]) +
                                     (q2[k] * q2[k] + q3[k] * q3[k])));
          }
        }
      }
    }
    if (A.diag_p) {
      pmax = warp_max(pmax);
      qmax = warp_max(qmax);
      if (lane == 0) {
        atomic_max_nonneg(A.diag_p + it - 1, pmax);
        atomic_max_nonneg(A.diag_q + it - 1, qmax);
      }
    }
    __syncthreads();
    // ---- primal descent on rows [it, EH-1-it]
#pragma unroll
    for (int j = 0; j < PY; ++j) {
      const int r = warp + NW * j;
      if (kSkipRows && (r < it || r > EH - 1 - it)) continue;
#pragma unroll
      for (int cx = 0; cx < CX; ++cx) {
        const int k = j * CX + cx;
        const int c = lane + 32 * cx;
        const int i = sidx(r, c, SW);
        const float dv = ((s_px[i] - s_px[i - 1]) + s_py[i]) - s_py[i - SW];
        const float d0 = ((s_q0x[i] - s_q0x[i - 1]) + s_q0y[i]) - s_q0y[i - SW];
        const float d1 = ((s_q1x[i] - s_q1x[i - 1]) + s_q1y[i]) - s_q1y[i - SW];
        float ub, vb0, vb1;
        primal_update(dv, d0, d1, tu[k], tv[k], g[k], rh[k], uo[k], p0[k], p1[k], A.lam,
                      A.alpha0, A.alpha1, A.theta, u[k], v0[k], v1[k], ub, vb0, vb1);
        s_ub[i] = ub; s_vb0[i] = vb0; s_vb1[i] = vb1;
      }
    }
    __syncthreads();
  }

  // ---- epilogue + store of the interior
  float dmax = 0.f;
  double dsum = 0.0;
#pragma unroll
  for (int j = 0; j < PY; ++j)
#pragma unroll
    for (int cx = 0; cx < CX; ++cx) {
      const int k = j * CX + cx;
      const int r = warp + NW * j, c = lane + 32 * cx;
      const int gx = ox + c, gy = oy + r;
      const bool interior = r >= R && r < EH - R && c >= R && c < EW - R &&
                            (unsigned)gx < (unsigned)A.w && (unsigned)gy < (unsigned)A.h;
      if (!interior) continue;
      const size_t gi = (size_t)gy * A.w + gx;
      const int i = sidx(r, c, SW);
      float uu = u[k], ub = s_ub[i];
      if (FIN) {  // solver.py:356-360
        const bool mk = bits >> (3 * k) & 1u;
        float du = fminf(fmaxf(uu - uo[k], -A.du_max), A.du_max);
        if (!mk) du = 0.f;
        uu = uo[k] + du;
        ub = uu;
        const float2 d = reinterpret_cast<const float2*>(A.dirs)[gi];
        float2 wv = reinterpret_cast<float2*>(A.wv)[gi];
        wv.x = wv.x + du * d.x;
        wv.y = wv.y + du * d.y;
        reinterpret_cast<float2*>(A.wv)[gi] = wv;
        dmax = fmaxf(dmax, fabsf(du));
        dsum += (double)fabsf(du);
      }
      if (LIN) A.u_omega[gi] = uo[k];
      A.dst.u[gi] = uu;
      A.dst.ub[gi] = ub;
      A.dst.v[gi] = v0[k]; A.dst.v[n + gi] = v1[k];
      A.dst.vb[gi] = s_vb0[i]; A.dst.vb[n + gi] = s_vb1[i];
      A.dst.p[gi] = p0[k]; A.dst.p[n + gi] = p1[k];
      A.dst.q[gi] = q0[k]; A.dst.q[n + gi] = q1[k];
      A.dst.q[2 * n + gi] = q2[k]; A.dst.q[3 * n + gi] = q3[k];
    }
  if (FIN && A.diag_du) {
    __shared__ double red_s[NW];
    __shared__ float red_m[NW];
    dmax = warp_max(dmax);
    dsum = warp_sum(dsum);
    if (lane == 0) { red_s[warp] = dsum; red_m[warp] = dmax; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      float m = 0.f;
      for (int k = 0; k < NW; ++k) { t += red_s[k]; m = fmaxf(m, red_m[k]); }
      A.partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
      atomic_max_nonneg(A.diag_du, m);
    }
  }
}

// Tile shapes (FSB_PD_TILE selects for tuning; larger tiles spill at 512 threads):
//   0: 64 x 32 ext tile, 256 threads x 8 px     1: 64 x 32, 512 threads x 4 px
template <int CX, int NW, int PY, int R, bool LIN, bool FIN>
int launch_shape(const BlockArgs& A, cudaStream_t st, int* nblocks) {
  using TL = Tile<CX, NW, PY, R>;
  static std::atomic<unsigned long long> attr{0};
  auto kern = k_pd_block<CX, NW, PY, R, LIN, FIN>;
  once_per_device(attr, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TL::SMEM);
  });
  dim3 grd((A.w + TL::TW - 1) / TL::TW, (A.h + TL::TH - 1) / TL::TH);
  if (nblocks) *nblocks = (int)(grd.x * grd.y);
  kern<<<grd, NW * 32, TL::SMEM, st>>>(A);
  return launch_status();
}

int tile_choice() {
  static const int t = [] {
    const char* e = getenv("FSB_PD_TILE");
    return e ? atoi(e) : 1;
  }();
  return t;
}

template <int R, bool LIN, bool FIN>
int launch_block(const BlockArgs& A, cudaStream_t st, int* nblocks) {
  switch (tile_choice()) {
    case 0: return launch_shape<2, 8, 4, R, LIN, FIN>(A, st, nblocks);
    default: return launch_shape<2, 16, 2, R, LIN, FIN>(A, st, nblocks);
  }
}

template <int R>
int launch_r(const BlockArgs& A, bool lin, bool fin, cudaStream_t st, int* nb) {
  if (lin && fin) return launch_block<R, true, true>(A, st, nb);
  if (lin) return launch_block<R, true, false>(A, st, nb);
  if (fin) return launch_block<R, false, true>(A, st, nb);
  return launch_block<R, false, false>(A, st, nb);
}

}  // namespace

// Halo (= maximum iterations per launch) compiled in.
int pd_block_max_iters() { return 5; }


int pd_block_launch(const BlockArgs& A, int halo, bool lin, bool fin, cudaStream_t st,
                    int* nblocks) {
  if (A.iters < 1 || A.iters > halo) return FSB_EINVAL;
  switch (halo) {
    case 1: return launch_r<1>(A, lin, fin, st, nblocks);
    case 2: return launch_r<2>(A, lin, fin, st, nblocks);
    case 3: return launch_r<3>(A, lin, fin, st, nblocks);
    case 5: return launch_r<5>(A, lin, fin, st, nblocks);
    default: return FSB_EINVAL;
  }
}

}  // namespace fsb
