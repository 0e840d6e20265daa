// Launch arguments of the blocked float64 primal-dual kernel (pd64_block.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace fsb {

struct B64 {
  int h, w;
  size_t n;
  const uint8_t* mask;
  const double* T;  // a, b, c planes
  const double* S;  // sigma_p, tau_u, tau_v planes
  const double* iu; const double* rho0;
  double* uo;  // read; written by the first launch of a warp (`first`)
  // first launch of a warp: the warp-start reset of k64_linearize (solver.py:
  // 347-350: u0 = u, u_bar = u, v_bar = v) is done here from the loaded u / v
  int first;
  // state sets (src read, dst written): u, u_bar, v (2), v_bar (2), p (2), q (4)
  const double *su, *sub, *sv, *svb, *sp, *sq;
  double *du, *dub, *dv, *dvb, *dp, *dq;
  double lam, alpha0, alpha1, theta, sigma_q, heps;
  int iters;
  float* diag_p; float* diag_q;  // per-cycle maxima (nullptr = off)
  // last launch of a warp: clip / accumulate epilogue of k64_finish fused in
  int fin;
  double du_max;
  const double* dirs; double* wv;
  float* diag_du; double* partials;  // max |du| and per-tile sums of |du| (nullptr = off)
  double* diag_du64;                 // max |du| in float64 (when set, instead of diag_du)
  // k64_tile with a work list: per-pixel edge codes (bit0 mask, bit1 x-edge, bit2 y-edge) and
  // the level's work list (tiles[0] = count, tiles[1 + k] = tile id; nullptr = all)
  const uint32_t* ecode;
  const int* tiles;
  int persist;   // k64_tile with a work list: persistent 2 CTAs / SM, second half staggered by this many ns (0 = one tile per CTA)
};

// `iters` (<= halo, halo in 1..3 or 5) cycles from the src set into the dst set.
int pd64_block_launch(const B64& A, int halo, cudaStream_t st);
size_t pd64_block_tiles(int w, int h, int halo);
// The issue-lean tile kernel (pd64_tile.cu): same arguments and semantics.
int pd64_tile_launch(const B64& A, int halo, cudaStream_t st);
int pd64_tile_launch_unchecked(const B64& A, int halo, cudaStream_t st);  // iters 0: timing
size_t pd64_tile_count(int w, int h, int halo);
int pd64_tile_tile_list(const uint8_t* mask, int w, int h, int halo, int* tiles, cudaStream_t st);
// Per-level edge codes (bit0 mask, bit1 x-edge, bit2 y-edge; pd64_tile.cu);
// with `codef`, also as a float64 plane (the 10th constant plane of k64_tma).
int pd64_edge_codes(const uint8_t* mask, int w, int h, uint32_t* code, double* codef,
                    cudaStream_t st);

// The TMA-fed tile kernel (pd64_tma.cu, halo-2 levels). Layout it requires:
// each state set one block of 12 planes of stride n = h*w in the order u, v0,
// v1, p0, p1, q0..q3, u_bar, v_bar0, v_bar1 (A.su .. A.svb point into it), the
// level's constants one block of 10 planes: tensor a b c, sigma_p, tau_u,
// tau_v, I_u, rho0, u_omega, edge code (float64); w % 4 == 0. Tensor maps:
// [set][0] all 12 planes, [set][1] the first 9 (the warp's first launch loads
// no u_bar / v_bar, its last stores none).
struct Tma64Level {
  CUtensorMap ld[2][2], st[2][2], cst;
};
bool pd64_tma_usable(int w, int h);
bool pd64_tma_level_maps(Tma64Level* M, const double* set0, const double* set1,
                         const double* cst, int w, int h);
int pd64_tma_launch(const B64& A, const Tma64Level& M, int src_set, cudaStream_t st);
size_t pd64_tma_tile_count(int w, int h);
int pd64_tma_tile_list(const uint8_t* mask, int w, int h, int* tiles, cudaStream_t st);

// Diagnostics slots of the whole-level kernel (pd64_level.cu): per-cycle |p| /
// |q| maxima from the level's first cycle, per-warp max |du| (float or
// float64) from its first warp, and N x CTAs partial sums of |du|.
struct LvlDiag {
  float* p; float* q; float* du; double* du64; double* partials;
};

// The cluster-tile kernel (pd64_ctile.cu, the large levels): same layout as
// k64_tma; regions of a cluster of CTAs exchange halos through DSMEM, R
// (pd64_ctile_halo) cycles per launch. Tensor maps: [set][0] 12 planes, [set][1] 9.
struct Ctile64Maps {
  CUtensorMap ld[2][2], cst;
};
int pd64_ctile_halo();
bool pd64_ctile_usable(int w, int h);
bool pd64_ctile_maps(Ctile64Maps* M, const double* set0, const double* set1, const double* cst,
                     int w, int h);
size_t pd64_ctile_partials(int w, int h);  // per-CTA partial sums of |du| (regions x CTAs)
int pd64_ctile_list(const uint8_t* mask, int w, int h, int* tiles, cudaStream_t st);
int pd64_ctile_launch(const B64& A, const Ctile64Maps& M, int src_set, cudaStream_t st);

}  // namespace fsb
