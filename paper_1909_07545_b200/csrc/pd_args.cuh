// Launch arguments of the temporally blocked primal-dual kernels
// (pd_block.cu per-pixel tiles, pd_pair.cu packed pixel pairs) and the driver.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/fsb200.h"

namespace fsb {

struct StateSet {   // plane stride n: v, vb, p hold 2 planes, q holds 4
  float* u; float* ub; float* v; float* vb; float* p; float* q;
};

struct BlockArgs {
  int h, w;
  size_t n;
  StateSet src, dst;
  const uint8_t* mask;
  const float* T;   // a, b, c planes
  const float* S;   // sigma_p, tau_u, tau_v planes
  float* iu; float* rho0; float* u_omega;
  float lam, alpha0, alpha1, theta, sigma_q, du_max;
  float huber_eps;  // > 0: Huber-TV dual step (fsb_params.regularizer)
  int iters;
  // FIN: w += du * dirs with this warp's directions (from k_warp_prologue)
  const float* dirs;
  float* wv;
  // diagnostics (nullptr = off)
  float* diag_p; float* diag_q; float* diag_du; double* partials;
  // TMA kernel work list (pd_tma_tile_list), nullptr = every tile
  const int* tile_list;
  // FIN launches: also store u_bar / v_bar (only the level's last warp needs them)
  int store_bars;
};

// TMA descriptors of one level for the persistent kernel (pd_tma.cu): the two
// 12-plane state blocks and the 10-plane constant block, 64 x 32 boxes.
struct TmaMaps {
  CUtensorMap state[2];
  CUtensorMap consts;
};
bool pd_tma_maps(TmaMaps* maps, const float* state_a, const float* state_b, const float* consts,
                 int w, int h);
int pd_tma_launch(const BlockArgs& A, const TmaMaps& maps, int src_set, int halo, bool lin,
                  bool fin, cudaStream_t st, int* nparts);

int pd_tma_tile_list(const uint8_t* mask, int w, int h, int halo, int* tiles, cudaStream_t st);
size_t pd_tma_partials(int w, int h, int halo);
int pd_num_sms();

int pd_block_launch(const BlockArgs& A, int halo, bool lin, bool fin, cudaStream_t st,
                    int* nblocks);
int pd_pair_launch(const BlockArgs& A, int halo, bool lin, bool fin, cudaStream_t st,
                   int* nblocks);

// Whole-level warp loop on one thread-block cluster (pd_cluster.cu) for levels
// small enough to live on <= 16 SMs.
bool level_cluster_fits(int h, int w, int warp_iters);
int level_cluster_solve(const fsb_level* L, const fsb_params* prm, const fsb_diag* diag,
                        int64_t pd_off, int64_t warp_off, cudaStream_t st);

}  // namespace fsb
