// Error report of a correspondence estimate: the reductions
// of evaluate.make_report (evaluate.py:62-98) on the GPU.
//
//   err      = |w_est - w_gt| per pixel, 0 outside `valid`   (evaluate.py:62-68)
//   pct_bad  = 100 * #(err > tau) / #valid per tau            (evaluate.py:71-78)
//   mean / median of err over valid pixels                    (evaluate.py:81-98)
//   mean |depth_est - depth_gt| over valid & finite & > 0
//
// Counts are exact integers. Sums are fp64 block partials added in block order
// (deterministic). The median is an exact radix select over the fp64 bit
// patterns (errors are >= 0, so the bit order is the value order): eight
// rounds of a 256-bin histogram plus a one-block pick, all on the device.

#include "fsb_common.cuh"

namespace fsb {
namespace {

constexpr int kThreads = 256, kMaxBlocks = 592, kMaxTaus = 16;
// per-block partial record: valid count, err sum, depth count, depth sum, tau counts
constexpr int kRec = 4 + kMaxTaus;

__global__ void k_err(const double* __restrict__ we, const double* __restrict__ wg,
                      const uint8_t* __restrict__ valid, int64_t n, const double* __restrict__ taus,
                      int ntaus, const double* __restrict__ de, const double* __restrict__ dg,
                      double* __restrict__ err, double* __restrict__ part) {
  __shared__ double s[kThreads / 32][kRec];
  double cnt = 0, sum = 0, dcnt = 0, dsum = 0, tc[kMaxTaus];
  for (int k = 0; k < kMaxTaus; ++k) tc[k] = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool v = valid[i];
    const double dx = we[2 * i] - wg[2 * i], dy = we[2 * i + 1] - wg[2 * i + 1];
    const double e = v ? sqrt(dx * dx + dy * dy) : 0.0;
    if (err) err[i] = e;
    if (!v) continue;
    cnt += 1;
    sum += e;
    for (int k = 0; k < ntaus; ++k) tc[k] += e > taus[k] ? 1 : 0;
    if (de && isfinite(de[i]) && de[i] > 0) {
      dcnt += 1;
      dsum += fabs(de[i] - dg[i]);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  cnt = warp_sum(cnt); sum = warp_sum(sum); dcnt = warp_sum(dcnt); dsum = warp_sum(dsum);
  for (int k = 0; k < ntaus; ++k) tc[k] = warp_sum(tc[k]);
  if (lane == 0) {
    s[wid][0] = cnt; s[wid][1] = sum; s[wid][2] = dcnt; s[wid][3] = dsum;
    for (int k = 0; k < ntaus; ++k) s[wid][4 + k] = tc[k];
  }
  __syncthreads();
  if (threadIdx.x < 4 + ntaus) {
    double t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += s[w][threadIdx.x];
    part[(size_t)blockIdx.x * kRec + threadIdx.x] = t;
  }
}

// Radix-select state: [0] prefix bits fixed so far, [1] k remaining (rank within
// the prefix class), one pair per selected rank.
__global__ void k_hist(const double* __restrict__ err, const uint8_t* __restrict__ valid,
                       int64_t n, const unsigned long long* __restrict__ sel, int shift,
                       unsigned* __restrict__ hist) {
  __shared__ unsigned h[2][256];
  for (int k = threadIdx.x; k < 512; k += blockDim.x) (&h[0][0])[k] = 0;
  __syncthreads();
  const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!valid[i]) continue;
    const unsigned long long b = __double_as_longlong(err[i]);
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if ((b & hi_mask) == (sel[2 * r] & hi_mask)) atomicAdd(&h[r][(b >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 512; k += blockDim.x)
    if ((&h[0][0])[k]) atomicAdd(hist + k, (&h[0][0])[k]);
}

__global__ void k_pick(unsigned* __restrict__ hist, unsigned long long* __restrict__ sel,
                       int shift) {
  const int r = threadIdx.x;  // one thread per selected rank
  if (r >= 2) return;
  unsigned long long k = sel[2 * r + 1];
  unsigned bin = 0;
  for (; bin < 256; ++bin) {
    const unsigned c = hist[r * 256 + bin];
    if (k < c) break;
    k -= c;
  }
  sel[2 * r] |= (unsigned long long)(bin & 255u) << shift;
  sel[2 * r + 1] = k;
  for (int b = 0; b < 256; ++b) hist[r * 256 + b] = 0;
}

__global__ void k_final(const double* __restrict__ part, int nblocks, int ntaus,
                        const unsigned long long* __restrict__ sel, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double t[kRec];
  for (int k = 0; k < kRec; ++k) t[k] = 0;
  for (int b = 0; b < nblocks; ++b)
    for (int k = 0; k < 4 + ntaus; ++k) t[k] += part[(size_t)b * kRec + k];
  const double n = t[0];
  out[0] = n;
  out[1] = n > 0 ? t[1] / n : NAN;
  const unsigned long long c = (unsigned long long)n;
  if (c == 0) {
    out[2] = NAN;
  } else {
    const double lo = __longlong_as_double(sel[0]), hi = __longlong_as_double(sel[2]);
    out[2] = (c & 1ull) ? hi : (lo + hi) / 2.0;  // numpy median of an even count
  }
  out[3] = t[2] > 0 ? t[3] / t[2] : NAN;
  out[4] = t[2];
  for (int k = 0; k < ntaus; ++k) out[5 + k] = n > 0 ? 100.0 * t[4 + k] / n : NAN;
}

__global__ void k_sel_init(unsigned long long* sel, const double* __restrict__ part, int nblocks) {
  if (threadIdx.x != 0) return;
  double n = 0;
  for (int b = 0; b < nblocks; ++b) n += part[(size_t)b * kRec];
  const unsigned long long c = (unsigned long long)n;
  sel[0] = 0; sel[1] = c ? (c - 1) / 2 : 0;  // lower middle (== upper for odd counts)
  sel[2] = 0; sel[3] = c / 2;                // upper middle
}

}  // namespace
}  // namespace fsb

using namespace fsb;

extern "C" {

size_t fsb_error_report_scratch_bytes(int64_t n) {
  return align_up((size_t)kMaxBlocks * kRec * sizeof(double)) + align_up(512 * sizeof(unsigned)) +
         align_up(4 * sizeof(unsigned long long)) + align_up((size_t)(n > 0 ? n : 1) * sizeof(double));
}

int fsb_error_report(const double* w_est, const double* w_gt, const uint8_t* valid, int64_t n,
                     const double* taus, int32_t ntaus, const double* depth_est,
                     const double* depth_gt, double* err_map, double* out, void* scratch,
                     size_t scratch_bytes, void* stream) {
  if (n < 0 || !w_est || !w_gt || !valid || !out || ntaus < 0 || ntaus > kMaxTaus ||
      (ntaus > 0 && !taus) || ((depth_est == nullptr) != (depth_gt == nullptr)) || !scratch)
    return FSB_EINVAL;
  if (scratch_bytes < fsb_error_report_scratch_bytes(n)) return FSB_ENOSPC;
  cudaStream_t st = as_stream(stream);
  char* p = static_cast<char*>(scratch);
  double* part = reinterpret_cast<double*>(p);
  p += align_up((size_t)kMaxBlocks * kRec * sizeof(double));
  unsigned* hist = reinterpret_cast<unsigned*>(p);
  p += align_up(512 * sizeof(unsigned));
  unsigned long long* sel = reinterpret_cast<unsigned long long*>(p);
  p += align_up(4 * sizeof(unsigned long long));
  double* err = err_map ? err_map : reinterpret_cast<double*>(p);
  int blocks = (int)((n + kThreads - 1) / kThreads);
  blocks = blocks < 1 ? 1 : (blocks > kMaxBlocks ? kMaxBlocks : blocks);
  k_err<<<blocks, kThreads, 0, st>>>(w_est, w_gt, valid, n, taus, ntaus, depth_est, depth_gt, err,
                                     part);
  cudaMemsetAsync(hist, 0, 512 * sizeof(unsigned), st);
  k_sel_init<<<1, 32, 0, st>>>(sel, part, blocks);
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_hist<<<blocks, kThreads, 0, st>>>(err, valid, n, sel, shift, hist);
    k_pick<<<1, 32, 0, st>>>(hist, sel, shift);
  }
  k_final<<<1, 32, 0, st>>>(part, blocks, ntaus, sel, out);
  return launch_status();
}

}  // extern "C"
