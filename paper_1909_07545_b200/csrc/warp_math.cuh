// Per-pixel warp-loop gathers shared by the standalone kernels (pd.cu) and the
// fused epilogue of the blocked PD kernel (pd_block.cu).
//
// Reference: solver.py:332-337 (i1w and trajectory directions at x + w),
// rasters.py:57-141 (masked bicubic).
#pragma once

#include "fsb_common.cuh"

namespace fsb {

struct SampleSrc {
  const float* i1;         // level image 1
  const uint8_t* mask;     // level mask
  const float* traj;       // (h,w,2)
  const uint8_t* traj_ok;
  const float4* packed;    // optional {i1, traj.x, traj.y, 0}
  const uint8_t* full16;   // optional: bit0 all 16 mask taps valid, bit1 all 16 traj taps valid
  int h, w;
};

// Fast path: every tap valid for both fields -> plain Catmull-Rom over the packed
// float4 texels (same tap order and weights as bicubic_at's all-valid branch,
// so bit-identical to the general path).
FSB_INLINE float4 cubic_packed(const float4* __restrict__ t, int w, int ix, int iy, float fx,
                               float fy) {
  float wx[4], wy[4];
  cubic_weights(fx, wx);
  cubic_weights(fy, wy);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float4* row = t + (size_t)(iy + a - 1) * w + (ix - 1);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const float4 v = __ldg(row + b);
      const float wt = wy[a] * wx[b];
      a0 = tap_acc(a0, wt, v.x);
      a1 = tap_acc(a1, wt, v.y);
      a2 = tap_acc(a2, wt, v.z);
    }
  }
  return make_float4(a0, a1, a2, 0.f);
}

// Renormalised trajectory direction, valid if norm > 0.5 (solver.py:336) —
// explicit rounding so every sampler produces the same bits.
FSB_INLINE bool unit_dir(float dr0, float dr1, float& d0, float& d1) {
  const float n2 = __fmaf_rn(dr0, dr0, __fmul_rn(dr1, dr1));
  if (!(n2 > 0.25f)) return false;
  const float r = rsqrtf(n2);
  d0 = __fmul_rn(dr0, r);
  d1 = __fmul_rn(dr1, r);
  return true;
}

// i1w / warp_ok and the renormalised direction / dir_ok at x + w for one pixel.
FSB_INLINE void warp_sample_px(const SampleSrc& S, int x, int y, float2 wv, bool mk, float& i1w,
                               bool& i1w_ok, float2& dir, bool& dir_ok) {
  int ix, iy;
  float fx, fy;
  float iv = 0.f, dr0 = 0.f, dr1 = 0.f;
  bool wok = false, dok = false;
  if (split_off(x, y, wv.x, wv.y, S.h, S.w, ix, iy, fx, fy)) {
    const bool inner = ix >= 1 && ix + 2 < S.w && iy >= 1 && iy + 2 < S.h;
    const uint8_t fl = (S.full16 && inner) ? S.full16[(size_t)iy * S.w + ix] : 0;
    if ((fl & 3) == 3) {
      const float4 r = cubic_packed(S.packed, S.w, ix, iy, fx, fy);
      iv = r.x; dr0 = r.y; dr1 = r.z;
      wok = dok = true;
    } else {
      float a[1], b[2];
      wok = bicubic_at<1, float>(S.i1, S.mask, S.h, S.w, ix, iy, fx, fy, a);
      dok = bicubic_at<2, float>(S.traj, S.traj_ok, S.h, S.w, ix, iy, fx, fy, b);
      iv = a[0]; dr0 = b[0]; dr1 = b[1];
    }
  }
  float d0 = 0.f, d1 = 0.f;
  if (dok) {
    // norm > 0.5 (solver.py:336) as norm^2 > 0.25; unit vector via rsqrt (<= 2 ulp)
    if (!(mk && unit_dir(dr0, dr1, d0, d1))) {
      d0 = d1 = 0.f;
      dok = false;
    }
  }
  i1w = wok ? iv : 0.f;
  i1w_ok = wok && mk;
  dir = make_float2(d0, d1);
  dir_ok = dok;
}

// Fallback branches of bicubic_bits (bilinear over the valid inner 2x2, else
// the nearest valid tap) on channel `ch` of the packed texels, C channels from
// ch on. Same operation order as bicubic_bits, so identical results.
template <int C>
FSB_INLINE void packed_fallback(const float4* __restrict__ P, int w, int ix, int iy, float fx,
                                float fy, unsigned okb, int ch, float out[C]) {
  const float* base = reinterpret_cast<const float*>(P) + ch;
  const float bx[2] = {1.f - fx, fx};
  const float by[2] = {1.f - fy, fy};
  float bil[C];
#pragma unroll
  for (int k = 0; k < C; ++k) bil[k] = 0.f;
  float bws = 0.f;
#pragma unroll
  for (int a = 1; a <= 2; ++a)
#pragma unroll
    for (int b = 1; b <= 2; ++b)
      if (okb >> (4 * a + b) & 1u) {
        const float* t = base + 4 * ((size_t)(iy + a - 1) * w + (ix + b - 1));
        const float bw = by[a - 1] * bx[b - 1];
#pragma unroll
        for (int k = 0; k < C; ++k) bil[k] = tap_acc(bil[k], bw, __ldg(t + k));
        bws += bw;
      }
  if (bws > 1e-12f) {
#pragma unroll
    for (int k = 0; k < C; ++k) out[k] = bil[k] / bws;
    return;
  }
  float nd2 = INFINITY;
  int best = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (okb >> (4 * a + b) & 1u) {
        const float ddx = float(b - 1) - fx, ddy = float(a - 1) - fy;
        const float d2 = dist2(ddx, ddy);
        if (d2 < nd2) { nd2 = d2; best = 4 * a + b; }
      }
  const float* t = base + 4 * ((size_t)(iy + (best >> 2) - 1) * w + (ix + (best & 3) - 1));
#pragma unroll
  for (int k = 0; k < C; ++k) out[k] = __ldg(t + k);
}

// Validity bits (bit 4a+b) of channel `ch` of the 16 taps around (ix, iy):
// in the image and not NaN.
FSB_INLINE unsigned packed_bits(const float4* __restrict__ P, int h, int w, int ix, int iy,
                                int ch) {
  const float* base = reinterpret_cast<const float*>(P) + ch;
  unsigned okb = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = iy + a - 1, c = ix + b - 1;
      const bool in = (unsigned)r < (unsigned)h && (unsigned)c < (unsigned)w;
      const bool v = in && !isnan(__ldg(base + 4 * ((size_t)r * w + c)));
      okb |= (v ? 1u : 0u) << (4 * a + b);
    }
  return okb;
}

// warp_sample_px (mk = true) on NaN-encoded packed texels {mask ? i1 : NaN,
// traj_ok ? traj : NaN, 0} (k_pack_level): one 16-B load per tap serves both
// gathers. The Catmull-Rom sums are formed unconditionally; an invalid tap
// makes its channel's sum NaN (w * NaN = NaN, also for w = 0), so the common
// all-valid case needs no per-tap validity work, and only stencils touching
// an invalid tap re-read their validity and take the bicubic_bits fallback
// (L1 hits). Same results as warp_sample_px (tools/sampler_check.cu).
// kInnerFast: separate unchecked tap loop for stencils inside the image (the
// common case; larger code, used by the standalone sampling kernel).
template <bool kInnerFast = true>
FSB_INLINE void warp_sample_nan(const float4* __restrict__ P, int h, int w, int x, int y,
                                float2 wv, float& i1w, bool& i1w_ok, float2& dir, bool& dir_ok) {
  i1w = 0.f;
  i1w_ok = false;
  dir = make_float2(0.f, 0.f);
  dir_ok = false;
  int ix, iy;
  float fx, fy;
  if (!split_off(x, y, wv.x, wv.y, h, w, ix, iy, fx, fy)) return;
  float wx[4], wy[4];
  cubic_weights(fx, wx);
  cubic_weights(fy, wy);
  const float qnan = __int_as_float(0x7fc00000);
  float a0 = 0.f, a1 = 0.f, a2 = 0.f;
  if (kInnerFast && ix >= 1 && ix + 2 < w && iy >= 1 && iy + 2 < h) {
    const float4* t0 = P + (size_t)(iy - 1) * w + (ix - 1);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float4 t = __ldg(t0 + (size_t)a * w + b);
        const float wt = wy[a] * wx[b];
        a0 = tap_acc(a0, wt, t.x);
        a1 = tap_acc(a1, wt, t.y);
        a2 = tap_acc(a2, wt, t.z);
      }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int r = iy + a - 1, c = ix + b - 1;
        const bool in = (unsigned)r < (unsigned)h && (unsigned)c < (unsigned)w;
        const float4 t = in ? __ldg(P + (size_t)r * w + c) : make_float4(qnan, qnan, qnan, 0.f);
        const float wt = wy[a] * wx[b];
        a0 = tap_acc(a0, wt, t.x);
        a1 = tap_acc(a1, wt, t.y);
        a2 = tap_acc(a2, wt, t.z);
      }
  }
  if (!isnan(a0)) {
    i1w = a0;
    i1w_ok = true;
  } else {
    const unsigned okb = packed_bits(P, h, w, ix, iy, 0);
    if (okb) {
      float v[1];
      packed_fallback<1>(P, w, ix, iy, fx, fy, okb, 0, v);
      i1w = v[0];
      i1w_ok = true;
    }
  }
  bool tok = true;
  float d0 = a1, d1 = a2;
  if (isnan(a1)) {
    const unsigned okb = packed_bits(P, h, w, ix, iy, 1);
    tok = okb != 0;
    if (tok) {
      float v[2];
      packed_fallback<2>(P, w, ix, iy, fx, fy, okb, 1, v);
      d0 = v[0];
      d1 = v[1];
    }
  }
  float e0, e1;
  if (tok && unit_dir(d0, d1, e0, e1)) {
    dir = make_float2(e0, e1);
    dir_ok = true;
  }
}

// Per-tap-validity variant of warp_sample_nan (validity bits gathered with the
// loads; preferred on small levels where many stencils touch the mask edge).
// warp_sample_px (mk = true) on NaN-encoded packed texels {mask ? i1 : NaN,
// traj_ok ? traj : NaN, 0} (k_pack_level): one 16-B load per tap serves both
// gathers and carries their validity, so there is no separate mask / flag
// gather and no divergent slow path; the rare partial stencils re-read their
// valid taps (L1 hits) in the fallback. Same results as warp_sample_px.
FSB_INLINE void warp_sample_nan_bits(const float4* __restrict__ P, int h, int w, int x, int y,
                                float2 wv, float& i1w, bool& i1w_ok, float2& dir, bool& dir_ok) {
  i1w = 0.f;
  i1w_ok = false;
  dir = make_float2(0.f, 0.f);
  dir_ok = false;
  int ix, iy;
  float fx, fy;
  if (!split_off(x, y, wv.x, wv.y, h, w, ix, iy, fx, fy)) return;
  float wx[4], wy[4];
  cubic_weights(fx, wx);
  cubic_weights(fy, wy);
  const bool inner = ix >= 1 && ix + 2 < w && iy >= 1 && iy + 2 < h;
  const float qnan = __int_as_float(0x7fc00000);
  unsigned oki = 0, okt = 0;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = iy + a - 1;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = ix + b - 1;
      const bool in = inner || ((unsigned)r < (unsigned)h && (unsigned)c < (unsigned)w);
      const float4 t = in ? __ldg(P + (size_t)r * w + c) : make_float4(qnan, qnan, qnan, 0.f);
      const float wt = wy[a] * wx[b];
      a0 = tap_acc(a0, wt, t.x);
      a1 = tap_acc(a1, wt, t.y);
      a2 = tap_acc(a2, wt, t.z);
      oki |= (isnan(t.x) ? 0u : 1u) << (4 * a + b);
      okt |= (isnan(t.y) ? 0u : 1u) << (4 * a + b);
    }
  }
  if (oki) {
    i1w_ok = true;
    if (oki == 0xFFFFu) {
      i1w = a0;
    } else {
      float v[1];
      packed_fallback<1>(P, w, ix, iy, fx, fy, oki, 0, v);
      i1w = v[0];
    }
  }
  if (okt) {
    float d0 = a1, d1 = a2;
    if (okt != 0xFFFFu) {
      float v[2];
      packed_fallback<2>(P, w, ix, iy, fx, fy, okt, 1, v);
      d0 = v[0];
      d1 = v[1];
    }
    float e0, e1;
    if (unit_dir(d0, d1, e0, e1)) {
      dir = make_float2(e0, e1);
      dir_ok = true;
    }
  }
}

}  // namespace fsb
