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
      a0 += wt * v.x;
      a1 += wt * v.y;
      a2 += wt * v.z;
    }
  }
  return make_float4(a0, a1, a2, 0.f);
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
    const float n2 = dr0 * dr0 + dr1 * dr1;
    if (n2 > 0.25f && mk) {
      const float r = rsqrtf(n2);
      d0 = dr0 * r;
      d1 = dr1 * r;
    } else {
      dok = false;
    }
  }
  i1w = wok ? iv : 0.f;
  i1w_ok = wok && mk;
  dir = make_float2(d0, d1);
  dir_ok = dok;
}

}  // namespace fsb
