// Debug harness: warp_sample_nan vs warp_sample_px on random fields/positions.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1909_07545_b200/csrc/warp_math.cuh"
using namespace fsb;
__global__ void k(SampleSrc S, const float4* P, int n, const float* px, float* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x = i % S.w, y = (i / S.w) % S.h;
  float2 wv = make_float2(px[2 * i], px[2 * i + 1]);
  float a, b; bool ao, bo, ad, bd; float2 da, db;
  warp_sample_px(S, x, y, wv, true, a, ao, da, ad);
  warp_sample_nan(P, S.h, S.w, x, y, wv, b, bo, db, bd);
  out[8 * i] = a; out[8 * i + 1] = b; out[8 * i + 2] = ao; out[8 * i + 3] = bo;
  out[8 * i + 4] = da.x; out[8 * i + 5] = db.x; out[8 * i + 6] = ad; out[8 * i + 7] = bd;
}
int main() {
  const int h = 40, w = 44, N = h * w * 20;
  std::vector<float> i1(h * w), tr(2 * h * w), pk(4 * h * w), pos(2 * N);
  std::vector<unsigned char> m(h * w), tok(h * w), f16(h * w);
  srand(3);
  auto rnd = [] { return rand() / (float)RAND_MAX; };
  for (int i = 0; i < h * w; ++i) {
    i1[i] = rnd(); tr[2 * i] = rnd() - 0.5f; tr[2 * i + 1] = rnd() - 0.5f;
    m[i] = rnd() > 0.15f; tok[i] = rnd() > 0.1f;
  }
  for (int y = 0; y < h; ++y) for (int x = 0; x < w; ++x) {
    int i = y * w + x; float q = __builtin_nanf("");
    pk[4 * i] = m[i] ? i1[i] : q; pk[4 * i + 1] = tok[i] ? tr[2 * i] : q;
    pk[4 * i + 2] = tok[i] ? tr[2 * i + 1] : q; pk[4 * i + 3] = 0;
    unsigned char fl = 0;
    if (x >= 1 && x + 2 < w && y >= 1 && y + 2 < h) {
      bool am = true, at = true;
      for (int a = -1; a <= 2; ++a) for (int b = -1; b <= 2; ++b) { int k = (y + a) * w + x + b; am = am && m[k]; at = at && tok[k]; }
      fl = (am ? 1 : 0) | (at ? 2 : 0);
    }
    f16[i] = fl;
  }
  for (int i = 0; i < 2 * N; ++i) pos[i] = (rnd() - 0.5f) * 8.f;
  float *di1, *dtr, *dpk, *dpos, *dout; unsigned char *dm, *dtok, *df;
  cudaMalloc(&di1, 4 * h * w); cudaMalloc(&dtr, 8 * h * w); cudaMalloc(&dpk, 16 * h * w);
  cudaMalloc(&dpos, 8 * N); cudaMalloc(&dout, 32 * N); cudaMalloc(&dm, h * w); cudaMalloc(&dtok, h * w); cudaMalloc(&df, h * w);
  cudaMemcpy(di1, i1.data(), 4 * h * w, cudaMemcpyHostToDevice);
  cudaMemcpy(dtr, tr.data(), 8 * h * w, cudaMemcpyHostToDevice);
  cudaMemcpy(dpk, pk.data(), 16 * h * w, cudaMemcpyHostToDevice);
  cudaMemcpy(dpos, pos.data(), 8 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dm, m.data(), h * w, cudaMemcpyHostToDevice);
  cudaMemcpy(dtok, tok.data(), h * w, cudaMemcpyHostToDevice);
  cudaMemcpy(df, f16.data(), h * w, cudaMemcpyHostToDevice);
  SampleSrc S{di1, dm, dtr, dtok, (const float4*)dpk, df, h, w};
  k<<<(N + 127) / 128, 128>>>(S, (const float4*)dpk, N, dpos, dout);
  std::vector<float> o(8 * N);
  cudaMemcpy(o.data(), dout, 32 * N, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < N && bad < 10; ++i) {
    bool diff = o[8*i+2] != o[8*i+3] || o[8*i+6] != o[8*i+7] || (o[8*i+2] && o[8*i] != o[8*i+1]) || (o[8*i+6] && o[8*i+4] != o[8*i+5]);
    if (diff) { ++bad; int X = i % w, Y = (i / w) % h; int ix = X + (int)floorf(pos[2*i]), iy = Y + (int)floorf(pos[2*i+1]); unsigned mm = 0, tt = 0; for (int a = 0; a < 4; ++a) for (int b = 0; b < 4; ++b) { int r = iy + a - 1, c = ix + b - 1; bool in = r >= 0 && r < h && c >= 0 && c < w; mm |= (in && m[r*w+c] ? 1u : 0u) << (4*a+b); tt |= (in && tok[r*w+c] ? 1u : 0u) << (4*a+b); } printf("i=%d mask=%04x tok=%04x i1 %a vs %a, d %a vs %a\n", i, mm, tt, o[8*i], o[8*i+1], o[8*i+4], o[8*i+5]); }
  }
  printf("mismatches (first 10 shown): %d of %d\n", bad, N);
  return 0;
}
