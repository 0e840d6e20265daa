// Minimal TMA 3-D box load probe (diagnostic tool, not part of the library).
// usage: tma_probe bx by bz x0 y0
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, float* out, int x0, int y0, int bytes) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  float* st = reinterpret_cast<float*>(base + 1024);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(s32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 :: "r"(s32(st)), "l"((uint64_t)&tm), "r"(x0), "r"(y0), "r"(0), "r"(s32(bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(s32(bar)), "r"(0) : "memory");
  for (int k = threadIdx.x; k < bytes / 4; k += blockDim.x) out[k] = st[k];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int bx = atoi(argv[1]), by = atoi(argv[2]), bz = atoi(argv[3]), x0 = atoi(argv[4]), y0 = atoi(argv[5]);
  int w = 64, h = 40, planes = 12;
  size_t n = (size_t)w * h;
  float *src, *out;
  cudaMalloc(&src, n * planes * 4);
  cudaMalloc(&out, 256 * 256 * 4);
  float* hs = (float*)malloc(n * planes * 4);
  for (size_t i = 0; i < n * planes; ++i) hs[i] = (float)i;
  cudaMemcpy(src, hs, n * planes * 4, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)w * 4, (cuuint64_t)n * 4};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz}, es[3] = {1, 1, 1};
  CUresult r = ((Enc)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = bx * by * bz * 4;
  int smem = bytes + 4096;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 256, smem>>>(tm, out, x0, y0, bytes);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[2];
  cudaMemcpy(ho, out + bx + 1, 8, cudaMemcpyDeviceToHost);
  printf("box %dx%dx%d at (%d,%d) enc=%d bytes=%d: %s  out[1][1]=%g (expect %g)\n", bx, by, bz, x0, y0, (int)r, bytes,
         cudaGetErrorString(e), ho[0], (double)((y0 + 1) * w + x0 + 1));
  return e != cudaSuccess;
}
