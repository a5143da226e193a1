// Which uint8 TMA box configurations execute on sm_100a?  usage: tma_u8 BOXW BOXH X Y ALIGN
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int x, int y, int bytes, int align, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  __shared__ uint64_t bar;
  uint8_t* dst = raw + align;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(su(dst)), "l"(&m), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" :: "r"(su(&bar)) : "memory");
  unsigned s = 0;
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) s += dst[i];
  atomicAdd(out, s);
}
int main(int argc, char** argv) {
  int bw = atoi(argv[1]), bh = atoi(argv[2]), x = atoi(argv[3]), y = atoi(argv[4]), align = atoi(argv[5]);
  const int W = 512, H = 512;
  uint8_t* img; unsigned* out;
  cudaMalloc(&img, W * H); cudaMemset(img, 1, W * H);
  cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  cuuint64_t str[1] = {(cuuint64_t)W};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int bytes = bw * bh;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 2048);
  k<<<1, 128, bytes + 2048>>>(m, x, y, bytes, align, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h = 0; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("box %dx%d at (%d,%d) align %d: encode %d, run: %s, sum %u\n", bw, bh, x, y, align, (int)r, cudaGetErrorString(e), h);
  return 0;
}
