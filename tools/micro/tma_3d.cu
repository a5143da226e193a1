// Which 3-D TMA box configurations execute on sm_100a?  usage: tma_3d BOX0 BOX1 X0 X1 ALIGN
// Tensor: uint32 (8, 1024, 64) -- the 4-row column tiles of a 1,024-wide plane viewed as 32-bit words.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, int x0, int x1, int z, int bytes, int align, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  __shared__ uint64_t bar;
  uint8_t* dst = raw + align;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 :: "r"(su(dst)), "l"(&m), "r"(x0), "r"(x1), "r"(z), "r"(su(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" :: "r"(su(&bar)) : "memory");
  unsigned s = 0;
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) s += reinterpret_cast<unsigned*>(dst)[i];
  atomicAdd(out, s);
}
int main(int argc, char** argv) {
  int b0 = atoi(argv[1]), b1 = atoi(argv[2]), x0 = atoi(argv[3]), x1 = atoi(argv[4]), align = atoi(argv[5]);
  const int D0 = 8, D1 = 1024, D2 = 64;
  unsigned* img; unsigned* out;
  cudaMalloc(&img, 4 * D0 * D1 * D2);
  {
    unsigned* h = (unsigned*)malloc(4 * D0 * D1 * D2);
    for (int i = 0; i < D0 * D1 * D2; ++i) h[i] = i % 7;
    cudaMemcpy(img, h, 4 * D0 * D1 * D2, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  void* f = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)D0, (cuuint64_t)D1, (cuuint64_t)D2};
  cuuint64_t str[2] = {(cuuint64_t)D0 * 4, (cuuint64_t)D0 * D1 * 4};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, img, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int bytes = b0 * b1 * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 2048);
  k<<<1, 128, bytes + 2048>>>(m, x0, x1, 3, bytes, align, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h = 0; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("box %dx%d at (%d,%d) align %d: encode %d, run: %s, sum %u\n", b0, b1, x0, x1, align, (int)r, cudaGetErrorString(e), h);
  return 0;
}
