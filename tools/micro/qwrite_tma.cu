// TMA-store variant of qwrite.cu: the column pass's store pattern issued as
// cp.async.bulk.tensor boxes from shared memory (no FFT), per warp one
// column per box ({8 words, 1, 256}) or a warp pair's two adjacent columns
// per box ({8, 2, 256}).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 qwrite_tma.cu -o qwrite_tma
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

constexpr int B = 32, F = 24, H = 1024, W = 1024;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void store3d(const CUtensorMap* m, int x, int y, int z, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
               :: "l"(m), "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// mode 0: 4 warps, one column each (2 direct + 2 mirror as in k_cols); mode 1: warp pairs store 2 columns
template <int MODE>
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m2) {
  extern __shared__ __align__(128) float2 sm[];
  const int b = blockIdx.y, cblk = blockIdx.x, g = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int kx0 = cblk * 2;
  float2* buf = sm + g * 1024;
  for (int i = t; i < 1024; i += 32) buf[i] = make_float2(1.f, 2.f);
  __syncthreads();
  for (int f = 0; f < F; ++f) {
    const int z = (b * F + f) * 256;
    if (MODE == 0) {
      const int x = g < 2 ? kx0 + g : W - 1 - kx0 - (g - 2);
      if (t == 0) { wait_read0(); store3d(&m1, 0, x, z, buf); commit(); }
      __syncwarp();
    } else {
      if ((g & 1) == 0 && t == 0) {
        wait_read0();
        const int x = g == 0 ? kx0 : W - 2 - kx0;
        store3d(&m2, 0, x, z, sm + (g >> 1) * 2048);
        commit();
      }
      __syncwarp();
    }
  }
  if (t == 0) wait0();
}

int main() {
  const size_t n = (size_t)B * F * H * W;
  float2* Q;
  if (cudaMalloc(&Q, n * sizeof(float2)) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  CUtensorMap m1, m2;
  cuuint64_t dims[3] = {8, (cuuint64_t)W, (cuuint64_t)B * F * (H / 4)};
  cuuint64_t strides[2] = {4 * sizeof(float2), (cuuint64_t)W * 4 * sizeof(float2)};
  cuuint32_t box1[3] = {8, 1, 256}, box2[3] = {8, 2, 256}, es[3] = {1, 1, 1};
  enc(&m1, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, Q, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, Q, dims, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 4 * 1024 * 8;
  cudaFuncSetAttribute(k_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  auto run = [&](const char* name, auto fn) {
    for (int i = 0; i < 2; ++i) fn();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(z);
    cudaEventSynchronize(z);
    float ms;
    cudaEventElapsedTime(&ms, a, z);
    ms /= 5;
    printf("%-12s %7.3f ms  %6.0f GB/s  (%s)\n", name, ms, n * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("tma_col1", [&] { k_tma<0><<<dim3(W / 4, B), 128, smem>>>(m1, m2); });
  run("tma_col2", [&] { k_tma<1><<<dim3(W / 4, B), 128, smem>>>(m1, m2); });
  return 0;
}
