// Microbenchmark: scalar FFMA/FADD vs packed FFMA2/FADD2 throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
__global__ void k_scalar(float* out, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_packed(float* out, float a, float b) {
  float2 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + 2 * i, threadIdx.x + 2 * i + 1);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], A, B);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd(float* out, float a) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = x[i] + (i & 1 ? a : -a);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fadd2(float* out, float a) {
  float2 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x + 2 * i, threadIdx.x + 2 * i + 1);
  const float2 A = make_float2(a, -a);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __fadd2_rn(x[i], A);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  const int blocks = 148 * 8, threads = 256;
  cudaMalloc(&out, blocks * threads * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double flops_elems = (double)blocks * threads * ITERS * 16;   // element-ops
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_scalar<<<blocks, threads>>>(out, 1.0001f, 0.5f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA  scalar: %.3f ms  %.1f Tfma/s\n", ms, flops_elems / ms / 1e9);
    cudaEventRecord(e0); k_packed<<<blocks, threads>>>(out, 1.0001f, 0.5f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2 packed: %.3f ms  %.1f Tfma/s\n", ms, flops_elems / ms / 1e9);
    cudaEventRecord(e0); k_fadd<<<blocks, threads>>>(out, 1.0001f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FADD  scalar: %.3f ms  %.1f Tadd/s\n", ms, flops_elems / ms / 1e9);
    cudaEventRecord(e0); k_fadd2<<<blocks, threads>>>(out, 1.0001f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("FADD2 packed: %.3f ms  %.1f Tadd/s\n", ms, flops_elems / ms / 1e9);
  }
  return 0;
}
