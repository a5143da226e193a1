// Write-pattern microbenchmark for the column pass's output (DESIGN 7c):
// 32 images x 24 planes x 1024^2 complex64 = 6.4 GB written per launch in
// different address orders.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 qwrite.cu -o qwrite
#include <cstdio>
#include <cuda_runtime.h>

constexpr int B = 32, F = 24, H = 1024, W = 1024;

// (a) the current layout and order: CTA = 4 warps = 2 direct + 2 mirror
// columns of one image, each warp writes its column of every plane as
// 4-row tile sectors: element (y, x) at ((y>>2)*W + x)*4 + (y&3)
__global__ void k_cols4(float2* Q) {
  const int b = blockIdx.y, cblk = blockIdx.x, g = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int kx = cblk * 2 + (g & 1);
  const int x = g < 2 ? kx : W - 1 - kx;
  float2* Qb = Q + (size_t)b * F * H * W;
  for (int f = 0; f < F; ++f) {
    float2* q = Qb + (size_t)f * H * W;
#pragma unroll 8
    for (int m = 0; m < 32; ++m) {
      const int y = t + 32 * m;
      q[((size_t)(y >> 2) * W + x) * 4 + (y & 3)] = make_float2(f, y);
    }
  }
}

// (b) 4 adjacent columns per warp: a store instruction writes two full
// 128-byte lines (tile rows j, j+1 x 4 columns x 4 rows)
__global__ void k_cols4x4(float2* Q) {
  const int b = blockIdx.y, cblk = blockIdx.x, g = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int x0 = (cblk * 4 + g) * 4;   // 4 warps x 4 columns = 16 columns per CTA
  float2* Qb = Q + (size_t)b * F * H * W;
  for (int f = 0; f < F; ++f) {
    float2* q = Qb + (size_t)f * H * W;
#pragma unroll 8
    for (int m = 0; m < 128; ++m) {         // 256 tile rows x 4 columns x 4 rows / 32 lanes
      const int j = 2 * m + (t >> 4), c = (t >> 2) & 3, r = t & 3;
      q[((size_t)j * W + x0 + c) * 4 + r] = make_float2(f, j);
    }
  }
}

// (b2) 2 adjacent columns per warp (a direct pair): 64 contiguous bytes per tile row
__global__ void k_cols2x4(float2* Q) {
  const int b = blockIdx.y, cblk = blockIdx.x, g = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int x0 = (cblk * 4 + g) * 2;   // 4 warps x 2 columns = 8 columns per CTA
  float2* Qb = Q + (size_t)b * F * H * W;
  for (int f = 0; f < F; ++f) {
    float2* q = Qb + (size_t)f * H * W;
#pragma unroll 8
    for (int m = 0; m < 64; ++m) {          // 256 tile rows x 2 columns x 4 rows / 32 lanes
      const int j = 4 * m + (t >> 3), c = (t >> 2) & 1, r = t & 3;
      q[((size_t)j * W + x0 + c) * 4 + r] = make_float2(f, j);
    }
  }
}

// (c) row-major planes, 16-column segments: a store writes rows y, y+1 x 16 columns
__global__ void k_rowseg16(float2* Q) {
  const int b = blockIdx.y, cblk = blockIdx.x, g = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int x0 = (cblk * 4 + g) * 4;
  (void)x0;
  const int xs = cblk * 16;
  float2* Qb = Q + (size_t)b * F * H * W;
  for (int f = 0; f < F; ++f) {
    float2* q = Qb + (size_t)f * H * W;
    if (g != 0) continue;
#pragma unroll 8
    for (int m = 0; m < 512; ++m) {
      const int y = 2 * m + (t >> 4), x = xs + (t & 15);
      q[(size_t)y * W + x] = make_float2(f, y);
    }
  }
}

// (d) contiguous
__global__ void k_fill(float2* Q, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    Q[i] = make_float2(1.f, 2.f);
}

int main() {
  const size_t n = (size_t)B * F * H * W;
  float2* Q;
  if (cudaMalloc(&Q, n * sizeof(float2)) != cudaSuccess) { printf("alloc failed\n"); return 1; }
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
    printf("%-10s %7.3f ms  %6.0f GB/s  (%s)\n", name, ms, n * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run("cols4", [&] { k_cols4<<<dim3(W / 4, B), 128>>>(Q); });
  run("cols4x4", [&] { k_cols4x4<<<dim3(W / 16, B), 128>>>(Q); });
  run("cols2x4", [&] { k_cols2x4<<<dim3(W / 8, B), 128>>>(Q); });
  run("rowseg16", [&] { k_rowseg16<<<dim3(W / 16, B), 128>>>(Q); });
  run("fill", [&] { k_fill<<<148 * 8, 256>>>(Q, n); });
  return 0;
}
