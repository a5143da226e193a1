// Internal interface of the per-patch index-map kernels (see patch.cu).
#pragma once
#include <cuda_runtime.h>

namespace r2 {

int patch_counts_run(const int* idx, const double* amp, int n, int height, int width, int n_orient, int grid,
                     double* hist, double* cells, cudaStream_t st);
int remap_run(int* idx, long long count, int n_orient, int pivot, int kind, cudaStream_t st);
int gather_run(const int* idx, const double* amp, int H, int W, double x, double y, int integer_kp, int size,
               double c, double s, int* out_idx, double* out_amp, int* oob, cudaStream_t st);

}  // namespace r2
