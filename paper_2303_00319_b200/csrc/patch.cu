// Per-patch index-map operations of the reference's unfused descriptor API:
//
//   ref: mim.py:58-66        patch_histogram  (counts, or amplitude mass, per index value)
//   ref: descriptor.py:145-164 encode         (per-cell index histograms; the float64
//                                             normalisation stays with the caller, as in
//                                             describe_*)
//   ref: mim.py:97-136       recode / cyclic_shift (value permutations of the ring)
//   ref: descriptor.py:85-125 extract_patch   (nearest-neighbour gather on a rotated grid)
//
// The batched descriptor kernel (describe.cu) fuses all of these; these
// kernels serve callers that use the steps one at a time.  Weighted sums
// are accumulated by one thread per bin in pixel order, so they round like
// the reference's np.bincount.
#include <cmath>

#include "common.cuh"
#include "patch.h"

namespace r2 {

// one CTA per patch (height x width; cells need a square patch): bins
// [n_orient] (hist) and/or [grid * grid * n_orient] (cells)
__global__ void __launch_bounds__(256) k_patch_counts(const int* __restrict__ idx, const double* __restrict__ amp,
                                                      int height, int width, int n_orient, int grid,
                                                      double* __restrict__ hist, double* __restrict__ cells) {
  const int p = blockIdx.x, size = width;
  const size_t np = (size_t)height * width;
  const int* ix = idx + p * np;
  const double* am = amp ? amp + p * np : nullptr;
  if (hist) {
    for (int v = threadIdx.x; v < n_orient; v += blockDim.x) {
      double acc = 0.0;
      for (size_t i = 0; i < np; ++i)
        if (ix[i] == v + 1) acc += am ? am[i] : 1.0;
      hist[(size_t)p * n_orient + v] = acc;
    }
  }
  if (cells) {
    const int cs = size / grid, nb = grid * grid * n_orient;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int cell = b / n_orient, v = b % n_orient + 1;
      const int r0 = (cell / grid) * cs, c0 = (cell % grid) * cs;
      double acc = 0.0;
      for (int r = r0; r < r0 + cs; ++r)
        for (int c = c0; c < c0 + cs; ++c) {
          const size_t i = (size_t)r * size + c;
          if (ix[i] == v) acc += am ? am[i] : 1.0;
        }
      cells[(size_t)p * nb + b] = acc;
    }
  }
}

int patch_counts_run(const int* idx, const double* amp, int n, int height, int width, int n_orient, int grid,
                     double* hist, double* cells, cudaStream_t st) {
  if (n > 0) k_patch_counts<<<n, 256, 0, st>>>(idx, amp, height, width, n_orient, grid, hist, cells);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// kind 0 recode: v >= p -> v - p + 1, else v + n - p + 1; kind 1 cyclic
// shift: (v - p) mod n + 1; value 0 stays 0
__global__ void __launch_bounds__(256) k_remap(int* __restrict__ idx, long long count, int n, int pivot, int kind) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    const int v = idx[i];
    if (v == 0) continue;
    idx[i] = kind == 0 ? (v >= pivot ? v - pivot + 1 : v + n - pivot + 1) : ((v - pivot) % n + n) % n + 1;
  }
}

int remap_run(int* idx, long long count, int n_orient, int pivot, int kind, cudaStream_t st) {
  if (count > 0) {
    const unsigned blocks = (unsigned)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
    k_remap<<<blocks, 256, 0, st>>>(idx, count, n_orient, pivot, kind);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// Rotated nearest-neighbour gather (ref: descriptor.py:46-64,70-82,114-125):
// sample (i, j) sits at u = j + 0.5 - size/2, v = i + 0.5 - size/2 rotated by
// (c, s) (snapped cos / sin from the caller); integer keypoints round the
// offset first and add the pixel (the reference's gather-table path),
// others round x + offset.  Products and sums are separately rounded (no
// FMA contraction) as numpy evaluates them.  *oob = 1 when any sample leaves
// the map (the caller returns None).
__global__ void __launch_bounds__(256) k_gather(const int* __restrict__ idx, const double* __restrict__ amp, int H,
                                                int W, double x, double y, int integer_kp, int size, double c,
                                                double s, int* __restrict__ out_idx, double* __restrict__ out_amp,
                                                int* __restrict__ oob) {
  const int n = size * size;
  const double half = size / 2.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int i = k / size, j = k % size;
    const double u = __dsub_rn(__dadd_rn((double)j, 0.5), half);
    const double v = __dsub_rn(__dadd_rn((double)i, 0.5), half);
    const double ux = __dsub_rn(__dmul_rn(c, u), __dmul_rn(s, v));
    const double vy = __dadd_rn(__dmul_rn(s, u), __dmul_rn(c, v));
    long long sx, sy;
    if (integer_kp) {
      sx = (long long)x + (long long)floor(__dadd_rn(ux, 0.5));
      sy = (long long)y + (long long)floor(__dadd_rn(vy, 0.5));
    } else {
      sx = (long long)floor(__dadd_rn(__dadd_rn(x, ux), 0.5));
      sy = (long long)floor(__dadd_rn(__dadd_rn(y, vy), 0.5));
    }
    if (sx < 0 || sy < 0 || sx >= W || sy >= H) {
      *oob = 1;
      continue;
    }
    const size_t q = (size_t)sy * W + sx;
    out_idx[k] = idx[q];
    if (out_amp) out_amp[k] = amp ? amp[q] : 0.0;
  }
}

int gather_run(const int* idx, const double* amp, int H, int W, double x, double y, int integer_kp, int size,
               double c, double s, int* out_idx, double* out_amp, int* oob, cudaStream_t st) {
  const int n = size * size;
  cudaMemsetAsync(oob, 0, sizeof(int), st);
  k_gather<<<(n + 255) / 256, 256, 0, st>>>(idx, amp, H, W, x, y, integer_kp, size, c, s, out_idx, out_amp, oob);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2
