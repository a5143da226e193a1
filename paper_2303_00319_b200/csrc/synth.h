// Internal interface of the on-device target synthesis (see synth.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace r2 {

constexpr int kSynthParams = 8;        // per image: inverse map (6), gamma, flags
constexpr int kSynthInverted = 1;      // flags bit 0: v -> 1 - v
constexpr int kSynthRadiometric = 2;   // flags bit 1: inversion / gamma / speckle / renormalisation

struct SynthArgs {
  const double* src;         // [n_images] source images, float64 H x W, image stride src_stride elements
  long long src_stride;
  int n_images, H, W;
  const double* params;      // [n_images][8]: i00 i01 i02 i10 i11 i12 (target -> source), gamma, flags
  const int32_t* looks;      // [n_images] speckle looks (0 = none)
  unsigned long long seed;   // Philox key
  int first_image;           // Philox counter word 2 = first_image + image
  float* dst;                // [n_images] targets, float32, image stride dst_stride
  long long dst_stride;
  float* dst_src_copy;       // optional float32 copy of each source (image stride copy_stride)
  long long copy_stride;
};

size_t synth_workspace_bytes(int n_images, int H, int W);
int blobs_run(const double* blobs, int n_images, int n_blobs, int H, int W, double* out, cudaStream_t st);
int normals_run(unsigned long long seed, int first_image, int n_images, size_t n, float* out, cudaStream_t st);
int synth_run(const SynthArgs& a, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace r2
