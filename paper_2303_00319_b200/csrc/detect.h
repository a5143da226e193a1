// Internal interface of the keypoint stage (see detect.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace r2 {

struct DetectArgs {
  int B, H, W;
  double threshold;
  int max_points, margin;
  bool single_map;
  int32_t* kp_x;
  int32_t* kp_y;
  double* kp_resp;
  uint8_t* kp_kind;
  int32_t* kp_count;
  const unsigned long long* range;   // nullable: per-image (min, max) keys of both maps from rift2_fields
};

size_t detect_workspace_bytes(int B, int H, int W, int max_points);
// min_maps / max_maps: [B][H][W]; with single_map only min_maps is read (kind 0)
int detect_run(const float* min_maps, const float* max_maps, const DetectArgs& a, void* ws, size_t ws_bytes,
               cudaStream_t st);
int detect_run(const double* min_maps, const double* max_maps, const DetectArgs& a, void* ws, size_t ws_bytes,
               cudaStream_t st);

}  // namespace r2
