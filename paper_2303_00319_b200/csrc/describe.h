// Internal interface of the descriptor stage (see describe.cu).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace r2 {

struct DescribeArgs {
  int B, H, W, O;
  const int32_t* kp_x;
  const int32_t* kp_y;
  const int32_t* kp_count;
  int kp_stride;
  int patch, grid;
  double ratio;
  bool rotate;
  int mode;            // 0 plain, 1 ring, 2 rift2
  __half* counts;      // [B][cap][stride]
  int stride, cap;
  int32_t* sqnorm;
  int32_t* kp;
  uint8_t* variant;
  int32_t* count;
  int32_t* skipped;
  const double* kp_xd = nullptr;   // float64 keypoints (rift2_describe_f64) instead of kp_x / kp_y
  const double* kp_yd = nullptr;
};

size_t describe_workspace_bytes(int B, int kp_stride, int grid, int O);
size_t describe_workspace_bytes_hw(int B, int H, int W, int kp_stride, int grid, int O);
int describe_run(const uint8_t* mim, const DescribeArgs& a, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace r2
