// Internal interface of the ground-truth evaluation (see evaluate.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace r2 {

struct EvalArgs {
  const int32_t* kp_x;       // [images][kp_stride]
  const int32_t* kp_y;
  const int32_t* kp_count;   // [images]
  int kp_stride;
  const int32_t* ref_img;    // [n_pairs] image index of each pair's reference / target
  const int32_t* tgt_img;
  const int32_t* m_ref;      // [n_pairs][m_stride] match rows (keypoint indices)
  const int32_t* m_tgt;
  const int32_t* m_count;    // [n_pairs]
  int m_stride, n_pairs;
  const double* gt;          // [n_pairs][6]: R00 R01 R10 R11 t0 t1 (reference -> target)
  double threshold, rmse_cap;
  int min_matches;
  int32_t* n_correct;        // [n_pairs]
  double* rmse;
  uint8_t* success;
  int32_t* bad;              // [n_pairs] 1 = a match index did not resolve
};

int evaluate_run(const EvalArgs& a, cudaStream_t st);

}  // namespace r2
