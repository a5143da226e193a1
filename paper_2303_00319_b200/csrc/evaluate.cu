// Ground-truth evaluation of match sets on the device.
//
// Restates ref: pkg/src/rift2/evalbench.py:63-96 (evaluate) for a batch of
// pairs: a match (r, t) is correct when the ground-truth transform carries
// reference keypoint r to within `residual_threshold` (strictly less) of
// target keypoint t; RMSE over the correct matches, clamped to rmse_cap,
// +inf with none; success = n_correct >= success_min_matches.  Indices that
// do not resolve to keypoints set the pair's `bad` flag (the reference raises
// IntegrityError, :69-71).
//
// One CTA per pair; float64 throughout with the reference's operation order
// (p' = p @ R^T + t, ref: imaging.py:71-74; residual = sqrt(dx^2 + dy^2),
// np.linalg.norm), products and sums rounded separately (no FMA contraction).
#include "common.cuh"
#include "evaluate.h"

namespace r2 {

namespace {

constexpr int kEvalThreads = 256;

__global__ void __launch_bounds__(kEvalThreads) k_evaluate(EvalArgs a) {
  __shared__ double s_sum[kEvalThreads / 32];
  __shared__ int s_cnt[kEvalThreads / 32], s_bad[kEvalThreads / 32];
  const int p = blockIdx.x;
  const int ri = a.ref_img[p], ti = a.tgt_img[p];
  const int n_ref = a.kp_count[ri], n_tgt = a.kp_count[ti];
  const int* rx = a.kp_x + (size_t)ri * a.kp_stride;
  const int* ry = a.kp_y + (size_t)ri * a.kp_stride;
  const int* tx = a.kp_x + (size_t)ti * a.kp_stride;
  const int* ty = a.kp_y + (size_t)ti * a.kp_stride;
  const int* mr = a.m_ref + (size_t)p * a.m_stride;
  const int* mt = a.m_tgt + (size_t)p * a.m_stride;
  const double* g = a.gt + 6 * (size_t)p;   // R00 R01 R10 R11 t0 t1
  const double r00 = g[0], r01 = g[1], r10 = g[2], r11 = g[3], t0 = g[4], t1 = g[5];
  const int n = a.m_count[p];
  double sum = 0.0;
  int cnt = 0, bad = 0;
  for (int i = threadIdx.x; i < n; i += kEvalThreads) {
    const int r = mr[i], t = mt[i];
    if (r < 0 || r >= n_ref || t < 0 || t >= n_tgt) { bad = 1; continue; }
    const double x = (double)rx[r], y = (double)ry[r];
    const double px = __dadd_rn(__dadd_rn(__dmul_rn(x, r00), __dmul_rn(y, r01)), t0);
    const double py = __dadd_rn(__dadd_rn(__dmul_rn(x, r10), __dmul_rn(y, r11)), t1);
    const double dx = __dsub_rn(px, (double)tx[t]), dy = __dsub_rn(py, (double)ty[t]);
    const double res = sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    if (res < a.threshold) {
      ++cnt;
      sum = __dadd_rn(sum, __dmul_rn(res, res));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_sum[w] = sum; s_cnt[w] = cnt; s_bad[w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0;
    int C = 0, B = 0;
    for (int k = 0; k < kEvalThreads / 32; ++k) { S += s_sum[k]; C += s_cnt[k]; B |= s_bad[k]; }
    a.n_correct[p] = C;
    a.rmse[p] = C > 0 ? fmin(sqrt(S / (double)C), a.rmse_cap) : __longlong_as_double(0x7ff0000000000000ll);
    a.success[p] = (uint8_t)(C >= a.min_matches);
    a.bad[p] = B;
  }
}

}  // namespace

int evaluate_run(const EvalArgs& a, cudaStream_t st) {
  if (a.n_pairs == 0) return 0;
  k_evaluate<<<a.n_pairs, kEvalThreads, 0, st>>>(a);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2
