// Internal interface of the matching stage (see match.cu).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace r2 {

struct MatchArgs {
  const __half* counts;    // [blocks][cap][stride]
  const int32_t* sqnorm;   // [blocks][cap]
  const int32_t* kp;       // [blocks][cap]
  const int32_t* count;    // [blocks]
  int stride, cap, dim, n_pairs, n_blocks;
  const int32_t* ref_block;   // device [n_pairs]
  const int32_t* tgt_block;   // device [n_pairs]
  int tgt_kp_cap;
  int32_t* out_ref;
  int32_t* out_tgt;
  double* out_dist;
  int32_t* out_count;
};

size_t match_workspace_bytes(int n_pairs, int cap, int tgt_kp_cap);
int match_run(const MatchArgs& a, void* ws, size_t ws_bytes, cudaStream_t st);
// row-sharded matching: GEMM partials [n_pairs][cap] of 16-byte records, and the
// exact combine of n_parts gathered partial arrays ([n_parts][n_pairs][cap])
int match_partial_run(const MatchArgs& a, void* parts, cudaStream_t st);
int match_finish_run(const MatchArgs& a, const void* parts, int n_parts, void* ws, size_t ws_bytes,
                     cudaStream_t st);

// generic float64 descriptor vectors (rows grouped by keypoint id)
size_t match_vectors_workspace_bytes(int nr, int nt);
int match_vectors_run(const double* R, const int* rkp, int nr, const double* T, const int* tkp, int nt, int dim,
                      int* out_ref, int* out_tgt, double* out_dist, int* out_count, void* ws, size_t ws_bytes,
                      cudaStream_t st);

}  // namespace r2
