// Internal interface of the filter-bank stage (see fields.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace r2 {

// Host-derived constants of the log-Gabor bank (double precision on the host).
struct BankConsts {
  int n_scales, n_orient;
  double log_lambda[8];
  double inv_den_r, inv_den_a;
  double angle[16], cos_a[16], sin_a[16];
  double spread_cutoff, spread_gain;
  double lp_lncut;
  double thr_factor;
};

struct FieldsOutputs {
  float* mmax;
  float* mmin;
  uint8_t* mim;
  float* a_o;   // nullable
  float* pc;    // nullable
  float* amax;  // nullable
  unsigned long long* range;   // nullable [B][2][2]: per-image (lo, hi) keys of moment_min, moment_max
};

// W_n^j = exp(-2 pi i j / n), j < n, cached per (device, n); nullptr on failure.
const float2* twiddle_table(int n);

size_t fields_workspace_bytes(int B, int H, int W, int S, int O);
int fields_run(const float* images, int B, int H, int W, const BankConsts& bk, const FieldsOutputs& out,
               void* ws, size_t ws_bytes, cudaStream_t st);

// unfused reference entry points (ref: loggabor.py:131-251, mim.py:43-55)
int filter_bank_run(int H, int W, int S, int O, double min_wl, double mult, double sigma_on_f, double sigma_theta,
                    double* transfer, cudaStream_t st);
size_t apply_bank_workspace_bytes(int H, int W, int S, int O);
int apply_bank_run(const float* image, int H, int W, int S, int O, const float* transfer, float* even, float* odd,
                   float* amp, void* ws, size_t ws_bytes, cudaStream_t st);
size_t pc_stack_workspace_bytes(int H, int W, int S, int O);
int pc_stack_run(const float* even, const float* odd, const float* amp, int H, int W, const BankConsts& bk,
                 float* a_o, float* pc, float* mmax, float* mmin, void* ws, size_t ws_bytes, cudaStream_t st);
int sum_scales_run(const double* amp, int S, int O, int H, int W, double* a_o, cudaStream_t st);
int build_mim_run(const double* a_o, int O, int H, int W, int* idx, double* amax, cudaStream_t st);

// diagnostics: exact median of |z| per plane through the filter bank's median kernels
size_t debug_median_workspace_bytes(int planes, int n);
int debug_median_run(const float2* z, int planes, int n, float* amps, float* med, void* ws, size_t ws_bytes,
                     cudaStream_t st);

}  // namespace r2
