// extern "C" boundary of librift2_b200.so (declared in include/rift2_b200.h).
//
// Argument validation mirrors the reference's preconditions so the Python
// layer can raise the same exception types:
//   ref: pkg/src/rift2/loggabor.py:57-67   (BankParams.__post_init__)
//   ref: pkg/src/rift2/loggabor.py:134-135 (filter bank needs >= 16 px)
//   ref: pkg/src/rift2/detector.py:96-99   (finite map, threshold > 0)
//   ref: pkg/src/rift2/matcher.py:105-106  (non-empty descriptor lists)
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/rift2_b200.h"
#include "detect.h"
#include "describe.h"
#include "evaluate.h"
#include "synth.h"
#include "fields.h"
#include "match.h"
#include "patch.h"

namespace {

thread_local char g_err[512] = "";

int32_t fail(int32_t code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int32_t cuda_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(RIFT2_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
  return RIFT2_OK;
}

int32_t map_internal(int32_t rc, const char* where) {
  if (rc == 0) return RIFT2_OK;
  if (rc == 3) {
    cudaError_t e = cudaGetLastError();
    return fail(RIFT2_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
  }
  if (rc == 1) return fail(RIFT2_BAD_ARGUMENT, "%s: workspace too small or bad argument", where);
  if (rc == 4) return fail(RIFT2_CAPACITY, "%s: output capacity exceeded", where);
  return fail(RIFT2_UNSUPPORTED, "%s: unsupported size or parameter", where);
}

// any length: radix-2/3/4/5/8 Stockham passes plus runtime-radix passes for
// the other prime factors (fft.cuh generic_pass_any)
bool fft_len_ok(int n) { return n >= 1; }

int32_t bank_consts(const rift2_bank_params* p, r2::BankConsts& k) {
  if (!p) return fail(RIFT2_BAD_ARGUMENT, "params is NULL");
  if (p->n_scales < 1) return fail(RIFT2_BAD_ARGUMENT, "n_scales must be >= 1");
  if (p->n_orient < 2) return fail(RIFT2_BAD_ARGUMENT, "n_orient must be >= 2");
  if (!(p->min_wavelength >= 2)) return fail(RIFT2_BAD_ARGUMENT, "min_wavelength must be >= 2");
  if (!(p->scale_mult > 1)) return fail(RIFT2_BAD_ARGUMENT, "scale_mult must be > 1");
  if (!(p->sigma_on_f > 0 && p->sigma_on_f < 1)) return fail(RIFT2_BAD_ARGUMENT, "sigma_on_f must be in (0, 1)");
  if (p->n_scales > 8 || p->n_orient > 16)
    return fail(RIFT2_UNSUPPORTED, "n_scales <= 8 and n_orient <= 16 supported");
  k.n_scales = p->n_scales;
  k.n_orient = p->n_orient;
  for (int s = 0; s < p->n_scales; ++s) k.log_lambda[s] = std::log(p->min_wavelength * std::pow(p->scale_mult, s));
  const double ls = std::log(p->sigma_on_f);
  k.inv_den_r = 1.0 / (2.0 * ls * ls);
  const double st = p->orientation_spread > 0 ? p->orientation_spread : M_PI / p->n_orient;
  k.inv_den_a = 1.0 / (2.0 * st * st);
  for (int o = 0; o < p->n_orient; ++o) {
    k.angle[o] = o * M_PI / p->n_orient;
    k.cos_a[o] = std::cos(k.angle[o]);
    k.sin_a[o] = std::sin(k.angle[o]);
  }
  k.spread_cutoff = p->spread_cutoff;
  k.spread_gain = p->spread_gain;
  k.lp_lncut = std::log(0.45);
  // ref: loggabor.py:221-227
  const double q = 1.0 / p->scale_mult;
  const double total = (1.0 - std::pow(q, p->n_scales)) / (1.0 - q);
  k.thr_factor = total / std::sqrt(std::log(4.0)) *
                 (std::sqrt(M_PI / 2.0) + p->noise_k * std::sqrt((4.0 - M_PI) / 2.0));
  return RIFT2_OK;
}

std::mutex g_tw_mu;
std::unordered_map<long long, float2*> g_tw;

}  // namespace

namespace r2 {
const float2* twiddle_table(int n) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  const long long key = ((long long)dev << 32) | (unsigned)n;
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  float2* host = new float2[n];
  for (int j = 0; j < n; ++j) {
    const double a = -2.0 * M_PI * (double)j / (double)n;
    host[j] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  float2* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(float2) * n);
  if (e == cudaSuccess) e = cudaMemcpy(d, host, sizeof(float2) * n, cudaMemcpyHostToDevice);
  delete[] host;
  if (e != cudaSuccess) { if (d) cudaFree(d); return nullptr; }
  g_tw[key] = d;
  return d;
}
}  // namespace r2

template <class T>
static int32_t detect_impl(const T* mins, const T* maxs, int32_t batch, int32_t height, int32_t width, double threshold,
                           int32_t max_points, int32_t border_margin, int32_t single_map, int32_t* kp_x,
                           int32_t* kp_y, double* kp_response, uint8_t* kp_kind, int32_t* kp_count,
                           const uint64_t* moment_range, void* workspace, size_t workspace_bytes, void* stream) {
  if (!(threshold > 0)) return fail(RIFT2_BAD_ARGUMENT, "FAST threshold must be positive");
  if (batch < 1 || height < 1 || width < 1 || max_points < 0 || border_margin < 0)
    return fail(RIFT2_BAD_ARGUMENT, "bad detect dimensions");
  if (!mins || (!single_map && !maxs) || !kp_count || !workspace || (max_points > 0 && (!kp_x || !kp_y || !kp_response || !kp_kind)))
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  if (moment_range && single_map) return fail(RIFT2_BAD_ARGUMENT, "moment_range applies to the two-map detector");
  r2::DetectArgs a{batch, height, width, threshold, max_points, border_margin, single_map != 0,
                   kp_x, kp_y, kp_response, kp_kind, kp_count,
                   reinterpret_cast<const unsigned long long*>(moment_range)};
  int32_t rc = r2::detect_run(mins, maxs, a, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_detect");
}

extern "C" {

int32_t rift2_version(void) { return 100; }

const char* rift2_last_error(void) { return g_err; }

// ------------------------------------------------------------------ fields
static int32_t check_fields_dims(int32_t batch, int32_t h, int32_t w) {
  if (batch < 1) return fail(RIFT2_BAD_ARGUMENT, "batch must be >= 1");
  if (h < 16 || w < 16) return fail(RIFT2_BAD_ARGUMENT, "filter bank needs width and height >= 16");
  if (!fft_len_ok(h) || !fft_len_ok(w)) return fail(RIFT2_UNSUPPORTED, "image %dx%d: bad FFT length", h, w);
  if ((w > 4096 || h > 4096) && !((w & (w - 1)) == 0 && (h & (h - 1)) == 0))
    return fail(RIFT2_UNSUPPORTED, "non power-of-two sizes above 4096 are not supported");
  if (w > 4096 || h > 4096) return fail(RIFT2_UNSUPPORTED, "sizes above 4096 are not supported");
  return RIFT2_OK;
}

int32_t rift2_fields_workspace_size(int32_t batch, int32_t height, int32_t width,
                                    const rift2_bank_params* params, size_t* bytes) {
  r2::BankConsts k;
  int32_t rc = bank_consts(params, k);
  if (rc) return rc;
  if ((rc = check_fields_dims(batch, height, width))) return rc;
  if (!bytes) return fail(RIFT2_BAD_ARGUMENT, "bytes is NULL");
  *bytes = r2::fields_workspace_bytes(batch, height, width, k.n_scales, k.n_orient);
  return RIFT2_OK;
}

int32_t rift2_fields(const float* images, int32_t batch, int32_t height, int32_t width,
                     const rift2_bank_params* params, float* moment_max, float* moment_min, uint8_t* mim,
                     float* a_o, float* pc_o, float* a_max, uint64_t* moment_range, void* workspace,
                     size_t workspace_bytes, void* stream) {
  r2::BankConsts k;
  int32_t rc = bank_consts(params, k);
  if (rc) return rc;
  if ((rc = check_fields_dims(batch, height, width))) return rc;
  if (!images || !moment_max || !moment_min || !mim || !workspace)
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  r2::FieldsOutputs out{moment_max, moment_min, mim, a_o, pc_o, a_max,
                        reinterpret_cast<unsigned long long*>(moment_range)};
  rc = r2::fields_run(images, batch, height, width, k, out, workspace, workspace_bytes,
                      static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_fields");
}

// ------------------------------------------------------------------ detect
int32_t rift2_detect_workspace_size(int32_t batch, int32_t height, int32_t width, int32_t max_points,
                                    size_t* bytes) {
  if (batch < 1 || height < 1 || width < 1 || max_points < 0 || !bytes)
    return fail(RIFT2_BAD_ARGUMENT, "bad detect dimensions");
  *bytes = r2::detect_workspace_bytes(batch, height, width, max_points);
  return RIFT2_OK;
}

int32_t rift2_detect_f32(const float* min_maps, const float* max_maps, int32_t batch, int32_t height,
                         int32_t width, double threshold,
                         int32_t max_points, int32_t border_margin, int32_t single_map, int32_t* kp_x,
                         int32_t* kp_y, double* kp_response, uint8_t* kp_kind, int32_t* kp_count,
                         const uint64_t* moment_range, void* workspace, size_t workspace_bytes, void* stream) {
  return detect_impl(min_maps, max_maps, batch, height, width, threshold, max_points, border_margin, single_map, kp_x, kp_y,
                     kp_response, kp_kind, kp_count, moment_range, workspace, workspace_bytes, stream);
}

int32_t rift2_detect_f64(const double* min_maps, const double* max_maps, int32_t batch, int32_t height,
                         int32_t width, double threshold,
                         int32_t max_points, int32_t border_margin, int32_t single_map, int32_t* kp_x,
                         int32_t* kp_y, double* kp_response, uint8_t* kp_kind, int32_t* kp_count,
                         const uint64_t* moment_range, void* workspace, size_t workspace_bytes, void* stream) {
  return detect_impl(min_maps, max_maps, batch, height, width, threshold, max_points, border_margin, single_map, kp_x, kp_y,
                     kp_response, kp_kind, kp_count, moment_range, workspace, workspace_bytes, stream);
}

// ---------------------------------------------------------------- describe
int32_t rift2_describe_workspace_size(int32_t batch, int32_t kp_stride, int32_t grid, int32_t n_orient,
                                      size_t* bytes) {
  if (batch < 1 || kp_stride < 0 || grid < 1 || grid > 16 || n_orient < 2 || n_orient > 16 || !bytes)
    return fail(RIFT2_BAD_ARGUMENT, "bad describe dimensions");
  *bytes = r2::describe_workspace_bytes(batch, kp_stride, grid, n_orient);
  return RIFT2_OK;
}

int32_t rift2_describe_workspace_size_hw(int32_t batch, int32_t height, int32_t width, int32_t kp_stride,
                                         int32_t grid, int32_t n_orient, size_t* bytes) {
  if (batch < 1 || height < 1 || width < 1 || kp_stride < 0 || grid < 1 || grid > 16 || n_orient < 2 ||
      n_orient > 16 || !bytes)
    return fail(RIFT2_BAD_ARGUMENT, "bad describe dimensions");
  *bytes = r2::describe_workspace_bytes_hw(batch, height, width, kp_stride, grid, n_orient);
  return RIFT2_OK;
}

}  // extern "C"

static int32_t describe_impl(const uint8_t* mim, int32_t batch, int32_t height, int32_t width, int32_t n_orient,
                             const int32_t* kp_x, const int32_t* kp_y, const double* kp_xd, const double* kp_yd,
                             const int32_t* kp_count, int32_t kp_stride, int32_t patch_size, int32_t grid,
                             double dominant_ratio, int32_t rotate_patch, int32_t mode, void* desc_counts,
                             int32_t desc_stride, int32_t desc_capacity, int32_t* desc_sqnorm, int32_t* desc_kp,
                             uint8_t* desc_variant, int32_t* desc_count, int32_t* desc_skipped, void* workspace,
                             size_t workspace_bytes, void* stream) {
  if (batch < 1 || height < 1 || width < 1 || kp_stride < 0) return fail(RIFT2_BAD_ARGUMENT, "bad dimensions");
  if (n_orient < 2 || n_orient > 16) return fail(RIFT2_UNSUPPORTED, "n_orient must be in [2, 16]");
  if (grid < 1 || patch_size < grid || patch_size % grid != 0)
    return fail(RIFT2_BAD_ARGUMENT, "patch %d does not divide into %d cells", patch_size, grid);
  if (patch_size > 256 || grid > 16 || grid * grid * n_orient > desc_stride)
    return fail(RIFT2_UNSUPPORTED, "patch_size <= 256, grid <= 16 and grid^2*n_orient <= desc_stride required");
  if (!(dominant_ratio > 0 && dominant_ratio <= 1)) return fail(RIFT2_BAD_ARGUMENT, "dominant_ratio in (0, 1]");
  if (mode < 0 || mode > 3)
    return fail(RIFT2_BAD_ARGUMENT, "mode must be 0 plain, 1 ring, 2 rift2, 3 ring reference / plain target");
  // every keypoint yields at most `per` rows, so this capacity can never overflow
  const int64_t per = mode == 0 ? 1 : ((mode == 1 || mode == 3) ? n_orient : 2);
  if ((int64_t)desc_capacity < per * kp_stride)
    return fail(RIFT2_CAPACITY, "desc_capacity %d < %lld rows per keypoint x kp_stride %d", desc_capacity,
                (long long)per, kp_stride);
  if (!mim || !kp_count || !desc_counts || !desc_sqnorm || !desc_kp || !desc_variant || !desc_count ||
      !desc_skipped || !workspace)
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  if (kp_stride > 0 && !((kp_x && kp_y) || (kp_xd && kp_yd))) return fail(RIFT2_BAD_ARGUMENT, "NULL keypoints");
  r2::DescribeArgs a{batch, height, width, n_orient, kp_x, kp_y, kp_count, kp_stride, patch_size, grid,
                     dominant_ratio, rotate_patch != 0, mode, static_cast<__half*>(desc_counts), desc_stride,
                     desc_capacity, desc_sqnorm, desc_kp, desc_variant, desc_count, desc_skipped, kp_xd, kp_yd};
  int32_t rc = r2::describe_run(mim, a, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_describe");
}

extern "C" {

int32_t rift2_describe(const uint8_t* mim, int32_t batch, int32_t height, int32_t width, int32_t n_orient,
                       const int32_t* kp_x, const int32_t* kp_y, const int32_t* kp_count, int32_t kp_stride,
                       int32_t patch_size, int32_t grid, double dominant_ratio, int32_t rotate_patch,
                       int32_t mode, void* desc_counts, int32_t desc_stride, int32_t desc_capacity,
                       int32_t* desc_sqnorm, int32_t* desc_kp, uint8_t* desc_variant, int32_t* desc_count,
                       int32_t* desc_skipped, void* workspace, size_t workspace_bytes, void* stream) {
  return describe_impl(mim, batch, height, width, n_orient, kp_x, kp_y, nullptr, nullptr, kp_count, kp_stride,
                       patch_size, grid, dominant_ratio, rotate_patch, mode, desc_counts, desc_stride,
                       desc_capacity, desc_sqnorm, desc_kp, desc_variant, desc_count, desc_skipped, workspace,
                       workspace_bytes, stream);
}

int32_t rift2_describe_f64(const uint8_t* mim, int32_t batch, int32_t height, int32_t width, int32_t n_orient,
                           const double* kp_x, const double* kp_y, const int32_t* kp_count, int32_t kp_stride,
                           int32_t patch_size, int32_t grid, double dominant_ratio, int32_t rotate_patch,
                           int32_t mode, void* desc_counts, int32_t desc_stride, int32_t desc_capacity,
                           int32_t* desc_sqnorm, int32_t* desc_kp, uint8_t* desc_variant, int32_t* desc_count,
                           int32_t* desc_skipped, void* workspace, size_t workspace_bytes, void* stream) {
  return describe_impl(mim, batch, height, width, n_orient, nullptr, nullptr, kp_x, kp_y, kp_count, kp_stride,
                       patch_size, grid, dominant_ratio, rotate_patch, mode, desc_counts, desc_stride,
                       desc_capacity, desc_sqnorm, desc_kp, desc_variant, desc_count, desc_skipped, workspace,
                       workspace_bytes, stream);
}

// ------------------------------------------------------------------- match
int32_t rift2_match_workspace_size(int32_t n_pairs, int32_t desc_capacity, int32_t tgt_kp_capacity,
                                   size_t* bytes) {
  if (n_pairs < 1 || desc_capacity < 0 || tgt_kp_capacity < 0 || !bytes)
    return fail(RIFT2_BAD_ARGUMENT, "bad match dimensions");
  *bytes = r2::match_workspace_bytes(n_pairs, desc_capacity, tgt_kp_capacity);
  return RIFT2_OK;
}

int32_t rift2_match(const void* desc_counts, const int32_t* desc_sqnorm, const int32_t* desc_kp,
                    const int32_t* desc_count, int32_t n_blocks, int32_t desc_stride, int32_t desc_capacity,
                    int32_t dim, int32_t n_pairs, const int32_t* ref_block, const int32_t* tgt_block, int32_t tgt_kp_capacity,
                    int32_t* out_ref, int32_t* out_tgt, double* out_dist, int32_t* out_count, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (n_pairs < 1 || n_blocks < 1 || desc_capacity < 1 || dim < 1 || dim > desc_stride || desc_stride % 8 != 0)
    return fail(RIFT2_BAD_ARGUMENT, "bad match dimensions");
  if (desc_stride != 224 && desc_stride != 256) return fail(RIFT2_UNSUPPORTED, "desc_stride must be 224 or 256");
  if (!desc_counts || !desc_sqnorm || !desc_kp || !desc_count || !ref_block || !tgt_block || !out_ref ||
      !out_tgt || !out_dist || !out_count || !workspace)
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  r2::MatchArgs a{static_cast<const __half*>(desc_counts), desc_sqnorm, desc_kp, desc_count, desc_stride,
                  desc_capacity, dim, n_pairs, n_blocks, ref_block, tgt_block, tgt_kp_capacity, out_ref, out_tgt,
                  out_dist, out_count};
  int32_t rc = r2::match_run(a, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_match");
}

static int32_t match_args_check(int32_t n_pairs, int32_t n_blocks, int32_t desc_capacity, int32_t dim,
                                int32_t desc_stride) {
  if (n_pairs < 1 || n_blocks < 1 || desc_capacity < 1 || dim < 1 || dim > desc_stride || desc_stride % 8 != 0)
    return fail(RIFT2_BAD_ARGUMENT, "bad match dimensions");
  if (desc_stride != 224 && desc_stride != 256) return fail(RIFT2_UNSUPPORTED, "desc_stride must be 224 or 256");
  return RIFT2_OK;
}

static_assert(sizeof(rift2_match_part) == 16, "rift2_match_part is the kernel's 16-byte partial record");

int32_t rift2_match_partial(const void* desc_counts, const int32_t* desc_sqnorm, const int32_t* desc_kp,
                            const int32_t* desc_count, int32_t n_blocks, int32_t desc_stride, int32_t desc_capacity,
                            int32_t dim, int32_t n_pairs, const int32_t* ref_block, const int32_t* tgt_block,
                            rift2_match_part* out_parts, void* stream) {
  if (int32_t rc = match_args_check(n_pairs, n_blocks, desc_capacity, dim, desc_stride)) return rc;
  if (!desc_counts || !desc_sqnorm || !desc_kp || !desc_count || !ref_block || !tgt_block || !out_parts)
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  r2::MatchArgs a{static_cast<const __half*>(desc_counts), desc_sqnorm, desc_kp, desc_count, desc_stride,
                  desc_capacity, dim, n_pairs, n_blocks, ref_block, tgt_block, 0, nullptr, nullptr, nullptr, nullptr};
  return map_internal(r2::match_partial_run(a, out_parts, static_cast<cudaStream_t>(stream)), "rift2_match_partial");
}

int32_t rift2_match_finish(const rift2_match_part* parts, int32_t n_parts, const void* desc_counts,
                           const int32_t* desc_sqnorm, const int32_t* desc_kp, const int32_t* desc_count,
                           int32_t n_blocks, int32_t desc_stride, int32_t desc_capacity, int32_t dim, int32_t n_pairs,
                           const int32_t* ref_block, const int32_t* tgt_block, int32_t tgt_kp_capacity,
                           int32_t* out_ref, int32_t* out_tgt, double* out_dist, int32_t* out_count, void* workspace,
                           size_t workspace_bytes, void* stream) {
  if (int32_t rc = match_args_check(n_pairs, n_blocks, desc_capacity, dim, desc_stride)) return rc;
  if (n_parts < 1) return fail(RIFT2_BAD_ARGUMENT, "n_parts must be >= 1");
  if (!parts || !desc_counts || !desc_sqnorm || !desc_kp || !desc_count || !ref_block || !tgt_block || !out_ref ||
      !out_tgt || !out_dist || !out_count || !workspace)
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  r2::MatchArgs a{static_cast<const __half*>(desc_counts), desc_sqnorm, desc_kp, desc_count, desc_stride,
                  desc_capacity, dim, n_pairs, n_blocks, ref_block, tgt_block, tgt_kp_capacity, out_ref, out_tgt,
                  out_dist, out_count};
  return map_internal(r2::match_finish_run(a, parts, n_parts, workspace, workspace_bytes,
                                           static_cast<cudaStream_t>(stream)), "rift2_match_finish");
}

int32_t rift2_match_vectors_workspace_size(int32_t n_ref, int32_t n_tgt, size_t* bytes) {
  if (n_ref < 1 || n_tgt < 1 || !bytes) return fail(RIFT2_BAD_ARGUMENT, "descriptor lists must be nonempty");
  *bytes = r2::match_vectors_workspace_bytes(n_ref, n_tgt);
  return RIFT2_OK;
}

int32_t rift2_match_vectors(const double* ref_vec, const int32_t* ref_kp, int32_t n_ref, const double* tgt_vec,
                            const int32_t* tgt_kp, int32_t n_tgt, int32_t dim, int32_t* out_ref, int32_t* out_tgt,
                            double* out_dist, int32_t* out_count, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (n_ref < 1 || n_tgt < 1) return fail(RIFT2_BAD_ARGUMENT, "descriptor lists must be nonempty");
  if (dim < 1 || !ref_vec || !ref_kp || !tgt_vec || !tgt_kp || !out_ref || !out_tgt || !out_dist || !out_count ||
      !workspace)
    return fail(RIFT2_BAD_ARGUMENT, "bad match_vectors arguments");
  int32_t rc = r2::match_vectors_run(ref_vec, ref_kp, n_ref, tgt_vec, tgt_kp, n_tgt, dim, out_ref, out_tgt,
                                     out_dist, out_count, workspace, workspace_bytes,
                                     static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_match_vectors");
}

int32_t rift2_evaluate(const int32_t* kp_x, const int32_t* kp_y, const int32_t* kp_count, int32_t kp_stride,
                       const int32_t* ref_img, const int32_t* tgt_img, const int32_t* match_ref,
                       const int32_t* match_tgt, const int32_t* match_count, int32_t match_stride, int32_t n_pairs,
                       const double* gt, double residual_threshold, double rmse_cap, int32_t success_min_matches,
                       int32_t* out_n_correct, double* out_rmse, uint8_t* out_success, int32_t* out_bad,
                       void* stream) {
  if (n_pairs < 0 || kp_stride < 0 || match_stride < 0) return fail(RIFT2_BAD_ARGUMENT, "negative size");
  if (n_pairs > 0 && (!kp_x || !kp_y || !kp_count || !ref_img || !tgt_img || !match_ref || !match_tgt ||
                      !match_count || !gt || !out_n_correct || !out_rmse || !out_success || !out_bad))
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  if (!(residual_threshold > 0.0) || !(rmse_cap > 0.0))
    return fail(RIFT2_BAD_ARGUMENT, "residual_threshold and rmse_cap must be > 0");
  r2::EvalArgs a{kp_x, kp_y, kp_count, kp_stride, ref_img, tgt_img, match_ref, match_tgt, match_count,
                 match_stride, n_pairs, gt, residual_threshold, rmse_cap, success_min_matches,
                 out_n_correct, out_rmse, out_success, out_bad};
  return map_internal(r2::evaluate_run(a, static_cast<cudaStream_t>(stream)), "rift2_evaluate");
}

int32_t rift2_synth_blobs(const double* blobs, int32_t n_images, int32_t n_blobs, int32_t height, int32_t width,
                          double* out, void* stream) {
  if (n_images < 0 || n_blobs < 0 || height < 1 || width < 1 || !out || (n_blobs > 0 && !blobs))
    return fail(RIFT2_BAD_ARGUMENT, "bad blob arguments");
  return map_internal(r2::blobs_run(blobs, n_images, n_blobs, height, width, out, static_cast<cudaStream_t>(stream)),
                      "rift2_synth_blobs");
}

int32_t rift2_synth_normals(uint64_t seed, int32_t first_image, int32_t n_images, int64_t n, float* out,
                            void* stream) {
  if (n_images < 0 || n < 0 || (n > 0 && !out)) return fail(RIFT2_BAD_ARGUMENT, "bad normals arguments");
  return map_internal(r2::normals_run(seed, first_image, n_images, (size_t)n, out, static_cast<cudaStream_t>(stream)),
                      "rift2_synth_normals");
}

int32_t rift2_synth_workspace_size(int32_t n_images, int32_t height, int32_t width, size_t* bytes) {
  if (n_images < 0 || height < 2 || width < 2 || !bytes) return fail(RIFT2_BAD_ARGUMENT, "bad synthesis sizes");
  *bytes = r2::synth_workspace_bytes(n_images, height, width);
  return RIFT2_OK;
}

int32_t rift2_synth_targets(const double* src, int64_t src_image_stride, int32_t n_images, int32_t height,
                            int32_t width, const double* params, const int32_t* looks, uint64_t seed,
                            int32_t first_image, float* dst, int64_t dst_image_stride, float* dst_src_copy,
                            int64_t copy_image_stride, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_images < 0 || height < 2 || width < 2 || (int64_t)height * width >= (1ll << 31))
    return fail(RIFT2_BAD_ARGUMENT, "bad synthesis sizes");
  const int64_t n = (int64_t)height * width;
  if (n_images > 1 && (src_image_stride < n || dst_image_stride < n || (dst_src_copy && copy_image_stride < n)))
    return fail(RIFT2_BAD_ARGUMENT, "image strides must be >= height * width");
  if (n_images > 0 && (!src || !params || !looks || !dst || !workspace))
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  r2::SynthArgs a{src, src_image_stride, n_images, height, width, params, looks, (unsigned long long)seed,
                  first_image, dst, dst_image_stride, dst_src_copy, copy_image_stride};
  return map_internal(r2::synth_run(a, workspace, workspace_bytes, static_cast<cudaStream_t>(stream)),
                      "rift2_synth_targets");
}

int32_t rift2_debug_median_workspace_size(int32_t planes, int32_t n, size_t* bytes) {
  if (planes < 1 || n < 1 || n >= (1 << 28) || !bytes) return fail(RIFT2_BAD_ARGUMENT, "bad median plane sizes");
  *bytes = r2::debug_median_workspace_bytes(planes, n);
  return RIFT2_OK;
}

int32_t rift2_debug_median(const void* planes_c64, int32_t planes, int32_t n, float* amplitudes, float* medians,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (planes < 1 || n < 1 || n >= (1 << 28)) return fail(RIFT2_BAD_ARGUMENT, "bad median plane sizes");
  if (!planes_c64 || !amplitudes || !medians || !workspace) return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  return map_internal(r2::debug_median_run(static_cast<const float2*>(planes_c64), planes, n, amplitudes, medians,
                                           workspace, workspace_bytes, static_cast<cudaStream_t>(stream)),
                      "rift2_debug_median");
}


// ------------------------------------------------- unfused reference entry points
int32_t rift2_filter_bank(int32_t height, int32_t width, const rift2_bank_params* params, double* transfer,
                          void* stream) {
  r2::BankConsts k;
  int32_t rc = bank_consts(params, k);
  if (rc) return rc;
  if (height < 16 || width < 16) return fail(RIFT2_BAD_ARGUMENT, "filter bank needs width and height >= 16");
  if (!transfer) return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  const double st = params->orientation_spread > 0 ? params->orientation_spread : M_PI / params->n_orient;
  rc = r2::filter_bank_run(height, width, params->n_scales, params->n_orient, params->min_wavelength,
                           params->scale_mult, params->sigma_on_f, st, transfer, static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_filter_bank");
}

int32_t rift2_apply_bank_workspace_size(int32_t height, int32_t width, int32_t n_scales, int32_t n_orient,
                                        size_t* bytes) {
  if (!bytes || n_scales < 1 || n_orient < 1) return fail(RIFT2_BAD_ARGUMENT, "bad apply_bank arguments");
  int32_t rc = check_fields_dims(1, height, width);
  if (rc) return rc;
  *bytes = r2::apply_bank_workspace_bytes(height, width, n_scales, n_orient);
  return RIFT2_OK;
}

int32_t rift2_apply_bank(const float* image, int32_t height, int32_t width, int32_t n_scales, int32_t n_orient,
                         const float* transfer, float* even, float* odd, float* amplitude, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (n_scales < 1 || n_orient < 1) return fail(RIFT2_BAD_ARGUMENT, "bad bank shape");
  int32_t rc = check_fields_dims(1, height, width);
  if (rc) return rc;
  if (!image || !transfer || !even || !odd || !amplitude || !workspace) return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  rc = r2::apply_bank_run(image, height, width, n_scales, n_orient, transfer, even, odd, amplitude, workspace,
                          workspace_bytes, static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_apply_bank");
}

int32_t rift2_pc_moments_workspace_size(int32_t height, int32_t width, const rift2_bank_params* params,
                                        size_t* bytes) {
  r2::BankConsts k;
  int32_t rc = bank_consts(params, k);
  if (rc) return rc;
  if (!bytes || height < 1 || width < 1) return fail(RIFT2_BAD_ARGUMENT, "bad pc_moments arguments");
  *bytes = r2::pc_stack_workspace_bytes(height, width, k.n_scales, k.n_orient);
  return RIFT2_OK;
}

int32_t rift2_pc_moments(const float* even, const float* odd, const float* amplitude, int32_t height,
                         int32_t width, const rift2_bank_params* params, float* a_o, float* pc, float* moment_max,
                         float* moment_min, void* workspace, size_t workspace_bytes, void* stream) {
  r2::BankConsts k;
  int32_t rc = bank_consts(params, k);
  if (rc) return rc;
  if (height < 1 || width < 1 || (long long)height * width > 0x7fffffffLL)
    return fail(RIFT2_BAD_ARGUMENT, "bad dimensions");
  const bool full = pc || moment_max || moment_min;
  if (!amplitude || (full && (!even || !odd || !pc || !moment_max || !moment_min || !workspace)))
    return fail(RIFT2_BAD_ARGUMENT, "NULL buffer");
  rc = r2::pc_stack_run(even, odd, amplitude, height, width, k, a_o, pc, moment_max, moment_min, workspace,
                        workspace_bytes, static_cast<cudaStream_t>(stream));
  return map_internal(rc, "rift2_pc_moments");
}

int32_t rift2_orientation_amplitudes(const double* amplitude, int32_t n_scales, int32_t n_orient, int32_t height,
                                     int32_t width, double* a_o, void* stream) {
  if (!amplitude || !a_o || n_scales < 1 || n_orient < 1 || height < 0 || width < 0)
    return fail(RIFT2_BAD_ARGUMENT, "bad orientation_amplitudes arguments");
  return map_internal(r2::sum_scales_run(amplitude, n_scales, n_orient, height, width, a_o,
                                         static_cast<cudaStream_t>(stream)), "rift2_orientation_amplitudes");
}

int32_t rift2_build_mim(const double* a_o, int32_t n_orient, int32_t height, int32_t width, int32_t* indices,
                        double* max_amplitude, void* stream) {
  if (n_orient < 2) return fail(RIFT2_BAD_ARGUMENT, "need >= 2 stacked channels");
  if (height < 1 || width < 1 || !a_o || !indices) return fail(RIFT2_BAD_ARGUMENT, "bad build_mim arguments");
  return map_internal(r2::build_mim_run(a_o, n_orient, height, width, indices, max_amplitude,
                                        static_cast<cudaStream_t>(stream)), "rift2_build_mim");
}

int32_t rift2_patch_counts(const int32_t* indices, const double* amplitude, int32_t n_patches, int32_t height,
                           int32_t width, int32_t n_orient, int32_t grid, double* hist, double* cells, void* stream) {
  if (n_patches < 0 || height < 1 || width < 1 || n_orient < 1 || !indices)
    return fail(RIFT2_BAD_ARGUMENT, "bad patch arguments");
  if (cells && (grid < 1 || height != width || width % grid != 0))
    return fail(RIFT2_BAD_ARGUMENT, "patch %dx%d does not divide into %dx%d cells", height, width, grid, grid);
  return map_internal(r2::patch_counts_run(indices, amplitude, n_patches, height, width, n_orient, grid, hist, cells,
                                           static_cast<cudaStream_t>(stream)), "rift2_patch_counts");
}

int32_t rift2_remap_indices(int32_t* indices, int64_t count, int32_t n_orient, int32_t pivot, int32_t kind,
                            void* stream) {
  if (count < 0 || (count > 0 && !indices) || n_orient < 1 || (kind != 0 && kind != 1))
    return fail(RIFT2_BAD_ARGUMENT, "bad remap arguments");
  if (pivot < 1 || pivot > n_orient) return fail(RIFT2_BAD_ARGUMENT, "index %d outside [1, %d]", pivot, n_orient);
  return map_internal(r2::remap_run(indices, count, n_orient, pivot, kind, static_cast<cudaStream_t>(stream)),
                      "rift2_remap_indices");
}

int32_t rift2_extract_patch(const int32_t* indices, const double* amplitude, int32_t height, int32_t width,
                            double x, double y, int32_t size, double cos_a, double sin_a, int32_t* out_indices,
                            double* out_amplitude, int32_t* out_of_bounds, void* stream) {
  if (!indices || !out_indices || !out_of_bounds || height < 1 || width < 1 || size < 1)
    return fail(RIFT2_BAD_ARGUMENT, "bad extract_patch arguments");
  if (!std::isfinite(x) || !std::isfinite(y)) return fail(RIFT2_BAD_ARGUMENT, "keypoint is not finite");
  const int integer_kp = (x == std::floor(x) && y == std::floor(y)) ? 1 : 0;
  return map_internal(r2::gather_run(indices, amplitude, height, width, x, y, integer_kp, size, cos_a, sin_a,
                                     out_indices, out_amplitude, out_of_bounds, static_cast<cudaStream_t>(stream)),
                      "rift2_extract_patch");
}
}  // extern "C"
