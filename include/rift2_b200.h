/*
 * rift2_b200 -- C ABI of the B200 RIFT2 feature pipeline.
 *
 * Plain pointers and sizes only.  Every device pointer is caller-owned
 * (the library allocates nothing per call; the only cached state is the
 * per-(device, length) FFT twiddle tables and per-angle descriptor gather
 * tables).  All work is enqueued on `stream` (a cudaStream_t, NULL = legacy
 * default stream) and the calls are reentrant across streams and devices.
 *
 * Status codes (mapped onto the reference's exception types by the Python
 * layer, ref: pkg/src/rift2/errors.py:4-21):
 *   0 RIFT2_OK
 *   1 RIFT2_BAD_ARGUMENT   -> ParameterError (ref preconditions, e.g.
 *                             loggabor.py:57-67, detector.py:96-99,146-149,
 *                             matcher.py:105-106)
 *   2 RIFT2_UNSUPPORTED    -> ParameterError (size/parameter outside the
 *                             kernels' range, e.g. an FFT length with a
 *                             prime factor other than 2, 3, 5)
 *   3 RIFT2_CUDA_ERROR     -> RiftError (text from rift2_last_error())
 *   4 RIFT2_CAPACITY       -> RiftError (an output buffer was too small)
 */
#ifndef RIFT2_B200_H
#define RIFT2_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RIFT2_OK 0
#define RIFT2_BAD_ARGUMENT 1
#define RIFT2_UNSUPPORTED 2
#define RIFT2_CUDA_ERROR 3
#define RIFT2_CAPACITY 4

/* Filter-bank parameters; mirrors ref: pkg/src/rift2/loggabor.py:35-80
 * (BankParams) and config.py:73-84.  orientation_spread <= 0 selects the
 * reference default pi / n_orient. */
typedef struct rift2_bank_params {
  int32_t n_scales;
  int32_t n_orient;
  double min_wavelength;
  double scale_mult;
  double sigma_on_f;
  double orientation_spread;
  double noise_k;
  double spread_cutoff;
  double spread_gain;
} rift2_bank_params;

/* Library version (major*10000 + minor*100 + patch). */
int32_t rift2_version(void);

/* Human-readable text of the last non-zero status on this thread. */
const char* rift2_last_error(void);

/* ---- stage 1: phase-congruency moments + maximum index map -------------
 * Replaces ref: pkg/src/rift2/pipeline.py:42-50 (compute_fields), i.e.
 * loggabor.py:131-251 (build_filter_bank / apply_bank /
 * phase_congruency_moments / orientation_amplitudes) and mim.py:43-55
 * (build_mim), for a batch of `batch` images.
 *   images       [batch][height][width] float32, device
 *   moment_max   [batch][height][width] float32 out        (PCField.moment_max)
 *   moment_min   [batch][height][width] float32 out        (PCField.moment_min)
 *   mim          [batch][height][width] uint8 out, 1-based (IndexMap.indices)
 *   a_o, pc_o    [batch][n_orient][height][width] float32 out, may be NULL
 *   a_max        [batch][height][width] float32 out, may be NULL
 *   moment_range [batch][2][2] uint64 out, may be NULL: per image the (min,
 *                max) of moment_min, then of moment_max, as order-preserving
 *                keys of the float64 values (bit pattern | 2^63), reduced in
 *                the PC pass; rift2_detect_* reads them instead of
 *                re-reading the maps for the normalisation
 * height, width >= 16 with prime factors in {2, 3, 5}; n_scales <= 8,
 * n_orient <= 16. */
int32_t rift2_fields_workspace_size(int32_t batch, int32_t height, int32_t width,
                                    const rift2_bank_params* params, size_t* bytes);
int32_t rift2_fields(const float* images, int32_t batch, int32_t height, int32_t width,
                     const rift2_bank_params* params, float* moment_max, float* moment_min,
                     uint8_t* mim, float* a_o, float* pc_o, float* a_max, uint64_t* moment_range,
                     void* workspace, size_t workspace_bytes, void* stream);

/* ---- stage 2: FAST keypoints on both moment maps -------------------------
 * Replaces ref: pkg/src/rift2/detector.py:140-155 (detect_keypoints) for a
 * batch; with single_map != 0 it replaces detector.py:87-113 (detect_fast)
 * on `maps` alone (kind 0).
 *   min_maps     [batch][height][width] moment_min (corners, kind 0)
 *   max_maps     [batch][height][width] moment_max (edges, kind 1; unused
 *                with single_map); float32 (rift2_detect_f32) or float64
 *                (rift2_detect_f64), finite (the Python layer checks,
 *                ref: detector.py:96-97)
 *   kp_x, kp_y   [batch][max_points] int32 out
 *   kp_response  [batch][max_points] float64 out
 *   kp_kind      [batch][max_points] uint8 out (0 corner, 1 edge)
 *   moment_range rift2_fields' per-image map extrema, or NULL (then the
 *                detector reduces the maps itself); two-map mode only
 *   kp_count     [batch] int32 out
 * Keypoints are ordered by (-response, y, x), corner before edge on ties. */
int32_t rift2_detect_workspace_size(int32_t batch, int32_t height, int32_t width, int32_t max_points,
                                    size_t* bytes);
int32_t rift2_detect_f32(const float* min_maps, const float* max_maps, int32_t batch, int32_t height,
                         int32_t width, double threshold, int32_t max_points, int32_t border_margin, int32_t single_map,
                         int32_t* kp_x, int32_t* kp_y, double* kp_response, uint8_t* kp_kind,
                         int32_t* kp_count, const uint64_t* moment_range, void* workspace, size_t workspace_bytes,
                         void* stream);
int32_t rift2_detect_f64(const double* min_maps, const double* max_maps, int32_t batch, int32_t height,
                         int32_t width, double threshold, int32_t max_points, int32_t border_margin, int32_t single_map,
                         int32_t* kp_x, int32_t* kp_y, double* kp_response, uint8_t* kp_kind,
                         int32_t* kp_count, const uint64_t* moment_range, void* workspace, size_t workspace_bytes,
                         void* stream);

/* ---- stage 3: RIFT2 dominant-index descriptors ---------------------------
 * Replaces ref: pkg/src/rift2/descriptor.py:179-216 (describe_rift2),
 * :219-236 (describe_ring, mode 1) and :239-254 (describe_plain, mode 0).
 *   mim          [batch][height][width] uint8 (1..n_orient)
 *   kp_x, kp_y   [batch][kp_stride] int32, kp_count [batch] int32
 *   desc_counts  [batch][desc_capacity][desc_stride] float16 out: integer
 *                cell-histogram counts (zero padded to desc_stride >= dim)
 *   desc_sqnorm  [batch][desc_capacity] int32 out: sum of squared counts
 *   desc_kp      [batch][desc_capacity] int32 out: keypoint id
 *   desc_variant [batch][desc_capacity] uint8 out: dominant index / layer
 *   desc_count   [batch] int32 out, desc_skipped [batch] int32 out
 * Descriptors are ordered by keypoint, then [peak, runner-up] (rift2) or
 * layer 1..n (ring).  mode: 0 plain, 1 ring, 2 rift2, 3 the pipeline's ring
 * mode (ref: pipeline.py:53-64): even blocks (reference side) ring, odd
 * blocks (target side) plain.
 * desc_capacity must be >= rows-per-keypoint (1 plain, n_orient ring and
 * mode 3, 2 rift2) x kp_stride, else RIFT2_CAPACITY; kp_count values above
 * kp_stride are clamped to it. */
int32_t rift2_describe_workspace_size(int32_t batch, int32_t kp_stride, int32_t grid, int32_t n_orient,
                                      size_t* bytes);
/* The larger workspace that also holds a shift-byte copy of the index maps
 * (one pass before the per-keypoint kernel, so it stages them with no
 * in-place transform) and the dense 16 x 16 cell sums of every pixel (8
 * bytes per pixel: the axis-aligned patch of a keypoint is then 36 loads
 * instead of 9,216 counted pixels; 16-pixel cells and n_orient <= 6): a
 * workspace of this size makes rift2_describe faster at the same results;
 * the smaller size above stays valid, and a size in between gets the
 * shift-byte copy only. */
int32_t rift2_describe_workspace_size_hw(int32_t batch, int32_t height, int32_t width, int32_t kp_stride,
                                         int32_t grid, int32_t n_orient, size_t* bytes);
int32_t rift2_describe(const uint8_t* mim, int32_t batch, int32_t height, int32_t width, int32_t n_orient,
                       const int32_t* kp_x, const int32_t* kp_y, const int32_t* kp_count, int32_t kp_stride,
                       int32_t patch_size, int32_t grid, double dominant_ratio, int32_t rotate_patch,
                       int32_t mode, void* desc_counts, int32_t desc_stride, int32_t desc_capacity,
                       int32_t* desc_sqnorm, int32_t* desc_kp, uint8_t* desc_variant, int32_t* desc_count,
                       int32_t* desc_skipped, void* workspace, size_t workspace_bytes, void* stream);
/* As rift2_describe with float64 keypoint coordinates: keypoints need not
 * be integral (ref: descriptor.py:105-125 -- axis crop at
 * floor(x + 1 - patch/2), rotated samples at floor(x + ux + 0.5) from the
 * reference's continuous float64 offsets; integral coordinates take the
 * reference's integer-table path and give rift2_describe's result).  Any
 * n_orient <= 16 and any cell size (patch_size divisible by grid) are
 * accepted by both entry points; the BASELINE shape (6 orientations,
 * 16-pixel cells, integer keypoints) runs on the staged fast kernel, the
 * rest on a generic kernel with the same outputs. */
int32_t rift2_describe_f64(const uint8_t* mim, int32_t batch, int32_t height, int32_t width, int32_t n_orient,
                           const double* kp_x, const double* kp_y, const int32_t* kp_count, int32_t kp_stride,
                           int32_t patch_size, int32_t grid, double dominant_ratio, int32_t rotate_patch,
                           int32_t mode, void* desc_counts, int32_t desc_stride, int32_t desc_capacity,
                           int32_t* desc_sqnorm, int32_t* desc_kp, uint8_t* desc_variant, int32_t* desc_count,
                           int32_t* desc_skipped, void* workspace, size_t workspace_bytes, void* stream);

/* ---- stage 4: brute-force nearest-neighbour matching ---------------------
 * Replaces ref: pkg/src/rift2/matcher.py:102-148 (match_nn) for `n_pairs`
 * independent (reference, target) descriptor sets.  Descriptor blocks use
 * the stage-3 layout; pair p uses reference block ref_block[p] and target
 * block tgt_block[p] of the descriptor arrays (device int32 arrays);
 * n_blocks is the number of blocks the descriptor arrays hold.  desc_stride
 * must be 224 or 256 (the tensor-core tiles cover K <= 256).
 *   out_ref, out_tgt [n_pairs][tgt_kp_capacity] int32 out (keypoint ids)
 *   out_dist         [n_pairs][tgt_kp_capacity] float64 out
 *   out_count        [n_pairs] int32 out (= number of target keypoints
 *                    with a descriptor, at most tgt_kp_capacity; 0 when the
 *                    pair's reference set is empty -- the dataclass API
 *                    raises ParameterError there, ref: matcher.py:105-106)
 * Pairs are sorted by (dist, ref, tgt) as the reference returns them.
 * Ranking is exact: candidates are compared on integer dot products and
 * squared norms, ties resolve to the smallest reference keypoint id. */
int32_t rift2_match_workspace_size(int32_t n_pairs, int32_t desc_capacity, int32_t tgt_kp_capacity,
                                   size_t* bytes);
int32_t rift2_match(const void* desc_counts, const int32_t* desc_sqnorm, const int32_t* desc_kp,
                    const int32_t* desc_count, int32_t n_blocks, int32_t desc_stride, int32_t desc_capacity,
                    int32_t dim, int32_t n_pairs, const int32_t* ref_block, const int32_t* tgt_block,
                    int32_t tgt_kp_capacity, int32_t* out_ref, int32_t* out_tgt, double* out_dist,
                    int32_t* out_count, void* workspace, size_t workspace_bytes, void* stream);

/* ---- stage 4, row-sharded across processes ------
 * For one huge pair split over G GPUs: rank r matches ALL target
 * descriptors against its slice of the reference descriptors
 * (rift2_match_partial), the G partial arrays are all-gathered, and every
 * rank (or one) combines them exactly (rift2_match_finish) -- the same
 * result as rift2_match on the whole reference set, bit for bit.
 *
 * rift2_match_partial: arguments as rift2_match; out_parts
 *   [n_pairs][desc_capacity] records, one per target descriptor row: the
 *   exact best reference candidate of this call (ref_kp = -1 when none).
 *   Reference keypoint ids are taken from desc_kp, so a slice must carry
 *   global keypoint ids.  No workspace.
 * rift2_match_finish: parts [n_parts][n_pairs][desc_capacity] (the gathered
 *   partial arrays, any order of ranks); the target block must hold the
 *   FULL target set, the reference block may hold only this rank's slice
 *   (global keypoint ids, desc_capacity > every keypoint id): the winner of
 *   every target keypoint is exact and identical on all ranks, its float64
 *   distance is computed where the winner's reference rows are present and
 *   reported as +inf elsewhere (the rank owning the row supplies it, so
 *   reference rows never cross ranks); outputs and workspace as
 *   rift2_match (rift2_match_workspace_size). */
typedef struct rift2_match_part {
  int32_t dot;          /* integer dot product of the count vectors */
  int32_t ref_sqnorm;   /* sum of squared reference counts */
  int32_t ref_kp;       /* reference keypoint id, -1 = none */
  float score;          /* dot / |ref| (screening only) */
} rift2_match_part;

int32_t rift2_match_partial(const void* desc_counts, const int32_t* desc_sqnorm, const int32_t* desc_kp,
                            const int32_t* desc_count, int32_t n_blocks, int32_t desc_stride, int32_t desc_capacity,
                            int32_t dim, int32_t n_pairs, const int32_t* ref_block, const int32_t* tgt_block,
                            rift2_match_part* out_parts, void* stream);
int32_t rift2_match_finish(const rift2_match_part* parts, int32_t n_parts, const void* desc_counts,
                           const int32_t* desc_sqnorm, const int32_t* desc_kp, const int32_t* desc_count,
                           int32_t n_blocks, int32_t desc_stride, int32_t desc_capacity, int32_t dim, int32_t n_pairs,
                           const int32_t* ref_block, const int32_t* tgt_block, int32_t tgt_kp_capacity,
                           int32_t* out_ref, int32_t* out_tgt, double* out_dist, int32_t* out_count, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Generic variant of stage 4 for arbitrary float64 descriptor vectors (not
 * integer histograms), e.g. unit vectors built by the caller: the
 * reference's own key |r|^2 - 2 r.t in float64 (ref: matcher.py:125-135).
 * Rows must be grouped by keypoint id (stable order, ref: matcher.py:67-79).
 *   ref_vec [n_ref][dim], tgt_vec [n_tgt][dim] float64 device
 *   out_* [n_tgt] (one entry per target keypoint), sorted (dist, ref, tgt). */
int32_t rift2_match_vectors_workspace_size(int32_t n_ref, int32_t n_tgt, size_t* bytes);
int32_t rift2_match_vectors(const double* ref_vec, const int32_t* ref_kp, int32_t n_ref, const double* tgt_vec,
                            const int32_t* tgt_kp, int32_t n_tgt, int32_t dim, int32_t* out_ref, int32_t* out_tgt,
                            double* out_dist, int32_t* out_count, void* workspace, size_t workspace_bytes,
                            void* stream);

/* ---- ground-truth evaluation of match sets ----------
 * Replaces ref: pkg/src/rift2/evalbench.py:63-96 (evaluate) for a batch of
 * pairs laid out like rift2_detect / rift2_match outputs: keypoints
 * [images][kp_stride] with kp_count[images]; pair p compares image
 * ref_img[p] against tgt_img[p] with match rows match_ref / match_tgt
 * [n_pairs][match_stride] (match_count[p] live rows) and the 2x3 transform
 * gt[p] = (R00, R01, R10, R11, t0, t1) mapping reference to target points.
 * Per pair: number of matches with residual < residual_threshold, RMSE over
 * them (clamped to rmse_cap, +inf with none), success = n_correct >=
 * success_min_matches, and out_bad = 1 if a match index does not resolve
 * (the reference raises IntegrityError there). */
int32_t rift2_evaluate(const int32_t* kp_x, const int32_t* kp_y, const int32_t* kp_count, int32_t kp_stride,
                       const int32_t* ref_img, const int32_t* tgt_img, const int32_t* match_ref,
                       const int32_t* match_tgt, const int32_t* match_count, int32_t match_stride, int32_t n_pairs,
                       const double* gt, double residual_threshold, double rmse_cap, int32_t success_min_matches,
                       int32_t* out_n_correct, double* out_rmse, uint8_t* out_success, int32_t* out_bad,
                       void* stream);

/* ---- on-device target synthesis ----------------------
 * The BASELINE generator's target side on the GPU.  The reference ships no
 * generator; the warp keeps ref: pkg/src/rift2/imaging.py:208-247
 * (`warp_rigid`) semantics, generalised to any 2x3 map.  For image i:
 *   src  + i*src_image_stride : float64 [height][width] source (device)
 *   params[i][8] (device float64): the target->source map i00 i01 i02 i10
 *     i11 i12 (source x = i00 x + i01 y + i02, ...), gamma, flags (bit 0
 *     inverted, bit 1 radiometric: inversion, gamma, speckle, renormalise)
 *   looks[i] (device int32): Gamma(L, 1/L) speckle looks, 0 = none; the
 *     draws are Philox4x32-10 with counter (pixel, first_image + i, j) and
 *     key seed
 *   dst + i*dst_image_stride : float32 target (device)
 *   dst_src_copy + i*copy_image_stride : optional float32 copy of the source
 *     (NULL = none), e.g. the reference slot of a [ref, tgt, ...] batch. */
int32_t rift2_synth_workspace_size(int32_t n_images, int32_t height, int32_t width, size_t* bytes);
/* Image 1 of the generator on the device:
 * rift2_synth_blobs: out [n_images][height][width] float64 = the sum of
 *   n_blobs anisotropic Gaussian blobs per image, blobs [n_images][n_blobs]
 *   [11] = cx, cy, sx, sy, cos phi, sin phi, amp, x0, x1, y0, y1 (the
 *   blob's window [x0, x1) x [y0, y1)), added in order in float64;
 * rift2_synth_normals: out [n_images][n] float32 standard normals
 *   (Philox4x32-10, counter (pixel pair, first_image + i, 0x5eed), key
 *   seed; Box-Muller) -- the white noise of the band-limited component,
 *   which rift2_apply_bank with a 0/1 radial mask then filters. */
int32_t rift2_synth_blobs(const double* blobs, int32_t n_images, int32_t n_blobs, int32_t height, int32_t width,
                          double* out, void* stream);
int32_t rift2_synth_normals(uint64_t seed, int32_t first_image, int32_t n_images, int64_t n, float* out,
                            void* stream);
int32_t rift2_synth_targets(const double* src, int64_t src_image_stride, int32_t n_images, int32_t height,
                            int32_t width, const double* params, const int32_t* looks, uint64_t seed,
                            int32_t first_image, float* dst, int64_t dst_image_stride, float* dst_src_copy,
                            int64_t copy_image_stride, void* workspace, size_t workspace_bytes, void* stream);

/* ---- unfused reference entry points ----------------------------------------
 * The reference's step-by-step API for callers that use the stages one at a
 * time (the fused rift2_fields / rift2_describe are the pipeline path).
 *
 * rift2_filter_bank: ref loggabor.py:131-159 (build_filter_bank): transfer
 *   [n_scales][n_orient][height][width] float64 (device), same formulas in
 *   float64; height, width >= 16.
 * rift2_apply_bank: ref loggabor.py:162-185 (apply_bank) of a GIVEN bank:
 *   image [height][width] float32, transfer [S][O][height][width] float32
 *   (device) -> even, odd, amplitude [S][O][height][width] float32 (fp32
 *   FFTs; FFT lengths with factors 2, 3, 5).
 * rift2_pc_moments: ref loggabor.py:188-251 (orientation_amplitudes,
 *   phase_congruency_moments) from a response stack (float32 device planes
 *   as rift2_apply_bank writes them): a_o, pc [O][height][width], moment_max,
 *   moment_min [height][width] float32; pc / moment maps may all be NULL
 *   (then only a_o, and no workspace is used).  The noise floor uses the
 *   exact median of each scale-0 amplitude plane.
 * rift2_orientation_amplitudes: ref loggabor.py:188-190: amplitude
 *   [S][O][height][width] float64 -> a_o [O][height][width] float64 (sum
 *   over scales in scale order).
 * rift2_build_mim: ref mim.py:43-55 (build_mim): a_o [O][height][width]
 *   float64 -> indices int32 (1-based first argmax), max_amplitude float64
 *   (nullable).
 * rift2_patch_counts: ref mim.py:58-66 (patch_histogram) and
 *   descriptor.py:145-164 (encode, before normalisation), for n patches:
 *   indices [n][height][width] int32 (values 1..n_orient count, 0 is
 *   ignored), amplitude (same shape, float64, NULL = unweighted counts) ->
 *   hist [n][n_orient] and/or cells [n][grid*grid*n_orient] float64 (cells
 *   need square patches divisible into grid x grid cells).
 * rift2_remap_indices: ref mim.py:117-136, in place on count int32 values:
 *   kind 0 recode (pivot = dominant index), kind 1 cyclic_shift (pivot =
 *   initial layer).
 * rift2_extract_patch: ref descriptor.py:85-125 for a non-zero angle:
 *   indices [height][width] int32 (+ optional float64 amplitudes) ->
 *   out_indices [size][size] (+ out_amplitude, NULL to skip); cos_a / sin_a
 *   are the snapped cosine and sine; *out_of_bounds (device int32) is set
 *   when any sample leaves the map (the reference returns None). */
int32_t rift2_filter_bank(int32_t height, int32_t width, const rift2_bank_params* params, double* transfer,
                          void* stream);
int32_t rift2_apply_bank_workspace_size(int32_t height, int32_t width, int32_t n_scales, int32_t n_orient,
                                        size_t* bytes);
int32_t rift2_apply_bank(const float* image, int32_t height, int32_t width, int32_t n_scales, int32_t n_orient,
                         const float* transfer, float* even, float* odd, float* amplitude, void* workspace,
                         size_t workspace_bytes, void* stream);
int32_t rift2_pc_moments_workspace_size(int32_t height, int32_t width, const rift2_bank_params* params,
                                        size_t* bytes);
int32_t rift2_pc_moments(const float* even, const float* odd, const float* amplitude, int32_t height,
                         int32_t width, const rift2_bank_params* params, float* a_o, float* pc, float* moment_max,
                         float* moment_min, void* workspace, size_t workspace_bytes, void* stream);
int32_t rift2_orientation_amplitudes(const double* amplitude, int32_t n_scales, int32_t n_orient, int32_t height,
                                     int32_t width, double* a_o, void* stream);
int32_t rift2_build_mim(const double* a_o, int32_t n_orient, int32_t height, int32_t width, int32_t* indices,
                        double* max_amplitude, void* stream);
int32_t rift2_patch_counts(const int32_t* indices, const double* amplitude, int32_t n_patches, int32_t height,
                           int32_t width, int32_t n_orient, int32_t grid, double* hist, double* cells, void* stream);
int32_t rift2_remap_indices(int32_t* indices, int64_t count, int32_t n_orient, int32_t pivot, int32_t kind,
                            void* stream);
int32_t rift2_extract_patch(const int32_t* indices, const double* amplitude, int32_t height, int32_t width,
                            double x, double y, int32_t size, double cos_a, double sin_a, int32_t* out_indices,
                            double* out_amplitude, int32_t* out_of_bounds, void* stream);

/* ---- diagnostics ----------------------------------------------------------
 * The filter bank's exact-median stage (the Rayleigh noise estimate, ref:
 * loggabor.py:222, np.median) on caller-given complex64 planes
 * [planes][n]: amplitudes[i] = |z_i| as the bank computes it, medians[p] =
 * the exact median of plane p's amplitudes (mean of the two middle order
 * statistics for even n).  For tests; not on the pipeline path. */
int32_t rift2_debug_median_workspace_size(int32_t planes, int32_t n, size_t* bytes);
int32_t rift2_debug_median(const void* planes_c64, int32_t planes, int32_t n, float* amplitudes, float* medians,
                           void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RIFT2_B200_H */
