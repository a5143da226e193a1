// On-device target synthesis for the BASELINE generator.
//
// Each pair's target image is its reference image under a similarity, with
// the BASELINE radiometry.  The warp follows ref: pkg/src/rift2/imaging.py:208-247
// (`warp_rigid`): output pixel p takes the bilinear sample of the source at
// T^-1(p), 0 outside, exactly-on-grid samples along the far edges kept.  It
// is generalised to the 2x3 inverse map of a similarity.  Then:
//   * inversion (v -> 1 - v) when flagged;
//   * gamma (clip to [0, 1], then pow);
//   * multiplicative Gamma(L, 1/L) speckle: the mean of L unit exponentials
//     -log(u), u in (0, 1] drawn from Philox4x32-10 with counter
//     (pixel lo, pixel hi, image, j) and key (seed lo, seed hi);
//   * min-max renormalisation to [0, 1].
// Products and sums are rounded separately (no FMA contraction), in numpy's
// operation order, so the warp and the normalisation match the host
// generator (synth.py) bit for bit; pow / log are the CUDA double versions
// (<= 2 ulp).
//
// Data layout: the sources are float64 [image][H][W] (any image stride).  The
// float64 pre-normalisation values go to the workspace, followed by the
// per-image min / max keys.  The targets are written as float32, optionally
// with a float32 copy of each source, e.g. straight into the [ref, tgt, ...]
// batch layout the pipeline reads.  Bound: HBM, 8 B read + 8 B write + 8 B
// read + 4 (+4) B write per pixel, plus L logs per pixel (issue-bound for
// large L).
#include "common.cuh"
#include "synth.h"

namespace r2 {

namespace {

constexpr int kSynthThreads = 256;

R2_DEV unsigned long long ord_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
R2_DEV double ord_val(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// Philox4x32-10 (Salmon et al., SC'11)
R2_DEV uint4 philox(uint4 c, unsigned k0, unsigned k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// (0, 1] from two words: ((a >> 5) * 2^26 + (b >> 6) + 1) * 2^-53
R2_DEV double u53(unsigned a, unsigned b) {
  const unsigned long long m = (unsigned long long)(a >> 5) * (1ull << 26) + (b >> 6) + 1ull;
  return __dmul_rn((double)m, 1.1102230246251565e-16);
}

// min keys start at all-ones, max keys at zero
__global__ void k_synth_init(unsigned long long* __restrict__ mm, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n) { mm[2 * b] = ~0ull; mm[2 * b + 1] = 0ull; }
}

__global__ void __launch_bounds__(kSynthThreads) k_synth_pre(SynthArgs a, double* __restrict__ work,
                                                             unsigned long long* __restrict__ mm) {
  __shared__ unsigned long long s_lo[kSynthThreads / 32], s_hi[kSynthThreads / 32];
  const int b = blockIdx.y;
  const int H = a.H, W = a.W;
  const size_t n = (size_t)H * W;
  const double* src = a.src + (size_t)b * a.src_stride;
  const double* p = a.params + (size_t)b * kSynthParams;
  const double i00 = p[0], i01 = p[1], i02 = p[2], i10 = p[3], i11 = p[4], i12 = p[5], gamma = p[6];
  const int flags = (int)p[7];
  const int looks = a.looks[b];
  const unsigned image = (unsigned)(a.first_image + b);
  const unsigned k0 = (unsigned)a.seed, k1 = (unsigned)(a.seed >> 32);
  double* out = work + (size_t)b * n;
  float* copy = a.dst_src_copy ? a.dst_src_copy + (size_t)b * a.copy_stride : nullptr;
  unsigned long long lo = ~0ull, hi = 0ull;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i - (size_t)y * W);
    const double xs = (double)x, ys = (double)y;
    // ref: imaging.py:225-246
    const double sx = __dadd_rn(__dadd_rn(__dmul_rn(i00, xs), __dmul_rn(i01, ys)), i02);
    const double sy = __dadd_rn(__dadd_rn(__dmul_rn(i10, xs), __dmul_rn(i11, ys)), i12);
    const double flx = floor(sx), fly = floor(sy);
    const double fx = __dsub_rn(sx, flx), fy = __dsub_rn(sy, fly);
    double v = 0.0;
    if (flx >= 0.0 && flx < (double)(W - 1) && fly >= 0.0 && fly < (double)(H - 1)) {
      const int x0 = (int)flx, y0 = (int)fly;
      const double* r0 = src + (size_t)y0 * W + x0;
      const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);
      v = __dmul_rn(__dmul_rn(r0[0], gx), gy);
      v = __dadd_rn(v, __dmul_rn(__dmul_rn(r0[1], fx), gy));
      v = __dadd_rn(v, __dmul_rn(__dmul_rn(r0[W], gx), fy));
      v = __dadd_rn(v, __dmul_rn(__dmul_rn(r0[W + 1], fx), fy));
    } else if (fx == 0.0 && fy == 0.0 && flx >= 0.0 && flx < (double)W && fly >= 0.0 && fly < (double)H) {
      v = src[(size_t)fly * W + (size_t)flx];
    }
    if (flags & kSynthRadiometric) {
      if (flags & kSynthInverted) v = __dsub_rn(1.0, v);
      v = pow(fmin(fmax(v, 0.0), 1.0), gamma);
      if (looks > 0) {
        double s = 0.0;
        for (int j = 0; 2 * j < looks; ++j) {
          const uint4 r = philox(make_uint4((unsigned)i, (unsigned)((unsigned long long)i >> 32), image, (unsigned)j),
                                 k0, k1);
          s = __dadd_rn(s, -log(u53(r.x, r.y)));
          if (2 * j + 1 < looks) s = __dadd_rn(s, -log(u53(r.z, r.w)));
        }
        v = __dmul_rn(v, __ddiv_rn(s, (double)looks));
      }
      const unsigned long long k = ord_key(v);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
    out[i] = v;
    if (copy) copy[i] = __double2float_rn(src[i]);
  }
  if (!(flags & kSynthRadiometric)) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_lo[w] = lo; s_hi[w] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kSynthThreads / 32; ++k) { lo = s_lo[k] < lo ? s_lo[k] : lo; hi = s_hi[k] > hi ? s_hi[k] : hi; }
    atomicMin(&mm[2 * b], lo);
    atomicMax(&mm[2 * b + 1], hi);
  }
}

__global__ void __launch_bounds__(kSynthThreads) k_synth_norm(SynthArgs a, const double* __restrict__ work,
                                                              const unsigned long long* __restrict__ mm) {
  const int b = blockIdx.y;
  const size_t n = (size_t)a.H * a.W;
  const int flags = (int)a.params[(size_t)b * kSynthParams + 7];
  const double* in = work + (size_t)b * n;
  float* dst = a.dst + (size_t)b * a.dst_stride;
  if (flags & kSynthRadiometric) {
    // (v - min) / max(max - min, 1e-12), numpy's order
    const double mn = ord_val(mm[2 * b]), mx = ord_val(mm[2 * b + 1]);
    const double den = fmax(__dsub_rn(mx, mn), 1e-12);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      dst[i] = __double2float_rn(__ddiv_rn(__dsub_rn(in[i], mn), den));
  } else {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      dst[i] = __double2float_rn(in[i]);
  }
}

// Image 1 of the generator (synth.blob_field): the sum of anisotropic
// Gaussian blobs, one thread per pixel adding the blobs in draw order (the
// host adds them blob by blob in the same order), in numpy's operation
// order without FMA contraction; blob b of image i is blobs[(i * n + b) * 11]
// = cx, cy, sx, sy, cos phi, sin phi, amp, x0, x1, y0, y1 (window [x0, x1) x
// [y0, y1), empty windows skipped).
__global__ void __launch_bounds__(256) k_blobs(const double* __restrict__ blobs, int n_blobs, int H, int W,
                                               double* __restrict__ out) {
  const int img = blockIdx.y;
  const size_t n = (size_t)H * W;
  const double* bl = blobs + (size_t)img * n_blobs * 11;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i % W);
    double acc = 0.0;
    for (int b = 0; b < n_blobs; ++b) {
      const double* q = bl + (size_t)b * 11;
      if (x < (int)q[7] || x >= (int)q[8] || y < (int)q[9] || y >= (int)q[10]) continue;
      const double dx = __dsub_rn((double)x, q[0]), dy = __dsub_rn((double)y, q[1]);
      const double u = __dadd_rn(__dmul_rn(q[4], dx), __dmul_rn(q[5], dy));
      const double v = __dadd_rn(__dmul_rn(-q[5], dx), __dmul_rn(q[4], dy));
      const double a = __ddiv_rn(u, q[2]), c = __ddiv_rn(v, q[3]);
      const double e = exp(__dmul_rn(-0.5, __dadd_rn(__dmul_rn(a, a), __dmul_rn(c, c))));
      acc = __dadd_rn(acc, __dmul_rn(q[6], e));
    }
    out[(size_t)img * n + i] = acc;
  }
}

// Standard normals from Philox4x32-10 (Box-Muller on two 53-bit uniforms),
// counter (pixel pair, image, 0x5eed) and key seed: the device draw of the
// white noise behind the band-limited component.
__global__ void __launch_bounds__(256) k_normals(unsigned long long seed, int first_image, size_t n,
                                                 float* __restrict__ out) {
  const int img = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 r = philox(make_uint4((unsigned)i, (unsigned)(i >> 32), (unsigned)(first_image + img), 0x5eedu),
                           (unsigned)seed, (unsigned)(seed >> 32));
    const double u1 = u53(r.x, r.y), u2 = u53(r.z, r.w);
    const double rad = sqrt(-2.0 * log(u1));
    const double t = 6.283185307179586 * u2;
    float* o = out + (size_t)img * n;
    o[2 * i] = (float)(rad * cos(t));
    if (2 * i + 1 < n) o[2 * i + 1] = (float)(rad * sin(t));
  }
}

}  // namespace

int blobs_run(const double* blobs, int n_images, int n_blobs, int H, int W, double* out, cudaStream_t st) {
  if (n_images <= 0) return 0;
  const size_t n = (size_t)H * W;
  const unsigned gx = (unsigned)((n + 255) / 256 < 2048 ? (n + 255) / 256 : 2048);
  k_blobs<<<dim3(gx, n_images), 256, 0, st>>>(blobs, n_blobs, H, W, out);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

int normals_run(unsigned long long seed, int first_image, int n_images, size_t n, float* out, cudaStream_t st) {
  if (n_images <= 0) return 0;
  const unsigned gx = (unsigned)((n / 2 + 255) / 256 < 2048 ? (n / 2 + 255) / 256 : 2048);
  k_normals<<<dim3(gx, n_images), 256, 0, st>>>(seed, first_image, n, out);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

size_t synth_workspace_bytes(int n_images, int H, int W) {
  return (((size_t)n_images * H * W * sizeof(double) + 255) & ~(size_t)255) + (size_t)n_images * 16;
}

int synth_run(const SynthArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (a.n_images == 0) return 0;
  if (ws_bytes < synth_workspace_bytes(a.n_images, a.H, a.W)) return 1;
  double* work = static_cast<double*>(ws);
  auto* mm = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) +
                                                   (((size_t)a.n_images * a.H * a.W * sizeof(double) + 255) &
                                                    ~(size_t)255));
  k_synth_init<<<(a.n_images + 127) / 128, 128, 0, st>>>(mm, a.n_images);
  const size_t n = (size_t)a.H * a.W;
  const size_t want = (n + kSynthThreads * 4 - 1) / (kSynthThreads * 4);
  const int gx = (int)(want < 1184 ? want : 1184);
  const dim3 grid(gx, a.n_images);
  k_synth_pre<<<grid, kSynthThreads, 0, st>>>(a, work, mm);
  k_synth_norm<<<grid, kSynthThreads, 0, st>>>(a, work, mm);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2
