// Log-Gabor phase-congruency filter bank, moment maps and maximum index map.
//
// Replaces ref: loggabor.py:122-251 (build_filter_bank, apply_bank,
// orientation_amplitudes, phase_congruency_moments) and mim.py:43-55
// (build_mim) with a two-pass 2-D FFT whose inter-pass planes are the only
// per-filter HBM traffic:
//
//   K1 rows_fwd   real rows -> half spectrum rows (two rows per complex FFT)
//   K2 cols       column FFT once per column, then for each of the S*O filters
//                 multiply by the analytically generated transfer function and
//                 inverse-FFT the column (mirror columns from Hermitian symmetry)
//   K3a rows_amp0 inverse row FFT of the S=0 planes -> |response| + histogram
//   K4  median    exact np.median of each scale-0 amplitude plane (radix select)
//   K3b rows_pc   inverse row FFTs of all planes, fused phase congruency,
//                 moments, orientation amplitude sums and MIM argmax.
//
// Layouts (all row-major, batch-major):
//   image  [B][H][W] f32          P  [B][H][Wh] c64 (Wh = W/2+1)
//   Q      [B][S*O][H][W] c64     amp0 [B][O][H*W] f32
//   outputs M, m [B][H][W] f32, MIM [B][H][W] u8, optional a_o/pc [B][O][H][W], amax [B][H][W]
#include "fft.cuh"
#include "fields.h"

namespace r2 {

constexpr int kThreads = 256;
constexpr int kHistBins = 4096;   // float bits >> 19 of a non-negative float
constexpr int kMaxS = 8;
constexpr int kMaxO = 16;

struct FieldsConst {
  int B, H, W, Wh, S, O;
  float log_lambda[kMaxS];     // ln(lambda_s) = -ln(f0_s)
  float inv_den_r;             // 1 / (2 ln(sigma_on_f)^2)
  float inv_den_a;             // 1 / (2 sigma_theta^2)
  float ang[kMaxO], cos_a[kMaxO], sin_a[kMaxO];
  float spread_cutoff, spread_gain, inv_sm1;
  float lp_lncut;              // ln(0.45)
  float inv_hw;
  double thr_factor;           // T = median * thr_factor
  const float2* tw_w;          // W_W^j
  const float2* tw_h;          // W_H^j
  GenericPlan plan_w, plan_h;
};

// numpy.fft.fftfreq(n)[k]
R2_DEV float fftfreq(int k, int n) { return (float)(k < (n + 1) / 2 ? k : k - n) / (float)n; }

// ------------------------------------------------------------------ K1 ---
// Two real rows y0, y1 as one complex FFT z = r0 + i r1, then split:
// X0[k] = (Z[k] + conj Z[-k]) / 2, X1[k] = (Z[k] - conj Z[-k]) / (2i).
template <int G>
__global__ void __launch_bounds__(kThreads) k_rows_fwd(const float* __restrict__ img, float2* __restrict__ P,
                                                       const __grid_constant__ FieldsConst c) {
  extern __shared__ float2 sm[];
  const int W = c.W, H = c.H, Wh = c.Wh;
  const int b = blockIdx.y;
  const float* im = img + (size_t)b * H * W;
  float2* Pb = P + (size_t)b * H * Wh;
  if constexpr (G > 0) {
    constexpr int N = 32 * G;
    constexpr int NG = kThreads / G;
    const int g = threadIdx.x / G, t = threadIdx.x % G;
    float2* buf = sm + g * padded_len(N);
    const int y0 = 2 * (blockIdx.x * NG + g), y1 = y0 + 1;
    const bool v0 = y0 < H, v1 = y1 < H;
    float2 v[32];
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      const int x = t + G * m;
      v[m] = make_float2(v0 ? __ldg(&im[(size_t)y0 * W + x]) : 0.f, v1 ? __ldg(&im[(size_t)y1 * W + x]) : 0.f);
    }
    SyncWarp sw;
    SyncNamed sn{1 + g, G};
    if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_w, t, sw);
    else fft_fast<G>(v, buf, c.tw_w, t, sn);
#pragma unroll
    for (int m = 0; m < 32; ++m) buf[pad32(t + G * m)] = v[m];
    if constexpr (G <= 32) sw(); else sn();
    for (int k = t; k < Wh; k += G) {
      const float2 zk = buf[pad32(k)];
      const float2 zm = cconj(buf[pad32(k == 0 ? 0 : N - k)]);
      if (v0) Pb[(size_t)y0 * Wh + k] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y + zm.y));
      if (v1) Pb[(size_t)y1 * Wh + k] = make_float2(0.5f * (zk.y - zm.y), -0.5f * (zk.x - zm.x));
    }
  } else {
    float2* buf = sm;
    float2* scr = sm + padded_len(W);
    const int y0 = 2 * blockIdx.x, y1 = y0 + 1;
    const bool v1 = y1 < H;
    for (int x = threadIdx.x; x < W; x += blockDim.x)
      buf[pad32(x)] = make_float2(im[(size_t)y0 * W + x], v1 ? im[(size_t)y1 * W + x] : 0.f);
    __syncthreads();
    fft_generic(buf, scr, W, c.plan_w, c.tw_w, threadIdx.x, blockDim.x);
    for (int k = threadIdx.x; k < Wh; k += blockDim.x) {
      const float2 zk = buf[pad32(k)];
      const float2 zm = cconj(buf[pad32(k == 0 ? 0 : W - k)]);
      Pb[(size_t)y0 * Wh + k] = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y + zm.y));
      if (v1) Pb[(size_t)y1 * Wh + k] = make_float2(0.5f * (zk.y - zm.y), -0.5f * (zk.x - zm.x));
    }
  }
}

// ------------------------------------------------------------------ K2 ---
// Transfer function of filter (s, o) at a spectrum sample (ref: loggabor.py:131-159):
//   lowpass(r) * exp(-ln(r/f0)^2 / (2 ln(sigma)^2)) * exp(-dtheta^2 / (2 sigma_theta^2)),
// folded into one exp; geo = (ln r, lowpass/(H*W) (0 at DC), theta, theta_mirror).
R2_DEV float transfer(const FieldsConst& c, float4 geo, bool mirror, int s, int o) {
  const float dr = geo.x + c.log_lambda[s];
  float d = (mirror ? geo.w : geo.z) - c.ang[o];
  if (d > 3.14159265358979f) d -= 6.28318530717959f;
  if (d < -3.14159265358979f) d += 6.28318530717959f;
  return geo.y * __expf(-(dr * dr * c.inv_den_r + d * d * c.inv_den_a));
}

R2_DEV float4 geometry(const FieldsConst& c, int ky, int kx) {
  const float fy = fftfreq(ky, c.H);
  const float fx = fftfreq(kx, c.W);
  const float fxm = fftfreq(kx == 0 ? 0 : c.W - kx, c.W);
  const float r2 = fx * fx + fy * fy;
  float4 g;
  if (ky == 0 && kx == 0) {
    g = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    const float lnr = 0.5f * logf(r2);
    // 1 / (1 + (r / 0.45)^30)
    const float lp = 1.f / (1.f + expf(30.f * (lnr - c.lp_lncut)));
    g = make_float4(lnr, lp * c.inv_hw, atan2f(fy, fx), atan2f(fy, fxm));
  }
  return g;
}

template <int G>
__global__ void __launch_bounds__(kThreads) k_cols(const float2* __restrict__ P, float2* __restrict__ Q,
                                                   const __grid_constant__ FieldsConst c) {
  extern __shared__ float2 sm[];
  const int H = c.H, W = c.W, Wh = c.Wh, F = c.S * c.O;
  const int b = blockIdx.y;
  const float2* Pb = P + (size_t)b * H * Wh;
  if constexpr (G > 0) {
    constexpr int N = 32 * G;        // == H
    constexpr int NG = kThreads / G;
    constexpr int CG = NG / 2;       // direct columns per CTA (plus mirrors)
    constexpr int PL = padded_len(N);
    float2* S = sm;                                        // [CG][PL]
    float4* geo = reinterpret_cast<float4*>(sm + CG * PL); // [CG][N]
    float2* bufs = sm + CG * PL + 2 * CG * N;              // [NG][PL]
    const int g = threadIdx.x / G, t = threadIdx.x % G;
    float2* buf = bufs + g * PL;
    const int kx0 = blockIdx.x * CG;
    SyncWarp sw;
    SyncNamed sn{1 + g, G};
    auto gsync = [&]() { if constexpr (G <= 32) sw(); else sn(); };
    float2 v[32];
    // 1. forward column FFTs of the half spectrum
    if (g < CG) {
      const int kx = kx0 + g;
      const bool ok = kx < Wh;
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = ok ? Pb[(size_t)(t + G * m) * Wh + kx] : make_float2(0.f, 0.f);
      if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_h, t, sw); else fft_fast<G>(v, buf, c.tw_h, t, sn);
#pragma unroll
      for (int m = 0; m < 32; ++m) S[g * PL + pad32(t + G * m)] = v[m];
    }
    // 2. spectrum geometry of the CG columns (shared with their mirrors)
    for (int i = threadIdx.x; i < CG * N; i += kThreads) {
      const int cc = i / N, ky = i % N;
      geo[i] = geometry(c, ky, min(kx0 + cc, Wh - 1));
    }
    __syncthreads();
    // 3. per filter: multiply + inverse column FFT, then coalesced row-segment stores
    const int cc = g % CG, mir = g / CG;
    const int kx = kx0 + cc;
    const bool valid = kx < Wh && (mir == 0 || (kx != 0 && 2 * kx != W));
    for (int f = 0; f < F; ++f) {
      const int s = f / c.O, o = f % c.O;
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const int ky = t + G * m;
        float2 sv;
        if (mir) sv = cconj(S[cc * PL + pad32(ky == 0 ? 0 : N - ky)]);
        else sv = S[cc * PL + pad32(ky)];
        const float gval = valid ? transfer(c, geo[cc * N + ky], mir, s, o) : 0.f;
        v[m] = make_float2(sv.x * gval, -sv.y * gval);   // conj for the inverse
      }
      if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_h, t, sw); else fft_fast<G>(v, buf, c.tw_h, t, sn);
      gsync();
#pragma unroll
      for (int m = 0; m < 32; ++m) buf[pad32(t + G * m)] = cconj(v[m]);
      __syncthreads();
      float2* Qf = Q + ((size_t)b * F + f) * H * W;
      for (int i = threadIdx.x; i < 2 * CG * N; i += kThreads) {
        const int mm = i / (CG * N), rem = i % (CG * N);
        const int y = rem / CG, col = rem % CG;
        const int kxc = kx0 + col;
        const bool ok = kxc < Wh && (mm == 0 || (kxc != 0 && 2 * kxc != W));
        if (ok) {
          const int xo = mm ? W - kxc : kxc;
          Qf[(size_t)y * W + xo] = bufs[(mm * CG + col) * PL + pad32(y)];
        }
      }
      __syncthreads();
    }
  } else {
    // generic sizes: whole CTA per transform, 4 columns per CTA
    constexpr int CG = 4;
    const int PL = padded_len(H);
    float2* S = sm;                                        // [CG][PL]
    float2* buf = sm + CG * PL;
    float2* scr = buf + PL;
    const int kx0 = blockIdx.x * CG;
    for (int cc = 0; cc < CG; ++cc) {
      const int kx = kx0 + cc;
      for (int y = threadIdx.x; y < H; y += blockDim.x)
        buf[pad32(y)] = kx < Wh ? Pb[(size_t)y * Wh + kx] : make_float2(0.f, 0.f);
      __syncthreads();
      fft_generic(buf, scr, H, c.plan_h, c.tw_h, threadIdx.x, blockDim.x);
      for (int y = threadIdx.x; y < H; y += blockDim.x) S[cc * PL + pad32(y)] = buf[pad32(y)];
      __syncthreads();
    }
    for (int f = 0; f < F; ++f) {
      const int s = f / c.O, o = f % c.O;
      float2* Qf = Q + ((size_t)b * F + f) * H * W;
      for (int job = 0; job < 2 * CG; ++job) {
        const int cc = job % CG, mir = job / CG;
        const int kx = kx0 + cc;
        if (!(kx < Wh && (mir == 0 || (kx != 0 && 2 * kx != W)))) continue;
        for (int ky = threadIdx.x; ky < H; ky += blockDim.x) {
          float2 sv = mir ? cconj(S[cc * PL + pad32(ky == 0 ? 0 : H - ky)]) : S[cc * PL + pad32(ky)];
          const float gval = transfer(c, geometry(c, ky, kx), mir, s, o);
          buf[pad32(ky)] = make_float2(sv.x * gval, -sv.y * gval);
        }
        __syncthreads();
        fft_generic(buf, scr, H, c.plan_h, c.tw_h, threadIdx.x, blockDim.x);
        const int xo = mir ? W - kx : kx;
        for (int y = threadIdx.x; y < H; y += blockDim.x) Qf[(size_t)y * W + xo] = cconj(buf[pad32(y)]);
        __syncthreads();
      }
    }
  }
}

// ----------------------------------------------------------------- K3a ---
// Scale-0 amplitudes of orientation blockIdx.y for a block of rows, with a
// 4096-bin histogram of their float bits (radix-select level 1).
template <int G>
__global__ void __launch_bounds__(kThreads) k_rows_amp0(const float2* __restrict__ Q, float* __restrict__ amp0,
                                                        unsigned* __restrict__ hist,
                                                        const __grid_constant__ FieldsConst c) {
  extern __shared__ float2 sm[];
  const int H = c.H, W = c.W, F = c.S * c.O;
  const int o = blockIdx.y, b = blockIdx.z;
  const float2* Qp = Q + ((size_t)b * F + o) * H * W;   // filter (s=0, o)
  float* A = amp0 + ((size_t)b * c.O + o) * H * W;
  unsigned* sh;
  if constexpr (G > 0) {
    constexpr int N = 32 * G, NG = kThreads / G, PL = padded_len(N);
    sh = reinterpret_cast<unsigned*>(sm + NG * PL);
    for (int i = threadIdx.x; i < kHistBins; i += kThreads) sh[i] = 0;
    __syncthreads();
    const int g = threadIdx.x / G, t = threadIdx.x % G;
    float2* buf = sm + g * PL;
    const int y = blockIdx.x * NG + g;
    const bool ok = y < H;
    float2 v[32];
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = ok ? cconj(Qp[(size_t)y * W + t + G * m]) : make_float2(0.f, 0.f);
    SyncWarp sw;
    SyncNamed sn{1 + g, G};
    if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_w, t, sw); else fft_fast<G>(v, buf, c.tw_w, t, sn);
    if (ok) {
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const float a = sqrtf(v[m].x * v[m].x + v[m].y * v[m].y);
        A[(size_t)y * W + t + G * m] = a;
        atomicAdd(&sh[__float_as_uint(a) >> 19], 1u);
      }
    }
  } else {
    const int PL = padded_len(W);
    float2* buf = sm;
    float2* scr = sm + PL;
    sh = reinterpret_cast<unsigned*>(sm + 2 * PL);
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
    const int y = blockIdx.x;
    for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(Qp[(size_t)y * W + x]);
    __syncthreads();
    fft_generic(buf, scr, W, c.plan_w, c.tw_w, threadIdx.x, blockDim.x);
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
      const float2 z = buf[pad32(x)];
      const float a = sqrtf(z.x * z.x + z.y * z.y);
      A[(size_t)y * W + x] = a;
      atomicAdd(&sh[__float_as_uint(a) >> 19], 1u);
    }
  }
  __syncthreads();
  unsigned* gh = hist + ((size_t)b * c.O + o) * kHistBins;
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

// ------------------------------------------------------------------ K4 ---
// Exact median of each amp0 plane (ref: loggabor.py:222, np.median: mean of
// the two middle order statistics for even counts).
struct MedInfo {
  unsigned bin[2];     // level-1 bins of ranks n/2-1 (or n/2) and n/2
  unsigned rank[2];    // ranks inside those bins
};

__device__ void block_exclusive_scan_1024(unsigned* data, int n, unsigned* tmp) {
  // simple single-thread-per-chunk scan: n <= 4096, blockDim 1024
  const int tid = threadIdx.x, nth = blockDim.x;
  const int per = (n + nth - 1) / nth;
  unsigned s = 0;
  for (int i = 0; i < per; ++i) { const int k = tid * per + i; if (k < n) s += data[k]; }
  tmp[tid] = s;
  __syncthreads();
  for (int off = 1; off < nth; off <<= 1) {
    unsigned add = tid >= off ? tmp[tid - off] : 0u;
    __syncthreads();
    tmp[tid] += add;
    __syncthreads();
  }
  unsigned run = tid ? tmp[tid - 1] : 0u;
  __syncthreads();
  for (int i = 0; i < per; ++i) {
    const int k = tid * per + i;
    if (k < n) { const unsigned d = data[k]; data[k] = run; run += d; }
  }
  __syncthreads();
}

// locate the bins holding the two middle ranks
__global__ void __launch_bounds__(1024) k_med_bins(const unsigned* __restrict__ hist, MedInfo* __restrict__ info,
                                                   unsigned n) {
  __shared__ unsigned h[kHistBins];
  __shared__ unsigned tmp[1024];
  const unsigned* gh = hist + (size_t)blockIdx.x * kHistBins;
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) h[i] = gh[i];
  __syncthreads();
  block_exclusive_scan_1024(h, kHistBins, tmp);
  const unsigned k[2] = {(n - 1) / 2, n / 2};
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) {
    const unsigned lo = h[i];
    const unsigned hi = (i + 1 < kHistBins) ? h[i + 1] : n;
    for (int q = 0; q < 2; ++q)
      if (k[q] >= lo && k[q] < hi) { info[blockIdx.x].bin[q] = i; info[blockIdx.x].rank[q] = k[q] - lo; }
  }
}

// gather the float bits of every value falling into one of the two bins
__global__ void __launch_bounds__(256) k_med_collect(const float* __restrict__ amp0, const MedInfo* __restrict__ info,
                                                     unsigned* __restrict__ cand, unsigned* __restrict__ cnt,
                                                     unsigned n) {
  const int plane = blockIdx.y;
  const unsigned b0 = info[plane].bin[0], b1 = info[plane].bin[1];
  const float* Ap = amp0 + (size_t)plane * n;
  const float4* A = reinterpret_cast<const float4*>(Ap);
  unsigned* out = cand + (size_t)plane * n;
  const unsigned n4 = (n + 3) / 4;
  for (unsigned base = blockIdx.x * blockDim.x; base < n4; base += gridDim.x * blockDim.x) {
    const unsigned i = base + threadIdx.x;
    float4 q = make_float4(-1.f, -1.f, -1.f, -1.f);
    if (4 * i + 3 < n) q = A[i];
    else if (i < n4) {
      q.x = Ap[4 * i];
      if (4 * i + 1 < n) q.y = Ap[4 * i + 1];
      if (4 * i + 2 < n) q.z = Ap[4 * i + 2];
    }
    const float vals[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned bits = __float_as_uint(vals[e]);
      const bool hit = vals[e] >= 0.f && ((bits >> 19) == b0 || (bits >> 19) == b1);
      const unsigned slot = agg_inc(&cnt[plane], hit);
      if (hit) out[slot] = bits;
    }
  }
}

// radix select the exact values among the candidates, then the noise threshold
__global__ void __launch_bounds__(1024) k_med_final(const unsigned* __restrict__ cand, const unsigned* __restrict__ cnt,
                                                    const MedInfo* __restrict__ info, float* __restrict__ thr,
                                                    unsigned n, double thr_factor) {
  __shared__ unsigned h[1024];
  __shared__ unsigned tmp[1024];
  __shared__ unsigned sel_prefix, sel_rank;
  const int plane = blockIdx.x;
  const unsigned* cd = cand + (size_t)plane * n;
  const unsigned c = cnt[plane];
  double val[2];
  for (int q = 0; q < 2; ++q) {
    unsigned prefix = info[plane].bin[q];   // bits >> 19
    unsigned rank = info[plane].rank[q];
    // level 2: bits 18..9, level 3: bits 8..0
    const int shifts[2] = {9, 0};
    const int widths[2] = {10, 9};
    for (int lv = 0; lv < 2; ++lv) {
      const int sh = shifts[lv], nb = 1 << widths[lv];
      for (int i = threadIdx.x; i < 1024; i += blockDim.x) h[i] = 0;
      __syncthreads();
      for (unsigned i = threadIdx.x; i < c; i += blockDim.x) {
        const unsigned bits = cd[i];
        if ((bits >> (sh + widths[lv])) == prefix) atomicAdd(&h[(bits >> sh) & (nb - 1)], 1u);
      }
      __syncthreads();
      block_exclusive_scan_1024(h, nb, tmp);
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const unsigned lo = h[i];
        const unsigned hi = (i + 1 < nb) ? h[i + 1] : 0xffffffffu;
        if (rank >= lo && rank < hi) { sel_prefix = (prefix << widths[lv]) | i; sel_rank = rank - lo; }
      }
      __syncthreads();
      prefix = sel_prefix;
      rank = sel_rank;
      __syncthreads();
    }
    val[q] = (double)__uint_as_float(prefix);
  }
  if (threadIdx.x == 0) thr[plane] = (float)(0.5 * (val[0] + val[1]) * thr_factor);
}

// ----------------------------------------------------------------- K3b ---
struct PcOut {
  float* mmax;
  float* mmin;
  uint8_t* mim;
  float* a_o;    // nullable [B][O][H][W]
  float* pc;     // nullable [B][O][H][W]
  float* amax;   // nullable [B][H][W]
};

template <int G>
struct PcShape {
  static constexpr int PIX = G == 0 ? 16 : ((32 * G > 1024) ? (32 * G) / kThreads : 4);
};

template <int G>
__global__ void __launch_bounds__(kThreads) k_rows_pc(const float2* __restrict__ Q, const float* __restrict__ thr,
                                                      PcOut out, const __grid_constant__ FieldsConst c,
                                                      int rows, int ops) {
  extern __shared__ float2 sm[];
  const int H = c.H, W = c.W, S = c.S, O = c.O, F = S * O;
  const int b = blockIdx.y;
  const int y0 = blockIdx.x * rows;
  constexpr int PIX = PcShape<G>::PIX;
  const int PL = padded_len(W);
  const int nb = rows * S * ops;             // shared buffers per stage
  const int npix = rows * W;
  float acc_a[PIX], acc_b[PIX], acc_c[PIX], best[PIX];
  int bidx[PIX];
#pragma unroll
  for (int i = 0; i < PIX; ++i) { acc_a[i] = acc_b[i] = acc_c[i] = 0.f; best[i] = -1.f; bidx[i] = 1; }
  const float* thr_b = thr + (size_t)b * O;

  for (int o0 = 0; o0 < O; o0 += ops) {
    const int no = min(ops, O - o0);
    // --- FFT jobs: (row r, orientation o0+oo, scale s) -> buffer j
    if constexpr (G > 0) {
      constexpr int NG = kThreads / G;
      const int g = threadIdx.x / G, t = threadIdx.x % G;
      SyncWarp sw;
      SyncNamed sn{1 + g, G};
      for (int j0 = 0; j0 < nb; j0 += NG) {
        const int j = j0 + g;
        const int r = j / (S * ops), rem = j % (S * ops), oo = rem / S, s = rem % S;
        const int y = y0 + r;
        const bool ok = j < nb && oo < no && y < H;
        float2* buf = sm + (j < nb ? j : 0) * PL;
        float2 v[32];
        const float2* Qp = Q + (((size_t)b * F + s * O + o0 + oo) * H + (ok ? y : 0)) * W;
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = ok ? cconj(Qp[t + G * m]) : make_float2(0.f, 0.f);
        float2* xbuf = (j < nb) ? buf : sm + nb * PL + g * PL;   // spare scratch for idle groups
        if constexpr (G <= 32) fft_fast<G>(v, xbuf, c.tw_w, t, sw); else fft_fast<G>(v, xbuf, c.tw_w, t, sn);
        if constexpr (G <= 32) sw(); else sn();
        if (j < nb) {
#pragma unroll
          for (int m = 0; m < 32; ++m) buf[pad32(t + G * m)] = cconj(v[m]);
        }
      }
    } else {
      float2* scr = sm + nb * PL;
      for (int j = 0; j < nb; ++j) {
        const int oo = j / S, s = j % S;
        if (oo >= no) break;
        float2* buf = sm + j * PL;
        const float2* Qp = Q + (((size_t)b * F + s * O + o0 + oo) * H + y0) * W;
        for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(Qp[x]);
        __syncthreads();
        fft_generic(buf, scr, W, c.plan_w, c.tw_w, threadIdx.x, blockDim.x);
        for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(buf[pad32(x)]);
      }
    }
    __syncthreads();
    // --- per-pixel phase congruency for the orientations of this stage
#pragma unroll
    for (int i = 0; i < PIX; ++i) {
      const int p = threadIdx.x + kThreads * i;
      if (p >= npix) continue;
      const int r = p / W, x = p % W;
      if (y0 + r >= H) continue;
      for (int oo = 0; oo < no; ++oo) {
        const int o = o0 + oo;
        const float2* bb = sm + ((r * ops + oo) * S) * PL + pad32(x);
        float se = 0.f, so = 0.f, sa = 0.f, mx = 0.f;
        for (int s = 0; s < S; ++s) {
          const float2 z = bb[s * PL];
          const float a = sqrtf(z.x * z.x + z.y * z.y);
          se += z.x; so += z.y; sa += a; mx = fmaxf(mx, a);
        }
        const float xe = sqrtf(se * se + so * so) + 1e-4f;
        const float me = se / xe, mo = so / xe;
        float en = 0.f;
        for (int s = 0; s < S; ++s) {
          const float2 z = bb[s * PL];
          en += z.x * me + z.y * mo - fabsf(z.x * mo - z.y * me);
        }
        en = fmaxf(en - thr_b[o], 0.f);
        const float spread = (sa / (mx + 1e-4f) - 1.f) * c.inv_sm1;
        const float wgt = 1.f / (1.f + expf(c.spread_gain * (c.spread_cutoff - spread)));
        const float pc = wgt * en / (sa + 1e-4f);
        const float pcc = pc * c.cos_a[o], pcs = pc * c.sin_a[o];
        acc_a[i] += pcc * pcc;
        acc_b[i] += pcc * pcs;
        acc_c[i] += pcs * pcs;
        if (sa > best[i]) { best[i] = sa; bidx[i] = o + 1; }
        const size_t po = (((size_t)b * O + o) * H + (y0 + r)) * W + x;
        if (out.a_o) out.a_o[po] = sa;
        if (out.pc) out.pc[po] = pc;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < PIX; ++i) {
    const int p = threadIdx.x + kThreads * i;
    if (p >= npix) continue;
    const int r = p / W, x = p % W;
    if (y0 + r >= H) continue;
    const float a = acc_a[i], bq = 2.f * acc_b[i], cq = acc_c[i];
    const float root = sqrtf(bq * bq + (a - cq) * (a - cq));
    const size_t po = ((size_t)b * H + (y0 + r)) * W + x;
    out.mmax[po] = 0.5f * (cq + a + root);
    out.mmin[po] = fmaxf(0.5f * (cq + a - root), 0.f);
    out.mim[po] = (uint8_t)bidx[i];
    if (out.amax) out.amax[po] = best[i];
  }
}

// ================================================================ host side

static int fast_g(int n) {
  if (n < 32 || n > 4096 || (n & (n - 1))) return 0;
  return n / 32;
}

static bool make_plan(int n, GenericPlan& p) {
  p.n_pass = 0;
  int m = n;
  const int order[5] = {5, 3, 8, 4, 2};
  for (int r : order) {
    while (m % r == 0 && p.n_pass < 16) {
      if (r == 8 && m % 8 != 0) break;
      p.radix[p.n_pass++] = r;
      m /= r;
    }
  }
  return m == 1;
}

struct FieldsPlan {
  int B, H, W, Wh, S, O, F;
  int gw, gh;
  size_t off_P, off_Q, off_amp0, off_hist, off_info, off_cand, off_cnt, off_thr, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static FieldsPlan plan_fields(int B, int H, int W, int S, int O) {
  FieldsPlan p{};
  p.B = B; p.H = H; p.W = W; p.Wh = W / 2 + 1; p.S = S; p.O = O; p.F = S * O;
  p.gw = fast_g(W); p.gh = fast_g(H);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
  const size_t n = (size_t)H * W;
  p.off_P = take((size_t)B * H * p.Wh * sizeof(float2));
  p.off_Q = take((size_t)B * p.F * n * sizeof(float2));
  p.off_amp0 = take((size_t)B * O * n * sizeof(float));
  p.off_hist = take((size_t)B * O * kHistBins * sizeof(unsigned));
  p.off_info = take((size_t)B * O * sizeof(MedInfo));
  p.off_cand = take((size_t)B * O * n * sizeof(unsigned));
  p.off_cnt = take((size_t)B * O * sizeof(unsigned));
  p.off_thr = take((size_t)B * O * sizeof(float));
  p.total = off;
  return p;
}

size_t fields_workspace_bytes(int B, int H, int W, int S, int O) {
  return plan_fields(B, H, W, S, O).total;
}

template <class K>
static cudaError_t set_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int G>
static cudaError_t launch_rows_fwd(const float* img, float2* P, const FieldsConst& c, cudaStream_t st) {
  size_t smem;
  dim3 grid;
  if constexpr (G > 0) {
    const int NG = kThreads / G;
    smem = (size_t)NG * padded_len(32 * G) * sizeof(float2);
    grid = dim3(((c.H + 1) / 2 + NG - 1) / NG, c.B);
  } else {
    smem = (size_t)2 * padded_len(c.W) * sizeof(float2);
    grid = dim3((c.H + 1) / 2, c.B);
  }
  cudaError_t e = set_smem(k_rows_fwd<G>, smem);
  if (e != cudaSuccess) return e;
  k_rows_fwd<G><<<grid, kThreads, smem, st>>>(img, P, c);
  return cudaGetLastError();
}

template <int G>
static cudaError_t launch_cols(const float2* P, float2* Q, const FieldsConst& c, cudaStream_t st) {
  size_t smem;
  dim3 grid;
  if constexpr (G > 0) {
    const int N = 32 * G, NG = kThreads / G, CG = NG / 2, PL = padded_len(N);
    smem = ((size_t)CG * PL + 2 * (size_t)CG * N + (size_t)NG * PL) * sizeof(float2);
    grid = dim3((c.Wh + CG - 1) / CG, c.B);
  } else {
    const int PL = padded_len(c.H);
    smem = (size_t)(4 * PL + 2 * PL) * sizeof(float2);
    grid = dim3((c.Wh + 3) / 4, c.B);
  }
  cudaError_t e = set_smem(k_cols<G>, smem);
  if (e != cudaSuccess) return e;
  k_cols<G><<<grid, kThreads, smem, st>>>(P, Q, c);
  return cudaGetLastError();
}

template <int G>
static cudaError_t launch_amp0(const float2* Q, float* amp0, unsigned* hist, const FieldsConst& c, cudaStream_t st) {
  size_t smem;
  dim3 grid;
  if constexpr (G > 0) {
    const int NG = kThreads / G;
    smem = (size_t)NG * padded_len(32 * G) * sizeof(float2) + kHistBins * sizeof(unsigned);
    grid = dim3((c.H + NG - 1) / NG, c.O, c.B);
  } else {
    smem = (size_t)2 * padded_len(c.W) * sizeof(float2) + kHistBins * sizeof(unsigned);
    grid = dim3(c.H, c.O, c.B);
  }
  cudaError_t e = set_smem(k_rows_amp0<G>, smem);
  if (e != cudaSuccess) return e;
  k_rows_amp0<G><<<grid, kThreads, smem, st>>>(Q, amp0, hist, c);
  return cudaGetLastError();
}

template <int G>
static cudaError_t launch_pc(const float2* Q, const float* thr, const PcOut& out, const FieldsConst& c,
                             cudaStream_t st) {
  int rows, ops;
  size_t nbuf;
  if constexpr (G > 0) {
    const int NG = kThreads / G;
    rows = NG / (c.S * c.O);
    if (rows < 1) rows = 1;
    if (rows > 1) ops = c.O;
    else { ops = NG / c.S; if (ops < 1) ops = 1; if (ops > c.O) ops = c.O; }
    // PIX bound: rows*W pixels over kThreads threads
    while (rows > 1 && rows * c.W > kThreads * PcShape<G>::PIX) --rows;
    const int nb = rows * c.S * ops;
    nbuf = nb + NG;   // + spare scratch for idle groups
  } else {
    rows = 1; ops = 1;
    nbuf = c.S + 1;
  }
  const size_t smem = nbuf * padded_len(c.W) * sizeof(float2);
  cudaError_t e = set_smem(k_rows_pc<G>, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((c.H + rows - 1) / rows, c.B);
  k_rows_pc<G><<<grid, kThreads, smem, st>>>(Q, thr, out, c, rows, ops);
  return cudaGetLastError();
}

#define R2_DISPATCH_G(g, FN, ...)                       \
  switch (g) {                                          \
    case 1: e = FN<1>(__VA_ARGS__); break;              \
    case 2: e = FN<2>(__VA_ARGS__); break;              \
    case 4: e = FN<4>(__VA_ARGS__); break;              \
    case 8: e = FN<8>(__VA_ARGS__); break;              \
    case 16: e = FN<16>(__VA_ARGS__); break;            \
    case 32: e = FN<32>(__VA_ARGS__); break;            \
    case 64: e = FN<64>(__VA_ARGS__); break;            \
    case 128: e = FN<128>(__VA_ARGS__); break;          \
    default: e = FN<0>(__VA_ARGS__); break;             \
  }

int fields_run(const float* images, int B, int H, int W, const BankConsts& bk, const FieldsOutputs& o,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  const FieldsPlan p = plan_fields(B, H, W, bk.n_scales, bk.n_orient);
  if (ws_bytes < p.total) return 1;
  FieldsConst c{};
  c.B = B; c.H = H; c.W = W; c.Wh = p.Wh; c.S = bk.n_scales; c.O = bk.n_orient;
  for (int s = 0; s < c.S; ++s) c.log_lambda[s] = (float)bk.log_lambda[s];
  c.inv_den_r = (float)bk.inv_den_r;
  c.inv_den_a = (float)bk.inv_den_a;
  for (int o = 0; o < c.O; ++o) {
    c.ang[o] = (float)bk.angle[o];
    c.cos_a[o] = (float)bk.cos_a[o];
    c.sin_a[o] = (float)bk.sin_a[o];
  }
  c.spread_cutoff = (float)bk.spread_cutoff;
  c.spread_gain = (float)bk.spread_gain;
  c.inv_sm1 = (float)(1.0 / (c.S > 1 ? c.S - 1 : 1));
  c.lp_lncut = (float)bk.lp_lncut;
  c.inv_hw = (float)(1.0 / ((double)H * W));
  c.thr_factor = bk.thr_factor;
  c.tw_w = twiddle_table(W);
  c.tw_h = twiddle_table(H);
  if (!c.tw_w || !c.tw_h) return 3;
  if (!p.gw && !make_plan(W, c.plan_w)) return 2;
  if (!p.gh && !make_plan(H, c.plan_h)) return 2;

  char* w = static_cast<char*>(ws);
  float2* P = reinterpret_cast<float2*>(w + p.off_P);
  float2* Q = reinterpret_cast<float2*>(w + p.off_Q);
  float* amp0 = reinterpret_cast<float*>(w + p.off_amp0);
  unsigned* hist = reinterpret_cast<unsigned*>(w + p.off_hist);
  MedInfo* info = reinterpret_cast<MedInfo*>(w + p.off_info);
  unsigned* cand = reinterpret_cast<unsigned*>(w + p.off_cand);
  unsigned* cnt = reinterpret_cast<unsigned*>(w + p.off_cnt);
  float* thr = reinterpret_cast<float*>(w + p.off_thr);

  cudaError_t e;
  if ((e = cudaMemsetAsync(hist, 0, (size_t)B * c.O * kHistBins * sizeof(unsigned), st)) != cudaSuccess) return 3;
  if ((e = cudaMemsetAsync(cnt, 0, (size_t)B * c.O * sizeof(unsigned), st)) != cudaSuccess) return 3;
  R2_DISPATCH_G(p.gw, launch_rows_fwd, images, P, c, st);
  if (e != cudaSuccess) return 3;
  R2_DISPATCH_G(p.gh, launch_cols, P, Q, c, st);
  if (e != cudaSuccess) return 3;
  R2_DISPATCH_G(p.gw, launch_amp0, Q, amp0, hist, c, st);
  if (e != cudaSuccess) return 3;
  const unsigned n = (unsigned)((size_t)H * W);
  k_med_bins<<<B * c.O, 1024, 0, st>>>(hist, info, n);
  {
    dim3 grid((unsigned)min((size_t)64, ((size_t)n / 4 + 255) / 256 + 1), B * c.O);
    k_med_collect<<<grid, 256, 0, st>>>(amp0, info, cand, cnt, n);
  }
  k_med_final<<<B * c.O, 1024, 0, st>>>(cand, cnt, info, thr, n, c.thr_factor);
  if (cudaGetLastError() != cudaSuccess) return 3;
  PcOut po{o.mmax, o.mmin, o.mim, o.a_o, o.pc, o.amax};
  R2_DISPATCH_G(p.gw, launch_pc, Q, thr, po, c, st);
  if (e != cudaSuccess) return 3;
  return 0;
}

}  // namespace r2
