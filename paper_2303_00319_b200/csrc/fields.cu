// Log-Gabor phase-congruency filter bank, moment maps and maximum index map.
//
// Replaces ref: loggabor.py:122-251 (build_filter_bank, apply_bank,
// orientation_amplitudes, phase_congruency_moments) and mim.py:43-55
// (build_mim) with a two-pass 2-D FFT whose inter-pass planes are the only
// per-filter HBM traffic:
//
//   K1  rows_fwd  real rows -> half-spectrum rows (two rows per complex FFT)
//   K2  cols      column FFT once per column; then, per filter and with no
//                 CTA barrier, multiply by the analytically generated
//                 transfer function and inverse-FFT the column (mirror
//                 columns from Hermitian symmetry), stored from registers
//   K3a rows_amp0 inverse row FFT of the scale-0 planes -> scale-0 responses
//                 (kept for K3b), |response| and a radix histogram
//   K4  median    exact np.median of each scale-0 amplitude plane
//   K3b rows_pc   inverse row FFTs of scales 1..S-1 (scale 0 re-loaded),
//                 fused phase congruency, moments, orientation amplitude
//                 sums and MIM argmax.
//
// Layouts (batch-major):
//   image [B][H][W] f32               P   [B][H][Wh] c64 (Wh = W/2+1), row-major
//   Q     [B][S*O][Hp/4][W][4] c64    4-row column tiles: element (y, x) at
//                                     ((y>>2)*W + x)*4 + (y&3), Hp = H rounded up to 4
//   R0    [B][O][H][W] c64            scale-0 responses, row-major
//   amp0  [B][O][H*W] f32
//   outputs M, m [B][H][W] f32, MIM [B][H][W] u8, optional a_o/pc [B][O][H][W], amax [B][H][W]
#include <algorithm>
#include <cmath>

#include "fft.cuh"
#include "fields.h"
#include "tma.cuh"

namespace r2 {

constexpr int kThreads = 256;
// K2 CTA size: two warps per direct+mirror column pair keeps smem per CTA low
// enough for three CTAs per SM
template <int G>
struct ColsCfg { static constexpr int T = G == 0 ? 256 : (G >= 64 ? 2 * G : 128); };
constexpr int kHistBins = 4096;   // float bits >> 19 of a non-negative float
constexpr int kAmpRows = 4;       // row groups per k_rows_amp0 CTA
constexpr int kPcTmaBox = 256;    // columns per TMA box of the row passes (box dims <= 256)
constexpr int kMaxS = 8;
constexpr int kMaxO = 16;
constexpr float kPi = 3.14159265358979f;
constexpr float kTwoPi = 6.28318530717959f;

struct FieldsConst {
  int B, H, W, Wh, Hp, S, O;
  float log_lambda[kMaxS];     // ln(lambda_s) = -ln(f0_s)
  float a2;                    // log2(e) / (2 ln(sigma_on_f)^2)
  float b2;                    // log2(e) / (2 sigma_theta^2)
  // the fast column passes work on pre-scaled coordinates, so a transfer
  // value is exp2(-(d^2 + dr^2)): ln r and ln(lambda) times sqrt(a2),
  // angles times sqrt(b2)
  float sa, sb;                // sqrt(a2), sqrt(b2)
  float ll_s[kMaxS], ang_s[kMaxO];
  float pi_s, two_pi_s;
  float ang[kMaxO], cos_a[kMaxO], sin_a[kMaxO];
  float spread_cutoff, spread_gain, inv_sm1;
  float lp_lncut;              // ln(0.45)
  float log2_inv_hw;           // log2(1 / (H*W)): the inverse-FFT scale folded into the exponent
  double thr_factor;           // T = median * thr_factor
  const float* xfer;           // explicit transfer [S*O][H][W] (apply_bank of a given bank) or nullptr
  float inv_hw;                // 1 / (H*W) for the explicit transfer
  const float2* tw_w;          // W_W^j
  const float2* tw_h;          // W_H^j
  GenericPlan plan_w, plan_h;
  int out_vec;                 // the map outputs take two-pixel vector stores (8-byte aligned floats, 2-byte aligned MIM)
};

// numpy.fft.fftfreq(n)[k]
R2_DEV float fftfreq(int k, int n) { return (float)(k < (n + 1) / 2 ? k : k - n) / (float)n; }

// 4-row column-tile plane index: a 32-byte sector holds rows 4j..4j+3 of one
// column, so a column FFT's stores fill whole sectors
#ifndef R2_QT
#define R2_QT 4
#endif
// rows per column tile: 4 makes every k_cols store instruction write whole
// 32-byte sectors; 2 would halve the row kernels' L1 wavefronts
// (rows_pc -15 %, amp0 -13 % measured) but k_cols's half-sector stores then
// force DRAM fill reads (k_cols 2.3 -> 9.3 ms) -- see DESIGN 7b
constexpr int kQT = R2_QT;
R2_DEV size_t tq(int y, int x, int W) { return ((size_t)(y / kQT) * W + x) * kQT + (y % kQT); }

R2_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

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
    SyncWarp sw{group_mask(G)};
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
// Spectrum geometry of column kx (ref: loggabor.py:122-159, r = hypot(fx, fy),
// theta = atan2(fy, fx), lowpass 1 / (1 + (r/0.45)^30), DC zeroed):
//   lnr, L2 = log2(lowpass / (H*W)) (-inf at DC), theta of the direct column.
// The mirror column W - kx has the same r and theta_m = +-pi - theta.
R2_DEV void geometry(const FieldsConst& c, int ky, int kx, float& lnr, float& L2, float& th) {
  const float fy = fftfreq(ky, c.H);
  const float fx = fftfreq(kx, c.W);
  if (ky == 0 && kx == 0) {
    lnr = 0.f;
    L2 = -INFINITY;
    th = 0.f;
    return;
  }
  lnr = 0.5f * logf(fx * fx + fy * fy);
  const float lp = 1.f / (1.f + expf(30.f * (lnr - c.lp_lncut)));
  L2 = log2f(lp) + c.log2_inv_hw;
  th = atan2f(fy, fx);
}

// transfer of filter (s, o) as exp2(L2 - a2 (ln r - ln f0)^2 - b2 dtheta^2)
R2_DEV float transfer(float lnr, float L2, float th, float ll, float ang, float a2, float b2) {
  float d = fabsf(th - ang);
  d = d > kPi ? kTwoPi - d : d;
  const float dr = lnr + ll;
  return ex2(fmaf(d * d, -b2, fmaf(dr * dr, -a2, L2)));
}

// transfer of filter (s, o) without the radius-only factor lowpass / (H*W),
// which the fast column pass folds into the spectrum once per column; all
// arguments pre-scaled (FieldsConst::sa / sb): the wrapped angle distance is
// min(d, 2 pi - d) and the exponent -(d^2 + dr^2)
R2_DEV float transfer_s(float lnr_s, float th_s, float ll_s, float ang_s, float two_pi_s) {
  float d = fabsf(th_s - ang_s);
  d = fminf(d, two_pi_s - d);
  const float dr = lnr_s + ll_s;
  return ex2(-fmaf(d, d, dr * dr));
}

// Per-filter multiply + inverse column FFT + store for one column (direct or
// mirror), G >= 32.  One instruction stream serves both kinds of warp (two
// unrolled copies thrash the instruction cache); the differences are
// per-thread constants: with t < G and G a multiple of 32 every padded
// spectrum index is a base plus a signed compile-time multiple of m, the
// mirror angle is +-pi - theta with the sign fixed per unrolled element
// (ky < N/2 <=> m < 16), and the imaginary part takes a sign.  The spectrum
// buffer holds the periodic copy S[N] = S[0], so the mirror index needs no wrap.
template <int G, class Sync>
R2_DEV void cols_filters(const FieldsConst& c, const float2* Sc, const float2* Geo,
                         float2* buf, float2* Qb, int xo, int t, bool mir, Sync& sync,
                         const CUtensorMap* qst, int b) {
  constexpr int N = 32 * G;
  constexpr int PS = G + G / 32;                          // padded stride of one m step
  const int W = c.W, F = c.S * c.O;
  // pad32(N - t - G m) and pad32(t + G m) as base -/+ PS * m (t < G, G % 32 == 0)
  const float2* sp = Sc + (mir ? (N + N / 32) - t - ((t + 31) >> 5) : t + (t >> 5));
  const int sstep = mir ? -PS : PS;
  const float tsg = mir ? -1.f : 1.f;                     // theta_m = +-pi - theta
  const float tpi = mir ? c.pi_s : 0.f;
  const float ysg = mir ? 1.f : -1.f;                     // conj for the direct column
  const float two_pi_s = c.two_pi_s;
  float2 v[32];
  for (int f = 0; f < F; ++f) {
    const int s = f / c.O, o = f % c.O;
    const float ll = c.ll_s[s], ang = c.ang_s[o];
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      const int ky = t + G * m;
      const float2 sv = sp[sstep * m];
      const float2 gq = Geo[ky];                         // (ln r, theta): one 8-byte load
      const float th = fmaf(tsg, gq.y, m < 16 ? tpi : -tpi);
      const float gv = transfer_s(gq.x, th, ll, ang, two_pi_s);
      // conj(spectrum * G) for the inverse; the mirror reads S(-ky, kx) = conj S(ky, W - kx)
      v[m] = __fmul2_rn(sv, make_float2(gv, gv * ysg));
    }
    if (qst) {
      // the previous filter's tensor stores have read buf before the FFT reuses it
      if (t == 0) bulk_wait_read0();
      sync();
    }
    fft_fast<G>(v, buf, c.tw_h, t, sync);
    if (qst) {
      // the column in natural row order is N / 1,024 {4 rows x 1 column x 256
      // tiles} boxes of the 4-row tile plane: stage it, one thread stores them
      sync();
#pragma unroll
      for (int m = 0; m < 32; ++m) buf[t + G * m] = cconj(v[m]);
      fence_proxy_async();
      sync();
      if (t == 0) {
#ifndef R2_EXP_NOSTORE
        for (int k = 0; k < N / 1024; ++k)
          tma_store_3d(qst, 0, xo, (b * c.S * c.O + f) * (c.Hp >> 2) + 256 * k, buf + 1024 * k);
#endif
        bulk_commit();
      }
      continue;
    }
    // y = t + G m: tile row (t >> 2) + (G / 4) m, lane t & 3.  W is re-read
    // opaquely each filter so the compiler does not hoist 32 64-bit store
    // addresses across the loop (register spills)
    int wv;
    asm volatile("mov.b32 %0, %1;" : "=r"(wv) : "r"(W));
    float2* q = Qb + (size_t)f * c.Hp * wv + ((size_t)(t / kQT) * wv + xo) * kQT + (t % kQT);
    const size_t step = (size_t)G * wv;           // (G / 4) tile rows of 4 W elements
#pragma unroll
    for (int m = 0; m < 32; ++m) q[m * step] = cconj(v[m]);
  }
  if (qst && t == 0) bulk_wait0();               // the last stores have left shared memory
}

template <int G>
__global__ void __launch_bounds__(ColsCfg<G>::T, ColsCfg<G>::T == 128 ? 3 : 1) k_cols(const __grid_constant__ CUtensorMap qst,
                                                   const float2* __restrict__ P, float2* __restrict__ Q,
                                                   const __grid_constant__ FieldsConst c, int use_tma) {
  extern __shared__ float2 sm_raw[];
  // 128-byte aligned base (TMA store sources)
  float2* sm = reinterpret_cast<float2*>(reinterpret_cast<char*>(sm_raw) + ((128u - (smem_u32(sm_raw) & 127u)) & 127u));
  const int H = c.H, W = c.W, Wh = c.Wh, F = c.S * c.O;
  const int b = blockIdx.y;
  const float2* Pb = P + (size_t)b * H * Wh;
  float2* Qb = Q + (size_t)b * F * c.Hp * W;
  if constexpr (G > 0) {
    constexpr int N = 32 * G;        // == H
    constexpr int NG = ColsCfg<G>::T / G;
    // A CTA owns direct columns kx0..kx0+CG-1 and their mirrors W-kx.
    constexpr int CG = NG / 2;
    constexpr int NS = CG;           // spectrum columns held
    constexpr int PL = padded_len(N), PLA = (PL + 15) & ~15;   // buffer pitch: 128-byte multiple
    float2* bufs = sm;                                           // [NG][PLA]
    float2* S = bufs + NG * PLA;                                 // [NS][PL]
    float2* geo = S + NS * PL;                                   // [NS][N] (ln r, theta)
    const int g = threadIdx.x / G, t = threadIdx.x % G;
    float2* buf = bufs + g * PLA;
    const int kx0 = blockIdx.x * CG;
    SyncWarp sw{group_mask(G)};
    SyncNamed sn{1 + g, G};
    float2 v[32];
    // 1. forward column FFTs of the half spectrum
    if (g < NS) {
      const int kx = kx0 + g;
      const bool ok = kx < Wh;
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = ok ? Pb[(size_t)(t + G * m) * Wh + kx] : make_float2(0.f, 0.f);
      if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_h, t, sw); else fft_fast<G>(v, buf, c.tw_h, t, sn);
#pragma unroll
      for (int m = 0; m < 32; ++m) S[g * PL + pad32(t + G * m)] = v[m];
    }
    __syncthreads();
    // 2. spectrum geometry of the NS columns
    for (int i = threadIdx.x; i < NS * N; i += ColsCfg<G>::T) {
      float lnr, L2, th;
      geometry(c, i % N, min(kx0 + i / N, Wh - 1), lnr, L2, th);
      geo[i] = make_float2(lnr * c.sa, th * c.sb);
      // the radius-only factor lowpass / (H*W) goes into the spectrum (the
      // mirror column has the same radius); 0 at DC
      const int cc = i / N, ky = i % N;
      const float2 sv = cscale(S[cc * PL + pad32(ky)], ex2(L2));
      S[cc * PL + pad32(ky)] = sv;
      if (ky == 0) S[cc * PL + pad32(N)] = sv;   // periodic copy for the mirror index
    }
    __syncthreads();
    // 3. every group independently: per filter multiply + inverse column FFT,
    //    stored straight from registers into the 4-row column-tile plane
    const int mir = g / CG;
    const int cc = g % CG;           // local spectrum column
    const int kx = kx0 + cc;
    const bool valid = mir == 0 ? kx < Wh : (kx != 0 && 2 * kx < W);
    if (!valid) return;              // whole group idles; no CTA barrier follows
    const int xo = mir ? W - kx : kx;
    const float2* Sc = S + cc * PL;
    const float2* Geo = geo + cc * N;
    if constexpr (G >= 32) {
      const CUtensorMap* qs = use_tma ? &qst : nullptr;
      if constexpr (G <= 32) cols_filters<G>(c, Sc, Geo, buf, Qb, xo, t, mir != 0, sw, qs, b);
      else cols_filters<G>(c, Sc, Geo, buf, Qb, xo, t, mir != 0, sn, qs, b);
      return;
    } else {
    // 512-row columns (G = 16) also leave by TMA: one {4 rows x 1 column x 128
    // tiles} box per column and filter, staged in natural row order in the
    // group's exchange buffer
    const CUtensorMap* qs = (G == 16 && use_tma) ? &qst : nullptr;
    for (int f = 0; f < F; ++f) {
      const int s = f / c.O, o = f % c.O;
      const float ll = c.ll_s[s], ang = c.ang_s[o];
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const int ky = t + G * m;
        float th = Geo[ky].y;
        float2 sv;
        if (mir) {
          sv = Sc[pad32((N - ky) & (N - 1))];       // S(-ky, kx) = conj S(ky, W - kx)
          th = (ky < N / 2 ? c.pi_s : -c.pi_s) - th;
        } else {
          sv = Sc[pad32(ky)];
          sv.y = -sv.y;
        }
        const float gv = transfer_s(Geo[ky].x, th, ll, ang, c.two_pi_s);
        v[m] = make_float2(sv.x * gv, sv.y * gv);   // conj(spectrum * G) for the inverse
      }
      if (qs) {
        // the previous filter's tensor store has read buf before the FFT reuses it
        if (t == 0) bulk_wait_read0();
        sw();
      }
      fft_fast<G>(v, buf, c.tw_h, t, sw);
      if (qs) {
        sw();
#pragma unroll
        for (int m = 0; m < 32; ++m) buf[t + G * m] = cconj(v[m]);
        fence_proxy_async();
        sw();
        if (t == 0) {
          tma_store_3d(qs, 0, xo, (b * F + f) * (c.Hp >> 2), buf);
          bulk_commit();
        }
        continue;
      }
      float2* Qf = Qb + (size_t)f * c.Hp * W;
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const int y = t + G * m;
        Qf[tq(y, xo, W)] = cconj(v[m]);
      }
    }
    if (qs && t == 0) bulk_wait0();                // the last store has left shared memory
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
      float2* Qf = Qb + (size_t)f * c.Hp * W;
      for (int job = 0; job < 2 * CG; ++job) {
        const int cc = job % CG, mir = job / CG;
        const int kx = kx0 + cc;
        if (!(kx < Wh && (mir == 0 || (kx != 0 && 2 * kx != W)))) continue;
        for (int ky = threadIdx.x; ky < H; ky += blockDim.x) {
          float lnr, L2, th;
          geometry(c, ky, kx, lnr, L2, th);
          float2 sv;
          if (mir) {
            sv = S[cc * PL + pad32(ky == 0 ? 0 : H - ky)];
            th = (2 * ky < H ? kPi : -kPi) - th;
          } else {
            sv = S[cc * PL + pad32(ky)];
            sv.y = -sv.y;
          }
          const float gv = c.xfer ? c.xfer[((size_t)f * H + ky) * W + (mir ? W - kx : kx)] * c.inv_hw
                                  : transfer(lnr, L2, th, c.log_lambda[s], c.ang[o], c.a2, c.b2);
          buf[pad32(ky)] = make_float2(sv.x * gv, sv.y * gv);
        }
        __syncthreads();
        fft_generic(buf, scr, H, c.plan_h, c.tw_h, threadIdx.x, blockDim.x);
        const int xo = mir ? W - kx : kx;
        for (int y = threadIdx.x; y < H; y += blockDim.x) Qf[tq(y, xo, W)] = cconj(buf[pad32(y)]);
        __syncthreads();
      }
    }
  }
}

// ----------------------------------------------------------------- K3a ---
// Scale-0 responses of orientation blockIdx.y for a block of rows: written
// out (for K3b) with |response| and a 4096-bin histogram of its float bits
// (radix-select level 1 of the median).
// bulk L2 prefetch of `bytes` (multiple of 16) from a 16-byte aligned address
R2_DEV void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}
R2_DEV float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int G>
__global__ void __launch_bounds__(kThreads) k_rows_amp0(const float2* __restrict__ Q, float2* __restrict__ R0,
                                                        float* __restrict__ amp0, unsigned* __restrict__ hist,
                                                        const __grid_constant__ FieldsConst c, int ahead,
                                                        int write_r0) {
  extern __shared__ float2 sm[];
  const int H = c.H, W = c.W, F = c.S * c.O;
  const int o = blockIdx.y, b = blockIdx.z;
  const float2* Qp = Q + ((size_t)b * F + o) * c.Hp * W;   // filter (s=0, o)
  float* A = amp0 + ((size_t)b * c.O + o) * H * W;
  float2* Rp = R0 + ((size_t)b * c.O + o) * H * W;
  unsigned* sh;
  if constexpr (G > 0) {
    constexpr int NG = kThreads / G, PL = padded_len(32 * G);
    sh = reinterpret_cast<unsigned*>(sm + NG * PL);
    for (int i = threadIdx.x; i < kHistBins; i += kThreads) sh[i] = 0;
    __syncthreads();
    const int g = threadIdx.x / G, t = threadIdx.x % G;
    float2* buf = sm + g * PL;
    // kAmpRows row groups per CTA amortise the histogram zero / flush
    const int yend = min(H, (blockIdx.x + 1) * NG * kAmpRows);
    for (int y = blockIdx.x * NG * kAmpRows + g; y < yend; y += NG) {
      if (threadIdx.x == 0) {
        if (y + NG < yend) {                      // the next row group's Q tiles into L2
          for (int yt = (y + NG) & ~(kQT - 1); yt < min(yend, y + 2 * NG); yt += kQT)
            l2_prefetch(Qp + (size_t)yt * W, (unsigned)(kQT * W * sizeof(float2)));
        } else if (ahead > 0) {                   // the first row group of the CTA `ahead` slots later
          const long long lin = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x + ahead;
          if (lin < (long long)gridDim.x * gridDim.y * gridDim.z) {
            const int nx = (int)(lin % gridDim.x), no = (int)((lin / gridDim.x) % gridDim.y);
            const int nbz = (int)(lin / ((long long)gridDim.x * gridDim.y));
            const float2* nQ = Q + ((size_t)nbz * F + no) * c.Hp * W;
            const int ny = nx * NG * kAmpRows;
            for (int yt = ny & ~(kQT - 1); yt < min(H, ny + NG); yt += kQT)
              l2_prefetch(nQ + (size_t)yt * W, (unsigned)(kQT * W * sizeof(float2)));
          }
        }
      }
      float2 v[32];
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = cconj(Qp[tq(y, t + G * m, W)]);
      SyncWarp sw{group_mask(G)};
      SyncNamed sn{1 + g, G};
      if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_w, t, sw); else fft_fast<G>(v, buf, c.tw_w, t, sn);
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const float2 z = cconj(v[m]);
        // MUFU sqrt: the median only needs amplitudes consistent with themselves
        const float a = sqrt_approx(fmaf(z.x, z.x, z.y * z.y));
        if (write_r0) Rp[(size_t)y * W + t + G * m] = z;   // not needed when K3b recomputes scale 0
        A[(size_t)y * W + t + G * m] = a;
        atomicAdd(&sh[__float_as_uint(a) >> 19], 1u);
      }
      if constexpr (G <= 32) sw(); else sn();   // buf is rewritten by the next row
    }
  } else {
    const int PL = padded_len(W);
    float2* buf = sm;
    float2* scr = sm + PL;
    sh = reinterpret_cast<unsigned*>(sm + 2 * PL);
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
    const int y = blockIdx.x;
    for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(Qp[tq(y, x, W)]);
    __syncthreads();
    fft_generic(buf, scr, W, c.plan_w, c.tw_w, threadIdx.x, blockDim.x);
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
      const float2 z = cconj(buf[pad32(x)]);
      const float a = sqrt_approx(fmaf(z.x, z.x, z.y * z.y));
      Rp[(size_t)y * W + x] = z;
      A[(size_t)y * W + x] = a;
      atomicAdd(&sh[__float_as_uint(a) >> 19], 1u);
    }
  }
  __syncthreads();
  unsigned* gh = hist + ((size_t)b * c.O + o) * kHistBins;
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&gh[i], sh[i]);
}


// K3a for 1,024-point rows with TMA inputs: per row group (8 rows) the four
// row pairs arrive as 3-D boxes {2 rows of a 4-row column tile, 256 columns}
// in the FFT buffers of the pair's two groups (128-byte pitch), so the
// groups read their rows from shared memory; otherwise as k_rows_amp0<32>.
#ifndef R2_AMP_TILE
#define R2_AMP_TILE 1
#endif
constexpr bool kAmpTile = R2_AMP_TILE;   // K3a stages whole 4-row tile rows (bulk copies) instead of 2-row boxes
__global__ void __launch_bounds__(kThreads) k_rows_amp0_tma(const __grid_constant__ CUtensorMap qmap,
                                                            const float2* __restrict__ Q, float2* __restrict__ R0,
                                                            float* __restrict__ amp0, unsigned* __restrict__ hist,
                                                            const __grid_constant__ FieldsConst c, int ahead,
                                                            int write_r0) {
  constexpr int G = 32, W = 1024, NG = kThreads / G, PL = (padded_len(W) + 15) & ~15;
  extern __shared__ float2 sm_raw[];
  __shared__ uint64_t s_bar[NG / 2];              // one per row pair: its two groups start on their own rows
  float2* sm = reinterpret_cast<float2*>(reinterpret_cast<char*>(sm_raw) + ((128u - (smem_u32(sm_raw) & 127u)) & 127u));
  const int H = c.H, F = c.S * c.O;
  const int o = blockIdx.y, b = blockIdx.z;
  const float2* Qp = Q + ((size_t)b * F + o) * c.Hp * W;   // filter (s=0, o)
  float* A = amp0 + ((size_t)b * c.O + o) * H * W;
  float2* Rp = R0 + ((size_t)b * c.O + o) * H * W;
  unsigned* sh = reinterpret_cast<unsigned*>(sm + NG * PL);
  for (int i = threadIdx.x; i < kHistBins; i += kThreads) sh[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(&qmap) : "memory");
    for (int q = 0; q < NG / 2; ++q) mbar_init(&s_bar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int g = threadIdx.x / G, t = threadIdx.x % G;
  float2* buf = sm + g * PL;
  const int y_lo = blockIdx.x * NG * kAmpRows, yend = min(H, y_lo + NG * kAmpRows);
  int it = 0;
  for (int yg = y_lo; yg < yend; yg += NG, ++it) {
    if (threadIdx.x == 0) {
      fence_proxy_async();                         // the previous group's buffers are free (barrier below)
      if constexpr (kAmpTile) {
        // whole 4-row tile rows (32 KB contiguous: one bulk copy, every byte used)
        for (int p = 0; p < NG / 4; ++p) {
          const int z = (b * F + o) * (c.Hp >> 2) + ((yg + 4 * p) >> 2);
          mbar_expect_tx(&s_bar[p], (uint32_t)(4 * W * sizeof(float2)));
          bulk_load(sm + 4 * p * PL, Q + (size_t)z * 4 * W, (uint32_t)(4 * W * sizeof(float2)), &s_bar[p]);
        }
      } else
      for (int p = 0; p < NG / 2; ++p) {
        const int y = yg + 2 * p;
        const int z = (b * F + o) * (c.Hp >> 2) + (y >> 2);
        mbar_expect_tx(&s_bar[p], (uint32_t)(2 * W * sizeof(float2)));
        for (int k = 0; k < W / kPcTmaBox; ++k)
          tma_load_3d(sm + 2 * p * PL + 2 * kPcTmaBox * k, &qmap, 2 * (y & 3), kPcTmaBox * k, z, &s_bar[p]);
      }
      if (yg + NG < yend) {                        // the next row group's Q tiles into L2
        l2_prefetch(Qp + (size_t)(yg + NG) * W, (unsigned)(NG * W * sizeof(float2)));
      } else if (ahead > 0) {                      // the first row group of the CTA `ahead` slots later
        const long long lin = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x + ahead;
        if (lin < (long long)gridDim.x * gridDim.y * gridDim.z) {
          const int nx = (int)(lin % gridDim.x), no = (int)((lin / gridDim.x) % gridDim.y);
          const int nbz = (int)(lin / ((long long)gridDim.x * gridDim.y));
          const int ny = nx * NG * kAmpRows;
          if (ny < H) l2_prefetch(Q + ((size_t)nbz * F + no) * c.Hp * W + (size_t)ny * W, (unsigned)(NG * W * sizeof(float2)));
        }
      }
    }
    constexpr int RT = kAmpTile ? 4 : 2;           // rows staged together
    mbar_wait(&s_bar[g / RT], (uint32_t)(it & 1));
    const int y = yg + g;
    const float2* st = sm + (g & ~(RT - 1)) * PL;  // [x][row] of the RT rows staged with this one
    float2 v[32];
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = cconj(st[RT * (t + 32 * m) + (g & (RT - 1))]);
    SyncNamed pair{8 + g / RT, RT * G};            // all rows read before the FFT reuses the staging
    pair();
    SyncWarp sw{0xffffffffu};
    fft_fast<G>(v, buf, c.tw_w, t, sw);
    if (y < yend) {
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const float2 zz = cconj(v[m]);
        const float a = sqrt_approx(fmaf(zz.x, zz.x, zz.y * zz.y));   // as k_rows_amp0
        if (write_r0) Rp[(size_t)y * W + t + G * m] = zz;   // not needed when K3b recomputes scale 0
#ifndef R2_EXP_NOAMP
        A[(size_t)y * W + t + G * m] = a;
#endif
#ifndef R2_EXP_NOHIST
        atomicAdd(&sh[__float_as_uint(a) >> 19], 1u);
#else
        if (a < 0.f) sh[0] = 1;                          // keep the amplitude live
#endif
      }
    }
    __syncthreads();                               // the next group's TMA rewrites the buffers
  }
  unsigned* gh = hist + ((size_t)b * c.O + o) * kHistBins;
  for (int i = threadIdx.x; i < kHistBins; i += kThreads)
    if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

// ------------------------------------------------------------------ K4 ---
// Exact median of each amp0 plane (ref: loggabor.py:222, np.median: mean of
// the two middle order statistics for even counts).
struct MedInfo {
  unsigned bin[2];     // level-1 bins of ranks (n-1)/2 and n/2
  unsigned rank[2];    // ranks inside those bins
  unsigned pre[2];     // after level 2: float bits >> 9
  unsigned rank2[2];   // ranks inside those level-2 bins
};

__device__ void block_exclusive_scan_1024(unsigned* data, int n, unsigned* tmp) {
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

// gather the float bits of every value falling into one of the two bins;
// hits are appended warp-aggregated into a per-CTA shared buffer and flushed
// with one global atomic per CTA pass (16 values per thread per pass)
constexpr int kCollectVec = 8;                  // float4 loads per thread per pass (mask: 32 values)
__global__ void __launch_bounds__(256) k_med_collect(const float* __restrict__ amp0, const MedInfo* __restrict__ info,
                                                     unsigned* __restrict__ cand, unsigned* __restrict__ cnt,
                                                     unsigned n) {
  __shared__ unsigned s_buf[kCollectVec * 4 * 256];
  __shared__ unsigned s_n, s_base;
  const int plane = blockIdx.y;
  const unsigned b0 = info[plane].bin[0], b1 = info[plane].bin[1];
  const unsigned lo_bits = (b0 < b1 ? b0 : b1) << 19;
  const unsigned rng_bits = ((b0 < b1 ? b1 - b0 : b0 - b1) + 1u) << 19;
  const float* Ap = amp0 + (size_t)plane * n;
  const float4* A = reinterpret_cast<const float4*>(Ap);
  unsigned* out = cand + (size_t)plane * n;
  const unsigned n4 = (n + 3) / 4;
  const bool vec = (n & 3) == 0;                  // plane starts 16-byte aligned
  const unsigned lane = threadIdx.x & 31;
  const unsigned per_pass = kCollectVec * blockDim.x;
  for (unsigned base = blockIdx.x * per_pass; base < n4; base += gridDim.x * per_pass) {
    if (threadIdx.x == 0) {
      s_n = 0;
      // this CTA's next pass streams into L2 while this one filters / writes
      const unsigned next = base + gridDim.x * per_pass;
      if (vec && next < n4) l2_prefetch(A + next, (n4 - next < per_pass ? n4 - next : per_pass) * 16u);
    }
    __syncthreads();
    float4 qv[kCollectVec];
    if (vec && base + per_pass <= n4) {
#pragma unroll
      for (int k = 0; k < kCollectVec; ++k) qv[k] = __ldg(&A[base + k * blockDim.x + threadIdx.x]);
    } else {
      // tail: padding bits 0xFFFFFFFF never fall in the bin range below
      const float pad = __uint_as_float(0xFFFFFFFFu);
#pragma unroll
      for (int k = 0; k < kCollectVec; ++k) {
        const unsigned i = base + k * blockDim.x + threadIdx.x;
        qv[k] = make_float4(pad, pad, pad, pad);
        if (vec && 4 * i + 3 < n) qv[k] = __ldg(&A[i]);
        else if (i < n4) {
          qv[k].x = Ap[4 * i];
          if (4 * i + 1 < n) qv[k].y = Ap[4 * i + 1];
          if (4 * i + 2 < n) qv[k].z = Ap[4 * i + 2];
          if (4 * i + 3 < n) qv[k].w = Ap[4 * i + 3];
        }
      }
    }
    // per-thread hit mask over its 32 values: one unsigned range test on the
    // float bits (bins b_lo..b_hi; bins between them are empty, so the range
    // holds exactly the values of the two bins), one warp prefix sum, one
    // shared atomic per warp, then each thread writes its own hits
    unsigned mask = 0;
#pragma unroll
    for (int k = 0; k < kCollectVec; ++k) {
      const float vals[4] = {qv[k].x, qv[k].y, qv[k].z, qv[k].w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        mask |= (__float_as_uint(vals[e]) - lo_bits < rng_bits ? 1u : 0u) << (4 * k + e);
    }
    const unsigned cntt = __popc(mask);
    unsigned incl = cntt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= (unsigned)d) incl += t;
    }
    const unsigned wtot = __shfl_sync(0xffffffffu, incl, 31);
    unsigned wbase = 0;
    if (lane == 31 && wtot) wbase = atomicAdd(&s_n, wtot);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    unsigned pos = wbase + incl - cntt;
    if (mask) {                                     // static indices: qv stays in registers
#pragma unroll
      for (int k = 0; k < kCollectVec; ++k) {
        if (!((mask >> (4 * k)) & 0xFu)) continue;  // ~3 % of values hit: most groups are empty
        const float vals[4] = {qv[k].x, qv[k].y, qv[k].z, qv[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if ((mask >> (4 * k + e)) & 1u) s_buf[pos++] = __float_as_uint(vals[e]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_n) s_base = atomicAdd(&cnt[plane], s_n);
    __syncthreads();
    for (unsigned j = threadIdx.x; j < s_n; j += blockDim.x) out[s_base + j] = s_buf[j];
    __syncthreads();
  }
}

// Levels 2 (float bits 18..9) and 3 (bits 8..0) of the radix select over
// the candidates, as histograms spread over kMedBlk CTAs per plane (the
// candidate count is data dependent: ~3 % of a plane, 0.5 M at 4096^2) with
// the bin picks in small per-plane steps.
constexpr int kMedBlk = 16;                      // minimum CTAs per plane
constexpr int kMedH = 2 * 1024;                  // global histogram words per plane (two ranks)

// the bin holding `rank` in a 256-thread block scan of hist[0..nbins)
__device__ void med_pick(const unsigned* __restrict__ hist, int nbins, unsigned rank, unsigned* s_out) {
  __shared__ unsigned s_w[8];
  const int t = threadIdx.x, per = nbins / 256;
  unsigned loc[4], sum = 0;
  for (int k = 0; k < per; ++k) { loc[k] = hist[t * per + k]; sum += loc[k]; }
  unsigned incl = sum;
  const unsigned lane = t & 31, w = t >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= (unsigned)d) incl += v;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  unsigned run = incl - sum;
  for (int k = 0; k < (int)w; ++k) run += s_w[k];
  for (int k = 0; k < per; ++k) {
    if (rank >= run && rank < run + loc[k]) { s_out[0] = t * per + k; s_out[1] = rank - run; }
    run += loc[k];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_med_h2(const unsigned* __restrict__ cand, const unsigned* __restrict__ cnt,
                                                const MedInfo* __restrict__ info, unsigned* __restrict__ gh,
                                                unsigned n) {
  __shared__ unsigned h[2][1024];
  const int plane = blockIdx.y;
  const unsigned c = cnt[plane];
  const unsigned b0 = info[plane].bin[0], b1 = info[plane].bin[1];
  const unsigned lo_bits = (b0 < b1 ? b0 : b1) << 19;
  const unsigned rng_bits = ((b0 < b1 ? b1 - b0 : b0 - b1) + 1u) << 19;
  const unsigned* cd = cand + (size_t)plane * n;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const unsigned bits = cd[i], hb = bits >> 19, lv = (bits >> 9) & 1023u;
    if (hb == b0) atomicAdd(&h[0][lv], 1u);
    if (b1 != b0 && hb == b1) atomicAdd(&h[1][lv], 1u);
  }
  __syncthreads();
  unsigned* g = gh + (size_t)plane * kMedH;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(&g[i], (&h[0][0])[i]);
}

// every CTA picks the level-2 bins (same result), CTA 0 records them; then
// the level-3 histograms of the candidates under those prefixes
__global__ void __launch_bounds__(256) k_med_h3(const unsigned* __restrict__ cand, const unsigned* __restrict__ cnt,
                                                MedInfo* __restrict__ info, const unsigned* __restrict__ gh2,
                                                unsigned* __restrict__ gh3, unsigned n) {
  __shared__ unsigned h[2][512];
  __shared__ unsigned s_pick[2];
  const int plane = blockIdx.y;
  const unsigned c = cnt[plane];
  const MedInfo inf = info[plane];
  const unsigned* g2 = gh2 + (size_t)plane * kMedH;
  unsigned pre[2], rk[2];
  for (int q = 0; q < 2; ++q) {
    med_pick(g2 + (inf.bin[1] != inf.bin[0] ? q * 1024 : 0), 1024, inf.rank[q], s_pick);
    pre[q] = (inf.bin[q] << 10) | s_pick[0];
    rk[q] = s_pick[1];
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[plane].pre[0] = pre[0]; info[plane].pre[1] = pre[1];
    info[plane].rank2[0] = rk[0]; info[plane].rank2[1] = rk[1];
  }
  const unsigned* cd = cand + (size_t)plane * n;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const unsigned bits = cd[i], p9 = bits >> 9;
    if (p9 == pre[0]) atomicAdd(&h[0][bits & 511u], 1u);
    if (pre[1] != pre[0] && p9 == pre[1]) atomicAdd(&h[1][bits & 511u], 1u);
  }
  __syncthreads();
  unsigned* g = gh3 + (size_t)plane * kMedH;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(&g[i], (&h[0][0])[i]);
}

// level-3 picks -> the two middle order statistics -> the noise threshold
__global__ void __launch_bounds__(256) k_med_final(const MedInfo* __restrict__ info, const unsigned* __restrict__ gh3,
                                                   float* __restrict__ thr, double thr_factor) {
  __shared__ unsigned s_pick[2];
  const int plane = blockIdx.x;
  const MedInfo inf = info[plane];
  const unsigned* g3 = gh3 + (size_t)plane * kMedH;
  double val[2];
  for (int q = 0; q < 2; ++q) {
    med_pick(g3 + (inf.pre[1] != inf.pre[0] ? q * 512 : 0), 512, inf.rank2[q], s_pick);
    val[q] = (double)__uint_as_float((inf.pre[q] << 9) | s_pick[0]);
    __syncthreads();
  }
  if (threadIdx.x == 0) thr[plane] = (float)(0.5 * (val[0] + val[1]) * thr_factor);
}

static void launch_med_select(const unsigned* cand, const unsigned* cnt, MedInfo* info, unsigned* gh, float* thr,
                              int planes, unsigned n, double factor, cudaStream_t st) {
  unsigned* gh2 = gh;
  unsigned* gh3 = gh + (size_t)planes * kMedH;
  cudaMemsetAsync(gh, 0, (size_t)planes * 2 * kMedH * sizeof(unsigned), st);
  const unsigned blk = std::min(256u, std::max((unsigned)kMedBlk, n >> 16));   // ~3 % of n are candidates
  k_med_h2<<<dim3(blk, planes), 256, 0, st>>>(cand, cnt, info, gh2, n);
  k_med_h3<<<dim3(blk, planes), 256, 0, st>>>(cand, cnt, info, gh2, gh3, n);
  k_med_final<<<planes, 256, 0, st>>>(info, gh3, thr, factor);
}

// ----------------------------------------------------------------- K3b ---
struct PcOut {
  float* mmax;
  float* mmin;
  uint8_t* mim;
  float* a_o;    // nullable [B][O][H][W]
  float* pc;     // nullable [B][O][H][W]
  float* amax;   // nullable [B][H][W]
  unsigned long long* range;   // nullable [B][2 maps: min, max][lo, hi] ordered float64 keys
};

// Per-image min / max of the two moment maps, folded into the PC pass so
// the detector's normalisation (ref: detector.py:80-84) needs no re-read of
// the maps: per-thread running extrema, a CTA reduction, four atomics per
// CTA on order-preserving keys of the float64 value (the detector's own key
// format; the maps are >= 0).
R2_DEV unsigned long long range_key(float v) {
  return (unsigned long long)__double_as_longlong((double)v) | 0x8000000000000000ull;
}
struct RangeAcc {
  float lo0 = INFINITY, hi0 = -INFINITY, lo1 = INFINITY, hi1 = -INFINITY;   // map 0 = moment_min, 1 = moment_max
  R2_DEV void add(float vmin, float vmax) {
    lo0 = fminf(lo0, vmin); hi0 = fmaxf(hi0, vmin);
    lo1 = fminf(lo1, vmax); hi1 = fmaxf(hi1, vmax);
  }
  // two pixels per call: three-input min / max (FMNMX3)
  R2_DEV void add2(float vmin0, float vmax0, float vmin1, float vmax1) {
    lo0 = fminf(fminf(lo0, vmin0), vmin1); hi0 = fmaxf(fmaxf(hi0, vmin0), vmin1);
    lo1 = fminf(fminf(lo1, vmax0), vmax1); hi1 = fmaxf(fmaxf(hi1, vmax0), vmax1);
  }
  // all threads of the CTA; range = this image's four keys
  R2_DEV void flush(unsigned long long* range) {
    __shared__ float s_r[4][32];
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      lo0 = fminf(lo0, __shfl_xor_sync(0xffffffffu, lo0, d));
      hi0 = fmaxf(hi0, __shfl_xor_sync(0xffffffffu, hi0, d));
      lo1 = fminf(lo1, __shfl_xor_sync(0xffffffffu, lo1, d));
      hi1 = fmaxf(hi1, __shfl_xor_sync(0xffffffffu, hi1, d));
    }
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { s_r[0][w] = lo0; s_r[1][w] = hi0; s_r[2][w] = lo1; s_r[3][w] = hi1; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < nw; ++q) {
        lo0 = fminf(lo0, s_r[0][q]); hi0 = fmaxf(hi0, s_r[1][q]);
        lo1 = fminf(lo1, s_r[2][q]); hi1 = fmaxf(hi1, s_r[3][q]);
      }
      if (lo0 <= hi0) { atomicMin(&range[0], range_key(lo0)); atomicMax(&range[1], range_key(hi0)); }
      if (lo1 <= hi1) { atomicMin(&range[2], range_key(lo1)); atomicMax(&range[3], range_key(hi1)); }
    }
  }
};

__global__ void k_range_init(unsigned long long* range, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) range[i] = (i & 1) ? 0ull : ~0ull;
}

template <int G>
struct PcShape {
  // CTA size: 2048- and 4096-point rows use 512 threads (four / eight FFT
  // groups), so a thread carries 8 pixels' accumulators next to its FFT
  // slice without spilling and the stage's transforms are balanced
  static constexpr int T = (G == 64 || G == 128) ? 512 : kThreads;
  // pixels per thread: a CTA holds (up to) two rows (one at 4096 points)
  static constexpr int PIX = G == 0 ? 16 : (G >= 64 ? 8 : (G >= 4 ? G / 4 : 1));
};

#ifndef R2_PC_PREFETCH
#define R2_PC_PREFETCH 1
#endif
constexpr bool kPcPrefetch = R2_PC_PREFETCH;
#ifndef R2_PC_TMA
#define R2_PC_TMA 1
#endif
constexpr bool kPcTma = R2_PC_TMA;   // K3b inputs by TMA for 1,024-point rows
#ifndef R2_COLS_TMA
#define R2_COLS_TMA 1
#endif
constexpr bool kColsTma = R2_COLS_TMA;   // K2 stores by TMA for columns of >= 1,024 rows

R2_DEV float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Phase congruency of two pixels at once in the fp32x2 lanes (SC scales,
// ref: loggabor.py:193-251): the FP work of the pixel phase in packed
// instructions; square roots, reciprocals and exp stay per lane (MUFU).  The
// weight and 1 / (sum of amplitudes) share one reciprocal:
// pc = en / ((1 + exp(g (cut - spread))) (sa + eps)).
template <int SC>
R2_DEV void pc_core(const float2 (&X)[SC], const float2 (&Y)[SC], float T, float inv_sm1, float gain, float cut,
                    float2& sa, float2& pc);

template <int SC>
R2_DEV void pc_pair(const float2* __restrict__ b0, const float2* __restrict__ b1, int PL, float T, float inv_sm1,
                    float gain, float cut, float2& sa, float2& pc) {
  float2 X[SC], Y[SC];
#pragma unroll
  for (int s = 0; s < SC; ++s) {
    const float2 z0 = b0[s * PL], z1 = b1[s * PL];
    X[s] = make_float2(z0.x, z1.x);
    Y[s] = make_float2(z0.y, z1.y);
  }
  pc_core<SC>(X, Y, T, inv_sm1, gain, cut, sa, pc);
}

template <int SC>
R2_DEV void pc_core(const float2 (&X)[SC], const float2 (&Y)[SC], float T, float inv_sm1, float gain, float cut,
                    float2& sa, float2& pc) {
  float2 se = make_float2(0.f, 0.f), so = se;
  sa = se;
  float mx0 = 0.f, mx1 = 0.f;
#pragma unroll
  for (int s = 0; s < SC; ++s) {
    const float2 q = __ffma2_rn(X[s], X[s], __fmul2_rn(Y[s], Y[s]));
    const float2 a = make_float2(sqrt_approx(q.x), sqrt_approx(q.y));
    se = __fadd2_rn(se, X[s]);
    so = __fadd2_rn(so, Y[s]);
    sa = __fadd2_rn(sa, a);
    mx0 = fmaxf(mx0, a.x);
    mx1 = fmaxf(mx1, a.y);
  }
  const float2 q = __ffma2_rn(se, se, __fmul2_rn(so, so));
  const float2 ixe = make_float2(rcp_approx(sqrt_approx(q.x) + 1e-4f), rcp_approx(sqrt_approx(q.y) + 1e-4f));
  const float2 me = __fmul2_rn(se, ixe), mo = __fmul2_rn(so, ixe);
  const float2 nme = make_float2(-me.x, -me.y);
  // sum_s z_s . m = |S|^2 / (|S| + eps) = q * ixe: only the cross terms are per scale
  float2 en = __fmul2_rn(q, ixe);
#pragma unroll
  for (int s = 0; s < SC; ++s) {
    const float2 t2 = __ffma2_rn(X[s], mo, __fmul2_rn(Y[s], nme));
    en = make_float2(en.x - fabsf(t2.x), en.y - fabsf(t2.y));
  }
  en = make_float2(fmaxf(en.x - T, 0.f), fmaxf(en.y - T, 0.f));
  const float sp0 = fmaf(sa.x, rcp_approx(mx0 + 1e-4f), -1.f) * inv_sm1;
  const float sp1 = fmaf(sa.y, rcp_approx(mx1 + 1e-4f), -1.f) * inv_sm1;
  const float g2 = gain * 1.4426950408889634f;      // exp(x) = 2^(x log2 e): one MUFU, no range fix-up
  const float e0 = ex2(g2 * (cut - sp0)), e1 = ex2(g2 * (cut - sp1));
  pc = make_float2(en.x * rcp_approx((1.f + e0) * (sa.x + 1e-4f)), en.y * rcp_approx((1.f + e1) * (sa.y + 1e-4f)));
}

// One CTA per row pair (y0, y0+1).  Stage = `ops` orientations of `rr` rows;
// its buffers (row, orientation, scale) are filled by FFT jobs (scales >= 1)
// and plain loads of the K3a responses (scale 0), then the per-pixel phase
// congruency (ref: loggabor.py:193-251) consumes them.  SC > 0 fixes the
// scale count at compile time (the BASELINE / reference default is 4).
// Approximate sqrt / rcp / exp (relative error ~1e-7) stay far inside the
// 1e-4 map tolerance.
template <int G, int SC>
__global__ void __launch_bounds__(PcShape<G>::T, PcShape<G>::T == 512 ? 1 : 2) k_rows_pc(const float2* __restrict__ Q, const float2* __restrict__ R0,
                                                         const float* __restrict__ thr, PcOut out,
                                                         const __grid_constant__ FieldsConst c, int rr, int ops,
                                                         int ahead) {
  extern __shared__ float2 sm[];
  constexpr int SMAX = SC > 0 ? SC : kMaxS;
  const int H = c.H, O = c.O;
  const int W = G > 0 ? 32 * G : c.W;
  const int S = SC > 0 ? SC : c.S;
  const int F = S * O;
  const int b = blockIdx.y;
  const int y0 = 2 * blockIdx.x;
  constexpr int PIX = PcShape<G>::PIX;
  constexpr int TPC = PcShape<G>::T;
  const int PL = padded_len(W);
  const int nb = rr * ops * S;
  const float* thr_b = thr + (size_t)b * O;
  const float2* Qb = Q + (size_t)b * F * c.Hp * W;
  const float2* Rb = R0 + (size_t)b * O * H * W;
  const float inv_sm1 = c.inv_sm1, gain = c.spread_gain, cut = c.spread_cutoff;

  RangeAcc racc;
  for (int rbase = 0; rbase < 2; rbase += rr) {
    const int npix = rr * W;
    float acc_a[PIX], acc_b[PIX], acc_c[PIX], best[PIX];
    int bidx[PIX];
#pragma unroll
    for (int i = 0; i < PIX; ++i) { acc_a[i] = acc_b[i] = acc_c[i] = 0.f; best[i] = -1.f; bidx[i] = 1; }
    for (int o0 = 0; o0 < O; o0 += ops) {
      const int no = min(ops, O - o0);
      // prefetch the next stage's inputs into L2 while this stage runs: its
      // Q row tiles (4 rows x W, contiguous) and R0 rows.  After the last
      // stage comes the first stage of the CTA `ahead` positions later in
      // launch order -- about the one that takes a slot when this CTA ends
      // (L2 is shared, so which SM runs it does not matter)
      if (G > 0 && kPcPrefetch && threadIdx.x == 0) {
        int pb = b, py = y0 + rbase, o1 = o0 + ops;
        bool go = o1 < O;
        if (!go && rbase + rr < 2 && y0 + rbase + rr < H) { py = y0 + rbase + rr; o1 = 0; go = true; }
        else if (!go && rbase + rr >= 2) {
          const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + ahead;
          if (ahead > 0 && lin < (long long)gridDim.x * gridDim.y) {
            pb = (int)(lin / gridDim.x);
            py = 2 * (int)(lin % gridDim.x);
            o1 = 0;
            go = py < H;
          }
        }
        if (go) {
          const int n1 = min(ops, O - o1);
          const float2* pQ = Q + (size_t)pb * F * c.Hp * W;
          const float2* pR = R0 + (size_t)pb * O * H * W;
          for (int r = 0; r < rr; r += kQT - ((py + r) & (kQT - 1))) {
            const int y = py + r;
            if (y >= H) break;
            for (int oo = 0; oo < n1; ++oo)
              for (int s = 1; s < S; ++s)
                l2_prefetch(pQ + ((size_t)(s * O + o1 + oo) * c.Hp + (y & ~(kQT - 1))) * W,
                            (unsigned)(kQT * W * sizeof(float2)));
          }
          for (int oo = 0; oo < n1; ++oo)
            l2_prefetch(pR + ((size_t)(o1 + oo) * H + py) * W, (unsigned)(min(rr, H - py) * W * sizeof(float2)));
        }
      }
      if constexpr (G > 0) {
        constexpr int NG = TPC / G;
        const int g = threadIdx.x / G, t = threadIdx.x % G;
        SyncWarp sw{group_mask(G)};
        SyncNamed sn{1 + g, G};
        for (int j = g; j < nb; j += NG) {
          const int r = j / (ops * S), rem = j % (ops * S), oo = rem / S, s = rem % S;
          const int y = y0 + rbase + r;
          float2* buf = sm + j * PL;
          if (oo >= no || y >= H) continue;
          const int o = o0 + oo;
          if (s == 0) {
            const float2* Rp = Rb + ((size_t)o * H + y) * W;
            float2 v[32];
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = Rp[t + G * m];
#pragma unroll
            for (int m = 0; m < 32; ++m) buf[pad32(t + G * m)] = v[m];
          } else {
            const float2* Qp = Qb + (size_t)(s * O + o) * c.Hp * W;
            float2 v[32];
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = cconj(Qp[tq(y, t + G * m, W)]);
            if constexpr (G <= 32) fft_fast<G>(v, buf, c.tw_w, t, sw); else fft_fast<G>(v, buf, c.tw_w, t, sn);
            if constexpr (G <= 32) sw(); else sn();
#pragma unroll
            for (int m = 0; m < 32; ++m) buf[pad32(t + G * m)] = cconj(v[m]);
          }
        }
      } else {
        float2* scr = sm + nb * PL;
        for (int j = 0; j < nb; ++j) {
          const int oo = j / S, s = j % S;
          const int y = y0 + rbase;
          if (oo >= no || y >= H) break;
          const int o = o0 + oo;
          float2* buf = sm + j * PL;
          if (s == 0) {
            const float2* Rp = Rb + ((size_t)o * H + y) * W;
            for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = Rp[x];
          } else {
            const float2* Qp = Qb + (size_t)(s * O + o) * c.Hp * W;
            for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(Qp[tq(y, x, W)]);
            __syncthreads();
            fft_generic(buf, scr, W, c.plan_w, c.tw_w, threadIdx.x, blockDim.x);
            for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(buf[pad32(x)]);
          }
        }
      }
      __syncthreads();
      // --- per-pixel phase congruency for the orientations of this stage
      for (int oo = 0; oo < no; ++oo) {
        const int o = o0 + oo;
        const float T = thr_b[o], ca = c.cos_a[o], sa_o = c.sin_a[o];
        if constexpr (SC > 0 && PIX % 2 == 0) {
          // pixel pairs (i, i + 1) in the fp32x2 lanes when both are live
          // (warp-uniform: npix is a multiple of TPC for these sizes)
          if (npix == PIX * TPC && y0 + rbase + rr <= H) {
#pragma unroll
            for (int i = 0; i < PIX; i += 2) {
              const int p0 = threadIdx.x + TPC * i, p1 = p0 + TPC;
              const int r0 = p0 / W, x0 = p0 % W, r1 = p1 / W, x1 = p1 % W;
              const float2* b0 = sm + ((r0 * ops + oo) * S) * PL + pad32(x0);
              const float2* b1 = sm + ((r1 * ops + oo) * S) * PL + pad32(x1);
              float2 sa2, pc2;
              pc_pair<SC>(b0, b1, PL, T, inv_sm1, gain, cut, sa2, pc2);
              const float2 pcc = __fmul2_rn(pc2, make_float2(ca, ca)), pcs = __fmul2_rn(pc2, make_float2(sa_o, sa_o));
              acc_a[i] = fmaf(pcc.x, pcc.x, acc_a[i]);
              acc_a[i + 1] = fmaf(pcc.y, pcc.y, acc_a[i + 1]);
              acc_b[i] = fmaf(pcc.x, pcs.x, acc_b[i]);
              acc_b[i + 1] = fmaf(pcc.y, pcs.y, acc_b[i + 1]);
              acc_c[i] = fmaf(pcs.x, pcs.x, acc_c[i]);
              acc_c[i + 1] = fmaf(pcs.y, pcs.y, acc_c[i + 1]);
              if (sa2.x > best[i]) { best[i] = sa2.x; bidx[i] = o + 1; }
              if (sa2.y > best[i + 1]) { best[i + 1] = sa2.y; bidx[i + 1] = o + 1; }
              if (out.a_o || out.pc) {
                const size_t q0 = (((size_t)b * O + o) * H + y0 + rbase + r0) * W + x0;
                const size_t q1 = (((size_t)b * O + o) * H + y0 + rbase + r1) * W + x1;
                if (out.a_o) { out.a_o[q0] = sa2.x; out.a_o[q1] = sa2.y; }
                if (out.pc) { out.pc[q0] = pc2.x; out.pc[q1] = pc2.y; }
              }
            }
            continue;
          }
        }
#pragma unroll
        for (int i = 0; i < PIX; ++i) {
          const int p = threadIdx.x + TPC * i;
          if (p >= npix) continue;
          const int r = p / W, x = p % W;
          const int y = y0 + rbase + r;
          if (y >= H) continue;
          const float2* bb = sm + ((r * ops + oo) * S) * PL + pad32(x);
          float2 z[SMAX];
          float se = 0.f, so = 0.f, sa = 0.f, mx = 0.f;
#pragma unroll
          for (int s = 0; s < SMAX; ++s) {
            if (SC > 0 || s < S) {
              z[s] = bb[s * PL];
              const float a = sqrt_approx(fmaf(z[s].x, z[s].x, z[s].y * z[s].y));
              se += z[s].x; so += z[s].y; sa += a; mx = fmaxf(mx, a);
            }
          }
          const float qe = fmaf(se, se, so * so);
          const float ixe = rcp_approx(sqrt_approx(qe) + 1e-4f);
          const float me = se * ixe, mo = so * ixe;
          // sum_s z_s . m = |S|^2 / (|S| + eps): only the cross terms are per scale
          float en = qe * ixe;
#pragma unroll
          for (int s = 0; s < SMAX; ++s)
            if (SC > 0 || s < S) en -= fabsf(fmaf(z[s].x, mo, -z[s].y * me));
          en = fmaxf(en - T, 0.f);
          const float spread = fmaf(sa, rcp_approx(mx + 1e-4f), -1.f) * inv_sm1;
          const float wgt = rcp_approx(1.f + __expf(gain * (cut - spread)));
          const float pc = wgt * en * rcp_approx(sa + 1e-4f);
          const float pcc = pc * ca, pcs = pc * sa_o;
          acc_a[i] = fmaf(pcc, pcc, acc_a[i]);
          acc_b[i] = fmaf(pcc, pcs, acc_b[i]);
          acc_c[i] = fmaf(pcs, pcs, acc_c[i]);
          if (sa > best[i]) { best[i] = sa; bidx[i] = o + 1; }
          if (out.a_o || out.pc) {
            const size_t po = (((size_t)b * O + o) * H + y) * W + x;
            if (out.a_o) out.a_o[po] = sa;
            if (out.pc) out.pc[po] = pc;
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < PIX; ++i) {
      const int p = threadIdx.x + TPC * i;
      if (p >= npix) continue;
      const int r = p / W, x = p % W;
      const int y = y0 + rbase + r;
      if (y >= H) continue;
      const float a = acc_a[i], bq = 2.f * acc_b[i], cq = acc_c[i];
      const float root = sqrtf(bq * bq + (a - cq) * (a - cq));
      const size_t po = ((size_t)b * H + y) * W + x;
      const float vmax = 0.5f * (cq + a + root), vmin = fmaxf(0.5f * (cq + a - root), 0.f);
      out.mmax[po] = vmax;
      out.mmin[po] = vmin;
      out.mim[po] = (uint8_t)bidx[i];
      if (out.amax) out.amax[po] = best[i];
      if (out.range) racc.add(vmin, vmax);
    }
  }
  if (out.range) racc.flush(out.range + 4 * (size_t)b);
}


// K3b for 1,024-point rows with 4 scales (the BASELINE path), inputs by TMA.
// One CTA per row pair (y0, y0+1): each orientation stage's inputs arrive in
// shared memory by the tensor-memory accelerator -- the two rows of every
// scale as 3-D boxes {2 rows of a 4-row column tile, 256 columns} (the rows
// the CTA needs, gathered without load instructions), one mbarrier per
// scale -- and all eight warps run one row FFT each: scale 0 is transformed
// here again rather than read back from K3a, so K3a writes no R0 plane (1.6
// GB per 32 images) and no warp idles in the FFT phase.  Buffers: scale s,
// row r at s*R + r (a scale's rows are contiguous: the staging of its boxes
// as [x][row]); after its FFT a warp leaves its row there as a real and an
// imaginary plane.  The pixel phase first moves all of a thread's operands
// (4 pixel pairs x 4 scales) into registers; one barrier later the buffers
// are free, so the next stage's loads are issued *before* the pixel
// arithmetic and land while it runs (kPcEarly) instead of after it.
// Same arithmetic as k_rows_pc, and bit-identical scale-0 amplitudes (same
// FFT, same input).
#ifndef R2_PC_DIST
#define R2_PC_DIST 1
#endif
constexpr int kPcDist = R2_PC_DIST;   // L2 prefetch distance in stages (0: none)
#ifndef R2_PC_EARLY
#define R2_PC_EARLY 1
#endif
constexpr bool kPcEarly = R2_PC_EARLY;
#ifndef R2_PC_ROWS
#define R2_PC_ROWS 2
#endif
constexpr int kPcRows = R2_PC_ROWS;   // rows per CTA: 2 (two CTAs per SM) or 4 (whole column tiles, one CTA per SM)
// Instances: 1,024-point rows with R = 2 (two CTAs per SM; R = 4 measured
// slower: one CTA per SM runs its two phases in lockstep) and 512-point rows
// with R = 4 (whole tiles, 16 half-warp FFTs).
template <int R, int W>
__global__ void __launch_bounds__(4 * R * (W / 32), R * W == 2048 ? 2 : 1) k_rows_pc_tma(const __grid_constant__ CUtensorMap qmap,
                                                             const float2* __restrict__ Q,
                                                             const float* __restrict__ thr, PcOut out,
                                                             const __grid_constant__ FieldsConst c, int ahead) {
  // buffer pitch rounded to 128 bytes: TMA destinations must be 128-byte aligned
  constexpr int G = W / 32, S = 4, PL = (padded_len(W) + 15) & ~15, PIX = 8, NP = PIX / 2;
  constexpr int T = S * R * G;                    // G threads per (scale, row)
  static_assert(R * W == PIX * T, "8 pixels per thread");
  // plane offset of odd rows (floats, inside the pitch slack): two 16-thread
  // groups of one warp then store to different banks
  constexpr int POFF = G < 32 ? 16 : 0;
  static_assert(2 * W + POFF <= 2 * PL, "planes fit the buffer");
  extern __shared__ float2 sm_raw[];
  __shared__ uint64_t s_bar[4];                   // one per scale: its FFT warps start on their own rows
  float2* sm = reinterpret_cast<float2*>(reinterpret_cast<char*>(sm_raw) + ((128u - (smem_u32(sm_raw) & 127u)) & 127u));
  const int H = c.H, O = c.O, F = S * O;
  const int b = blockIdx.y, y0 = R * blockIdx.x;
  const float* thr_b = thr + (size_t)b * O;
  const float inv_sm1 = c.inv_sm1, gain = c.spread_gain, cut = c.spread_cutoff;
  const int g = threadIdx.x / G, t = threadIdx.x % G;
  // (thread 0) stage o: the CTA's rows of every scale into the buffers as
  // [x][row] -- W / 256 boxes of two rows, or the whole 4-row tile row
  // (contiguous: one bulk copy) -- and stage o + kPcDist (past the last stage:
  // that stage of the CTA one resident wave later) into L2
  auto issue_stage = [&](int o) {
#ifndef R2_EXP_NOLOAD                              // timing experiment: compute on stale shared memory
    fence_proxy_async();                           // earlier generic accesses of the buffers precede the async writes
    for (int s = 0; s < S; ++s) {
      const int z = (b * F + s * O + o) * (c.Hp >> 2) + (y0 >> 2);
      float2* dst = sm + s * R * PL;
      mbar_expect_tx(&s_bar[s], (uint32_t)(R * W * sizeof(float2)));
      if constexpr (R == 4) {
        bulk_load(dst, Q + (size_t)z * 4 * W, (uint32_t)(4 * W * sizeof(float2)), &s_bar[s]);
      } else {
        for (int k = 0; k < W / kPcTmaBox; ++k)
          tma_load_3d(dst + 2 * kPcTmaBox * k, &qmap, 2 * (y0 & 3), kPcTmaBox * k, z, &s_bar[s]);
      }
    }
#endif
    int pb = b, py = y0, o1 = o + kPcDist;
    bool go = o1 < O;
    if (!go && ahead > 0) {
      const long long lin = (long long)blockIdx.y * gridDim.x + blockIdx.x + ahead;
      if (lin < (long long)gridDim.x * gridDim.y) { pb = (int)(lin / gridDim.x); py = R * (int)(lin % gridDim.x); o1 -= O; go = true; }
    }
    if (go && kPcDist > 0) {
      const float2* pQ = Q + (size_t)pb * F * c.Hp * W;
      for (int s = 0; s < S; ++s)
        l2_prefetch(pQ + ((size_t)(s * O + o1) * c.Hp + (py & ~3)) * W, (unsigned)(4 * W * sizeof(float2)));
    }
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(&qmap) : "memory");
    for (int q = 0; q < 4; ++q) mbar_init(&s_bar[q], 1);
    mbar_fence_init();
    if (kPcEarly) issue_stage(0);
  }
  __syncthreads();
  float2 acc_a[NP], acc_b[NP], acc_c[NP], best[NP];
  int bidx[PIX];
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    acc_a[j] = acc_b[j] = acc_c[j] = make_float2(0.f, 0.f);
    best[j] = make_float2(-1.f, -1.f);
    bidx[2 * j] = bidx[2 * j + 1] = 1;
  }
  for (int o = 0; o < O; ++o) {
    // (late issue: the previous stage's pixel phase is done with the buffers,
    // the barrier at the end of the loop)
    if (!kPcEarly && threadIdx.x == 0) issue_stage(o);
    {                                              // 4 R FFT warps: scale g / R (0 included), row g % R
      const int s = g / R, r = g % R;
#ifndef R2_EXP_NOLOAD
      mbar_wait(&s_bar[s], (uint32_t)(o & 1));
#endif
      const float2* st = sm + s * R * PL;          // [x][row]
      float2 v[32];
#pragma unroll
      for (int m = 0; m < 32; ++m) v[m] = cconj(st[R * (t + G * m) + r]);
      SyncNamed grp{8 + s, R * G};                 // all rows read before the buffers are reused
      grp();
      float2* buf = sm + (s * R + r) * PL;
      SyncWarp sw{group_mask(G)};
      fft_fast<G>(v, buf, c.tw_w, t, sw);
      sw();
      // the row as two planes, real [W] then imaginary [W], so the pixel
      // phase loads two adjacent pixels' parts as one packed operand.  v is
      // the conjugate of the response (the inverse is conj FFT conj): left
      // as it is -- flipping the sign of every scale's odd part changes
      // neither the amplitudes nor |z x mean| nor z . mean
      float* pre = reinterpret_cast<float*>(buf) + (r & 1) * POFF;
#pragma unroll
      for (int m = 0; m < 32; ++m) { pre[t + G * m] = v[m].x; pre[W + t + G * m] = v[m].y; }
    }
    __syncthreads();
    // pixel phase: the thread's four pairs of adjacent pixels (pair j at
    // linear pixel 2 tid + 2 T j of the CTA's R rows) in the fp32x2 lanes
    const float T_o = thr_b[o], ca = c.cos_a[o], sa_o = c.sin_a[o];
    const float* pl = reinterpret_cast<const float*>(sm) + 2 * threadIdx.x;
    float2 X[NP][S], Y[NP][S];
    auto load_pair = [&](int j) {
      const int r = (2 * T * j) / W, x = (2 * T * j) % W;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const float* q = pl + (s * R + r) * (2 * PL) + (r & 1) * POFF + x;
        X[j][s] = *reinterpret_cast<const float2*>(q);
        Y[j][s] = *reinterpret_cast<const float2*>(q + W);
      }
    };
    if (kPcEarly) {
#pragma unroll
      for (int j = 0; j < NP; ++j) load_pair(j);
      __syncthreads();                             // every operand is in registers: the buffers are free
      if (threadIdx.x == 0 && o + 1 < O) issue_stage(o + 1);
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int r = (2 * T * j) / W, x = (2 * T * j) % W;
      if (!kPcEarly) load_pair(j);
      float2 sa2, pc2;
      pc_core<S>(X[j], Y[j], T_o, inv_sm1, gain, cut, sa2, pc2);
      const float2 pcc = __fmul2_rn(pc2, make_float2(ca, ca)), pcs = __fmul2_rn(pc2, make_float2(sa_o, sa_o));
      acc_a[j] = __ffma2_rn(pcc, pcc, acc_a[j]);
      acc_b[j] = __ffma2_rn(pcc, pcs, acc_b[j]);
      acc_c[j] = __ffma2_rn(pcs, pcs, acc_c[j]);
      if (sa2.x > best[j].x) { best[j].x = sa2.x; bidx[2 * j] = o + 1; }
      if (sa2.y > best[j].y) { best[j].y = sa2.y; bidx[2 * j + 1] = o + 1; }
      if (out.a_o || out.pc) {
        const size_t q0 = (((size_t)b * O + o) * H + y0 + r) * W + 2 * threadIdx.x + x;
        if (out.a_o) *reinterpret_cast<float2*>(out.a_o + q0) = sa2;
        if (out.pc) *reinterpret_cast<float2*>(out.pc + q0) = pc2;
      }
    }
    if (!kPcEarly) __syncthreads();                // the next stage's TMA rewrites the buffers
  }
  RangeAcc racc;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int r = (2 * T * j) / W, x = 2 * threadIdx.x + (2 * T * j) % W;
    const size_t po = ((size_t)b * H + y0 + r) * W + x;
    const float2 a = acc_a[j], bq = __fadd2_rn(acc_b[j], acc_b[j]), cq = acc_c[j];
    const float2 d = __fadd2_rn(a, make_float2(-cq.x, -cq.y)), sm2 = __fadd2_rn(a, cq);
    const float2 rr = __ffma2_rn(bq, bq, __fmul2_rn(d, d));
    const float root0 = sqrtf(rr.x), root1 = sqrtf(rr.y);
    const float2 vmax = make_float2(0.5f * (sm2.x + root0), 0.5f * (sm2.y + root1));
    const float2 vmin = make_float2(fmaxf(0.5f * (sm2.x - root0), 0.f), fmaxf(0.5f * (sm2.y - root1), 0.f));
    *reinterpret_cast<float2*>(out.mmax + po) = vmax;
    *reinterpret_cast<float2*>(out.mmin + po) = vmin;
    *reinterpret_cast<uchar2*>(out.mim + po) = make_uchar2((uint8_t)bidx[2 * j], (uint8_t)bidx[2 * j + 1]);
    if (out.amax) *reinterpret_cast<float2*>(out.amax + po) = best[j];
    if (out.range) racc.add2(vmin.x, vmax.x, vmin.y, vmax.y);
  }
  if (out.range) racc.flush(out.range + 4 * (size_t)b);   // CTA-uniform
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
      p.radix[p.n_pass++] = r;
      m /= r;
    }
  }
  // any remaining prime factors: runtime-radix passes (generic_pass_any)
  for (int r = 7; m > 1 && r * r <= m; r += 2) {
    while (m % r == 0 && p.n_pass < 16) {
      p.radix[p.n_pass++] = r;
      m /= r;
    }
  }
  if (m > 1 && p.n_pass < 16) {
    p.radix[p.n_pass++] = m;
    m = 1;
  }
  return m == 1;
}

struct FieldsPlan {
  int B, H, W, Wh, Hp, S, O, F;
  int gw, gh;
  size_t off_P, off_Q, off_R0, off_amp0, off_hist, off_info, off_cand, off_cnt, off_mh, off_thr, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static FieldsPlan plan_fields(int B, int H, int W, int S, int O) {
  FieldsPlan p{};
  p.B = B; p.H = H; p.W = W; p.Wh = W / 2 + 1; p.Hp = (H + 3) & ~3; p.S = S; p.O = O; p.F = S * O;
  p.gw = fast_g(W); p.gh = fast_g(H);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
  const size_t n = (size_t)H * W;
  p.off_P = take((size_t)B * H * p.Wh * sizeof(float2));
  p.off_Q = take((size_t)B * p.F * p.Hp * W * sizeof(float2));
  p.off_R0 = take((size_t)B * O * n * sizeof(float2));
  p.off_amp0 = take((size_t)B * O * n * sizeof(float));
  p.off_hist = take((size_t)B * O * kHistBins * sizeof(unsigned));
  p.off_info = take((size_t)B * O * sizeof(MedInfo));
  p.off_cand = take((size_t)B * O * n * sizeof(unsigned));
  p.off_cnt = take((size_t)B * O * sizeof(unsigned));
  p.off_mh = take((size_t)B * O * 2 * kMedH * sizeof(unsigned));
  p.off_thr = take((size_t)B * O * sizeof(float));
  p.total = off;
  return p;
}

size_t fields_workspace_bytes(int B, int H, int W, int S, int O) {
  return plan_fields(B, H, W, S, O).total;
}

template <class K>
static cudaError_t set_smem(K kern, size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  return e;
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
  return cudaPeekAtLastError();
}

template <int G>
static cudaError_t launch_cols(const float2* P, float2* Q, const FieldsConst& c, cudaStream_t st) {
  size_t smem;
  dim3 grid;
  CUtensorMap map{};
  int use_tma = 0;
  if constexpr (G > 0) {
    const int N = 32 * G, NG = ColsCfg<G>::T / G, CG = NG / 2, PL = padded_len(N), PLA = (PL + 15) & ~15;
    smem = ((size_t)CG * PL + (size_t)NG * PLA) * sizeof(float2) + 2 * (size_t)CG * N * sizeof(float) + 128;
    grid = dim3((c.Wh + CG - 1) / CG, c.B);
    if constexpr (G >= 16) {
      // columns of >= 512 rows leave by TMA: Q as 32-bit words (4 rows x 2
      // components, x, tile of all planes); a box is one column, 256 tiles
      // (128: the whole 512-row column)
      auto enc = get_encode();
      if (kColsTma && enc && ((uintptr_t)Q & 15) == 0 && c.Hp == N) {
        cuuint64_t dims[3] = {8, (cuuint64_t)c.W, (cuuint64_t)c.B * c.S * c.O * (c.Hp / 4)};
        cuuint64_t strides[2] = {4 * sizeof(float2), (cuuint64_t)c.W * 4 * sizeof(float2)};
        cuuint32_t box[3] = {8, 1, (cuuint32_t)(N >= 1024 ? 256 : N / 4)};
        cuuint32_t es[3] = {1, 1, 1};
        use_tma = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, Q, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      }
    }
  } else {
    const int PL = padded_len(c.H);
    smem = (size_t)(4 * PL + 2 * PL) * sizeof(float2) + 128;
    grid = dim3((c.Wh + 3) / 4, c.B);
  }
  cudaError_t e = set_smem(k_cols<G>, smem);
  if (e != cudaSuccess) return e;
  k_cols<G><<<grid, ColsCfg<G>::T, smem, st>>>(map, P, Q, c, use_tma);
  return cudaPeekAtLastError();
}

static bool pc_tma_applies(const float2* Q, const FieldsConst& c);
static bool launch_amp0_tma(const float2* Q, float2* R0, float* amp0, unsigned* hist, const FieldsConst& c,
                            cudaStream_t st, cudaError_t& e);

template <int G>
static cudaError_t launch_amp0(const float2* Q, float2* R0, float* amp0, unsigned* hist, const FieldsConst& c,
                               cudaStream_t st) {
  if constexpr (G == 32) {
    cudaError_t e = cudaSuccess;
    if (launch_amp0_tma(Q, R0, amp0, hist, c, st, e)) return e;
  }
  size_t smem;
  dim3 grid;
  if constexpr (G > 0) {
    const int NG = kThreads / G;
    smem = (size_t)NG * padded_len(32 * G) * sizeof(float2) + kHistBins * sizeof(unsigned);
    grid = dim3((c.H + NG * kAmpRows - 1) / (NG * kAmpRows), c.O, c.B);
  } else {
    smem = (size_t)2 * padded_len(c.W) * sizeof(float2) + kHistBins * sizeof(unsigned);
    grid = dim3(c.H, c.O, c.B);
  }
  cudaError_t e = set_smem(k_rows_amp0<G>, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, n_sm = 0;                // resident CTA slots: the prefetch look-ahead
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows_amp0<G>, kThreads, smem);
  k_rows_amp0<G><<<grid, kThreads, smem, st>>>(Q, R0, amp0, hist, c, per_sm * n_sm,
                                               (G > 0 && pc_tma_applies(Q, c)) ? 0 : 1);
  return cudaPeekAtLastError();
}

template <int G, int SC>
static cudaError_t launch_pc_s(const float2* Q, const float2* R0, const float* thr, const PcOut& out,
                               const FieldsConst& c, cudaStream_t st) {
  const size_t PLb = padded_len(c.W) * sizeof(float2);
  const size_t budget = 200 * 1024;
  int rr, ops;
  size_t nbuf;
  if constexpr (G > 0) {
    const int NG = PcShape<G>::T / G;
    rr = (2 * c.S * PLb <= budget) ? 2 : 1;
    ops = NG / (rr * c.S);
    if (ops < 1) ops = 1;
    if (ops > c.O) ops = c.O;
    while (ops > 1 && (size_t)rr * ops * c.S * PLb > budget) --ops;
    nbuf = (size_t)rr * ops * c.S;
  } else {
    rr = 1; ops = 1;
    nbuf = c.S + 1;
  }
  const size_t smem = nbuf * PLb;
  cudaError_t e = set_smem(k_rows_pc<G, SC>, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((c.H + 1) / 2, c.B);
  int per_sm = 0, dev = 0, n_sm = 0;                // resident CTA slots: the prefetch look-ahead
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows_pc<G, SC>, PcShape<G>::T, smem);
  k_rows_pc<G, SC><<<grid, PcShape<G>::T, smem, st>>>(Q, R0, thr, out, c, rr, ops, per_sm * n_sm);
  return cudaPeekAtLastError();
}

// Q (4-row column tiles of 1,024-wide planes) as a 3-D tensor of 32-bit words:
// (component of the row-in-tile, x, tile of all planes); a box of 4 words =
// the two rows y0, y0+1 of one column
static bool make_qmap(const float2* Q, const FieldsConst& c, CUtensorMap& map) {
  if (!kPcTma || c.W != 1024 || (c.Hp & 3) || ((uintptr_t)Q & 15)) return false;
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {8, (cuuint64_t)c.W, (cuuint64_t)c.B * c.S * c.O * (c.Hp / 4)};
  cuuint64_t strides[2] = {4 * sizeof(float2), (cuuint64_t)c.W * 4 * sizeof(float2)};
  cuuint32_t box[3] = {4, (cuuint32_t)kPcTmaBox, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<float2*>(Q), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int resident_ctas(const void* kern, int threads, size_t smem) {
  int per_sm = 0, dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  return per_sm * n_sm;
}

// whether K3b runs as k_rows_pc_tma (which recomputes scale 0, so K3a may skip R0):
// 1,024-point rows (2-row boxes through the tensor map) or 512-point rows
// (whole tile rows by bulk copies), 4 scales, two-pixel vector stores
static bool pc_tma_applies(const float2* Q, const FieldsConst& c) {
  if (!kPcTma || c.S != 4 || !c.out_vec || ((uintptr_t)Q & 15)) return false;
  if (c.W == 512) return c.H % 4 == 0;
  CUtensorMap map{};
  return c.W == 1024 && !(c.H & 1) && make_qmap(Q, c, map);
}

template <int R, int W>
static cudaError_t launch_pc_tma_rw(const CUtensorMap& map, const float2* Q, const float* thr, const PcOut& out,
                                    const FieldsConst& c, cudaStream_t st) {
  constexpr int T = 4 * R * (W / 32);
  const size_t smem = (size_t)4 * R * ((padded_len(W) + 15) & ~15) * sizeof(float2) + 128;
  cudaError_t e = set_smem(k_rows_pc_tma<R, W>, smem);
  if (e != cudaSuccess) return e;
  k_rows_pc_tma<R, W><<<dim3(c.H / R, c.B), T, smem, st>>>(map, Q, thr, out, c,
                                                           resident_ctas((const void*)k_rows_pc_tma<R, W>, T, smem));
  return cudaPeekAtLastError();
}

// the TMA variant of K3b; false when it does not apply (or the tensor map
// cannot be encoded)
static bool launch_pc_tma(const float2* Q, const float2* R0, const float* thr, const PcOut& out,
                          const FieldsConst& c, cudaStream_t st, cudaError_t& e) {
  (void)R0;
  if (!pc_tma_applies(Q, c)) return false;
  CUtensorMap map{};
  if (c.W == 512) { e = launch_pc_tma_rw<4, 512>(map, Q, thr, out, c, st); return true; }
  if (!make_qmap(Q, c, map)) return false;
  if (kPcRows == 4 && c.H % 4 == 0) e = launch_pc_tma_rw<4, 1024>(map, Q, thr, out, c, st);
  else e = launch_pc_tma_rw<2, 1024>(map, Q, thr, out, c, st);
  return true;
}

// the TMA variant of K3a for 1,024-point rows, H a multiple of 8
static bool launch_amp0_tma(const float2* Q, float2* R0, float* amp0, unsigned* hist, const FieldsConst& c,
                            cudaStream_t st, cudaError_t& e) {
  CUtensorMap map{};
  if ((c.H & 7) || !make_qmap(Q, c, map)) return false;
  constexpr int NG = kThreads / 32;
  const size_t smem = (size_t)NG * ((padded_len(1024) + 15) & ~15) * sizeof(float2) + kHistBins * sizeof(unsigned) + 128;
  if ((e = set_smem(k_rows_amp0_tma, smem)) != cudaSuccess) return true;
  const dim3 grid((c.H + NG * kAmpRows - 1) / (NG * kAmpRows), c.O, c.B);
  k_rows_amp0_tma<<<grid, kThreads, smem, st>>>(map, Q, R0, amp0, hist, c,
                                               resident_ctas((const void*)k_rows_amp0_tma, kThreads, smem),
                                               pc_tma_applies(Q, c) ? 0 : 1);
  e = cudaPeekAtLastError();
  return true;
}

template <int G>
static cudaError_t launch_pc(const float2* Q, const float2* R0, const float* thr, const PcOut& out,
                             const FieldsConst& c, cudaStream_t st) {
  if constexpr (G == 32 || G == 16) {
    cudaError_t e = cudaSuccess;
    if (launch_pc_tma(Q, R0, thr, out, c, st, e)) return e;
  }
  if (c.S == 4 && G >= 8 && G <= 128) return launch_pc_s<G, 4>(Q, R0, thr, out, c, st);
  return launch_pc_s<G, 0>(Q, R0, thr, out, c, st);
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
  const double log2e = 1.4426950408889634;
  FieldsConst c{};
  c.B = B; c.H = H; c.W = W; c.Wh = p.Wh; c.Hp = p.Hp; c.S = bk.n_scales; c.O = bk.n_orient;
  for (int s = 0; s < c.S; ++s) c.log_lambda[s] = (float)bk.log_lambda[s];
  c.a2 = (float)(bk.inv_den_r * log2e);
  c.b2 = (float)(bk.inv_den_a * log2e);
  const double sa = std::sqrt(bk.inv_den_r * log2e), sb = std::sqrt(bk.inv_den_a * log2e);
  c.sa = (float)sa;
  c.sb = (float)sb;
  for (int q = 0; q < c.S; ++q) c.ll_s[q] = (float)(bk.log_lambda[q] * sa);
  c.pi_s = (float)(M_PI * sb);
  c.two_pi_s = (float)(2.0 * M_PI * sb);
  for (int q = 0; q < c.O; ++q) {
    c.ang[q] = (float)bk.angle[q];
    c.ang_s[q] = (float)(bk.angle[q] * sb);
    c.cos_a[q] = (float)bk.cos_a[q];
    c.sin_a[q] = (float)bk.sin_a[q];
  }
  c.spread_cutoff = (float)bk.spread_cutoff;
  c.spread_gain = (float)bk.spread_gain;
  c.inv_sm1 = (float)(1.0 / (c.S > 1 ? c.S - 1 : 1));
  c.lp_lncut = (float)bk.lp_lncut;
  c.log2_inv_hw = (float)(-std::log2((double)H * (double)W));
  c.thr_factor = bk.thr_factor;
  c.tw_w = twiddle_table(W);
  c.tw_h = twiddle_table(H);
  if (!c.tw_w || !c.tw_h) return 3;
  if (!p.gw && !make_plan(W, c.plan_w)) return 2;
  if (!p.gh && !make_plan(H, c.plan_h)) return 2;
  {
    auto al8 = [](const void* q) { return ((uintptr_t)q & 7) == 0; };
    c.out_vec = al8(o.mmax) && al8(o.mmin) && al8(o.a_o) && al8(o.pc) && al8(o.amax) && ((uintptr_t)o.mim & 1) == 0;
  }

  char* w = static_cast<char*>(ws);
  float2* P = reinterpret_cast<float2*>(w + p.off_P);
  float2* Q = reinterpret_cast<float2*>(w + p.off_Q);
  float2* R0 = reinterpret_cast<float2*>(w + p.off_R0);
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
  R2_DISPATCH_G(p.gw, launch_amp0, Q, R0, amp0, hist, c, st);
  if (e != cudaSuccess) return 3;
  const unsigned n = (unsigned)((size_t)H * W);
  k_med_bins<<<B * c.O, 1024, 0, st>>>(hist, info, n);
  {
    // one resident wave: each CTA streams many passes of its plane
    const int waves = resident_ctas((const void*)k_med_collect, 256, 0);
    const size_t gx = std::max<size_t>(1, std::min<size_t>(((size_t)n / 4 + 255) / 256 + 1,
                                                           (size_t)waves / (size_t)(B * c.O)));
    dim3 grid((unsigned)gx, B * c.O);
    k_med_collect<<<grid, 256, 0, st>>>(amp0, info, cand, cnt, n);
  }
  launch_med_select(cand, cnt, info, reinterpret_cast<unsigned*>(w + p.off_mh), thr, B * c.O, n, c.thr_factor, st);
  if (cudaPeekAtLastError() != cudaSuccess) return 3;
  PcOut po{o.mmax, o.mmin, o.mim, o.a_o, o.pc, o.amax, o.range};
  if (o.range) k_range_init<<<(4 * B + 127) / 128, 128, 0, st>>>(o.range, 4 * B);
  R2_DISPATCH_G(p.gw, launch_pc, Q, R0, thr, po, c, st);
  if (e != cudaSuccess) return 3;
  return 0;
}


// ================================================= unfused reference entry points
// The reference's step-by-step API (ref: loggabor.py:131-251, mim.py:43-55)
// for callers that use the stages separately; the fused path above is what
// the pipeline runs.

// ref: loggabor.py:122-159 (_frequency_grids, build_filter_bank), in float64
// with the reference's own formulas: radial log-Gaussian x Butterworth
// low-pass (cutoff 0.45, order 15), angular Gaussian of the wrapped angle
// difference taken through atan2 of sin/cos differences, DC zeroed.
__global__ void __launch_bounds__(256) k_filter_bank(double* __restrict__ T, int H, int W, int S, int O,
                                                     double min_wl, double mult, double sigma_on_f,
                                                     double sigma_theta) {
  const size_t n = (size_t)H * W;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ky = (int)(i / W), kx = (int)(i % W);
    const double fy = (double)(ky < (H + 1) / 2 ? ky : ky - H) / (double)H;
    const double fx = (double)(kx < (W + 1) / 2 ? kx : kx - W) / (double)W;
    const bool dc = ky == 0 && kx == 0;
    const double radius = dc ? 1.0 : hypot(fx, fy);
    const double theta = atan2(fy, fx);
    const double lowpass = 1.0 / (1.0 + pow(radius / 0.45, 30.0));
    const double lsig2 = 2.0 * log(sigma_on_f) * log(sigma_on_f);
    const double st = sin(theta), ct = cos(theta);
    for (int o = 0; o < O; ++o) {
      const double a = (double)o * M_PI / (double)O;
      const double ds = st * cos(a) - ct * sin(a);
      const double dcos = ct * cos(a) + st * sin(a);
      const double dth = fabs(atan2(ds, dcos));
      const double ang = exp(-(dth * dth) / (2.0 * sigma_theta * sigma_theta));
      double wl = min_wl;
      for (int s = 0; s < S; ++s) {
        if (s) wl = min_wl * pow(mult, (double)s);
        const double l = log(radius / (1.0 / wl));
        const double rad = dc ? 0.0 : exp(-(l * l) / lsig2) * lowpass;
        T[((size_t)s * O + o) * n + i] = dc ? 0.0 : rad * ang;
      }
    }
  }
}

int filter_bank_run(int H, int W, int S, int O, double min_wl, double mult, double sigma_on_f, double sigma_theta,
                    double* transfer, cudaStream_t st) {
  const size_t n = (size_t)H * W;
  const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 4096);
  k_filter_bank<<<blocks, 256, 0, st>>>(transfer, H, W, S, O, min_wl, mult, sigma_on_f, sigma_theta);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// Inverse row FFT of every Q plane -> even / odd / amplitude planes
// [F][H][W] (ref: loggabor.py:178-184).
__global__ void __launch_bounds__(kThreads) k_rows_resp(const float2* __restrict__ Q, float* __restrict__ even,
                                                        float* __restrict__ odd, float* __restrict__ amp,
                                                        const __grid_constant__ FieldsConst c) {
  extern __shared__ float2 sm[];
  const int y = blockIdx.x, f = blockIdx.y, W = c.W, H = c.H;
  const float2* Qp = Q + (size_t)f * c.Hp * W;
  float2* buf = sm;
  float2* scr = sm + padded_len(W);
  for (int x = threadIdx.x; x < W; x += blockDim.x) buf[pad32(x)] = cconj(Qp[tq(y, x, W)]);
  __syncthreads();
  fft_generic(buf, scr, W, c.plan_w, c.tw_w, threadIdx.x, blockDim.x);
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    const float2 z = cconj(buf[pad32(x)]);
    const size_t o = ((size_t)f * H + y) * W + x;
    even[o] = z.x;
    odd[o] = z.y;
    amp[o] = hypotf(z.x, z.y);
  }
}

size_t apply_bank_workspace_bytes(int H, int W, int S, int O) {
  const FieldsPlan p = plan_fields(1, H, W, S, O);
  return p.off_Q + align_up((size_t)p.F * p.Hp * W * sizeof(float2));
}

// ref: loggabor.py:162-185 (apply_bank) for an explicit transfer array
// [S][O][H][W] (the bank as given): the generic mixed-radix passes, the
// transfer read from memory instead of generated
int apply_bank_run(const float* image, int H, int W, int S, int O, const float* transfer, float* even, float* odd,
                   float* amp, void* ws, size_t ws_bytes, cudaStream_t st) {
  const FieldsPlan p = plan_fields(1, H, W, S, O);
  if (ws_bytes < apply_bank_workspace_bytes(H, W, S, O)) return 1;
  FieldsConst c{};
  c.B = 1; c.H = H; c.W = W; c.Wh = p.Wh; c.Hp = p.Hp; c.S = S; c.O = O;
  c.tw_w = twiddle_table(W);
  c.tw_h = twiddle_table(H);
  if (!c.tw_w || !c.tw_h) return 3;
  if (!make_plan(W, c.plan_w) || !make_plan(H, c.plan_h)) return 2;
  c.xfer = transfer;
  c.inv_hw = (float)(1.0 / ((double)H * (double)W));
  char* w = static_cast<char*>(ws);
  float2* P = reinterpret_cast<float2*>(w + p.off_P);
  float2* Q = reinterpret_cast<float2*>(w + p.off_Q);
  cudaError_t e = launch_rows_fwd<0>(image, P, c, st);
  if (e == cudaSuccess) e = launch_cols<0>(P, Q, c, st);
  if (e != cudaSuccess) return 3;
  const size_t smem = (size_t)2 * padded_len(W) * sizeof(float2);
  if (set_smem(k_rows_resp, smem) != cudaSuccess) return 3;
  k_rows_resp<<<dim3(H, S * O), kThreads, smem, st>>>(Q, even, odd, amp, c);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// level-1 radix histogram of given amplitude planes (the exact-median input)
__global__ void __launch_bounds__(256) k_hist_planes(const float* __restrict__ a, unsigned* __restrict__ hist, unsigned n) {
  __shared__ unsigned sh[kHistBins];
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const float* ap = a + (size_t)blockIdx.y * n;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&sh[__float_as_uint(fmaxf(ap[i], 0.f)) >> 19], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[(size_t)blockIdx.y * kHistBins + i], sh[i]);
}

// Per-pixel phase congruency and moments from a response stack (ref:
// loggabor.py:188-251), float32; T[o] from the exact median of the scale-0
// amplitude plane.  pc == nullptr: orientation amplitude sums only.
struct Trig16 { float c[16], s[16]; };
__global__ void __launch_bounds__(256) k_pc_stack(const float* __restrict__ even, const float* __restrict__ odd,
                                                  const float* __restrict__ amp, int S, int O, size_t n,
                                                  const float* __restrict__ thr, float inv_sm1, float gain,
                                                  float cut, const Trig16 trig, float* __restrict__ a_o,
                                                  float* __restrict__ pc, float* __restrict__ mmax,
                                                  float* __restrict__ mmin) {
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
    float A = 0.f, B = 0.f, C = 0.f;
    for (int o = 0; o < O; ++o) {
      float se = 0.f, so = 0.f, sa = 0.f, mx = 0.f;
      for (int s = 0; s < S; ++s) {
        const size_t q = ((size_t)s * O + o) * n + p;
        se += even[q];
        so += odd[q];
        sa += amp[q];
        mx = fmaxf(mx, amp[q]);
      }
      if (a_o) a_o[(size_t)o * n + p] = sa;
      if (!pc) continue;
      const float xe = sqrtf(se * se + so * so) + 1e-4f;
      const float me = se / xe, mo = so / xe;
      float en = 0.f;
      for (int s = 0; s < S; ++s) {
        const size_t q = ((size_t)s * O + o) * n + p;
        const float e = even[q], d = odd[q];
        en += e * me + d * mo - fabsf(e * mo - d * me);
      }
      en = fmaxf(en - thr[o], 0.f);
      const float spread = (sa / (mx + 1e-4f) - 1.f) * inv_sm1;
      const float w = 1.f / (1.f + expf(gain * (cut - spread)));
      const float v = w * en / (sa + 1e-4f);
      pc[(size_t)o * n + p] = v;
      const float pcc = v * trig.c[o], pcs = v * trig.s[o];
      A += pcc * pcc;
      B += pcc * pcs;
      C += pcs * pcs;
    }
    if (!pc) continue;
    const float b2 = 2.f * B;
    const float root = sqrtf(b2 * b2 + (A - C) * (A - C));
    mmax[p] = 0.5f * (C + A + root);
    mmin[p] = fmaxf(0.5f * (C + A - root), 0.f);
  }
}

size_t pc_stack_workspace_bytes(int H, int W, int S, int O) {
  const size_t n = (size_t)H * W;
  return debug_median_workspace_bytes(O, (int)n) + align_up((size_t)O * sizeof(float));
}

int pc_stack_run(const float* even, const float* odd, const float* amp, int H, int W, const BankConsts& bk,
                 float* a_o, float* pc, float* mmax, float* mmin, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int S = bk.n_scales, O = bk.n_orient;
  const size_t n = (size_t)H * W;
  if (ws_bytes < pc_stack_workspace_bytes(H, W, S, O)) return 1;
  char* w = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* q = w; w += align_up(bytes); return q; };
  auto* hist = reinterpret_cast<unsigned*>(take((size_t)O * kHistBins * sizeof(unsigned)));
  auto* info = reinterpret_cast<MedInfo*>(take((size_t)O * sizeof(MedInfo)));
  auto* cand = reinterpret_cast<unsigned*>(take((size_t)O * n * sizeof(unsigned)));
  auto* cnt = reinterpret_cast<unsigned*>(take((size_t)O * sizeof(unsigned)));
  auto* mh = reinterpret_cast<unsigned*>(take((size_t)O * 2 * kMedH * sizeof(unsigned)));
  auto* thr = reinterpret_cast<float*>(take((size_t)O * sizeof(float)));
  Trig16 trig{};
  for (int o = 0; o < O; ++o) { trig.c[o] = (float)bk.cos_a[o]; trig.s[o] = (float)bk.sin_a[o]; }
  if (pc) {
    // exact median of each scale-0 amplitude plane (amp[0][o] = planes o of amp)
    cudaMemsetAsync(hist, 0, (size_t)O * kHistBins * sizeof(unsigned), st);
    cudaMemsetAsync(cnt, 0, (size_t)O * sizeof(unsigned), st);
    k_hist_planes<<<dim3(64, O), 256, 0, st>>>(amp, hist, (unsigned)n);
    k_med_bins<<<O, 1024, 0, st>>>(hist, info, (unsigned)n);
    k_med_collect<<<dim3(64, O), 256, 0, st>>>(amp, info, cand, cnt, (unsigned)n);
    launch_med_select(cand, cnt, info, mh, thr, O, (unsigned)n, bk.thr_factor, st);
  }
  const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 8192);
  k_pc_stack<<<blocks, 256, 0, st>>>(even, odd, amp, S, O, n, thr, (float)(1.0 / (S > 1 ? S - 1 : 1)),
                                     (float)bk.spread_gain, (float)bk.spread_cutoff, trig, a_o, pc, mmax, mmin);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// ref: loggabor.py:188-190 (orientation_amplitudes): sum over scales in
// float64, in scale order (as numpy's axis-0 reduction)
__global__ void __launch_bounds__(256) k_sum_scales(const double* __restrict__ amp, int S, int O, size_t n,
                                                    double* __restrict__ a_o) {
  const size_t total = (size_t)O * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    double acc = amp[i];
    for (int s = 1; s < S; ++s) acc += amp[(size_t)s * total + i];
    a_o[i] = acc;
  }
}

int sum_scales_run(const double* amp, int S, int O, int H, int W, double* a_o, cudaStream_t st) {
  const size_t total = (size_t)O * H * W;
  const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, 8192);
  if (total) k_sum_scales<<<blocks, 256, 0, st>>>(amp, S, O, (size_t)H * W, a_o);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// ref: mim.py:43-55 (build_mim): first argmax over channels, 1-based, in float64
__global__ void __launch_bounds__(256) k_build_mim(const double* __restrict__ a, int O, size_t n,
                                                   int* __restrict__ idx, double* __restrict__ amax) {
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
    double best = a[p];
    int bi = 0;
    for (int o = 1; o < O; ++o) {
      const double v = a[(size_t)o * n + p];
      if (v > best || (v != v && best == best)) { best = v; bi = o; }   // NaN wins first, as np.argmax
      if (best != best) break;
    }
    idx[p] = bi + 1;
    if (amax) amax[p] = best;
  }
}

int build_mim_run(const double* a_o, int O, int H, int W, int* idx, double* amax, cudaStream_t st) {
  const size_t n = (size_t)H * W;
  const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 8192);
  k_build_mim<<<blocks, 256, 0, st>>>(a_o, O, n, idx, amax);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

// ---------------------------------------------------------- diagnostics ---
// The exact-median stage on arbitrary complex planes: |z| of each element
// (as k_rows_amp0 computes it) and its radix histogram, then the same
// k_med_bins / k_med_collect / k_med_final kernels the filter bank runs.
__global__ void __launch_bounds__(256) k_debug_amp(const float2* __restrict__ z, float* __restrict__ amps,
                                                   unsigned* __restrict__ hist, unsigned n) {
  __shared__ unsigned sh[kHistBins];
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const size_t off = (size_t)blockIdx.y * n;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float2 v = z[off + i];
    const float a = sqrt_approx(fmaf(v.x, v.x, v.y * v.y));
    amps[off + i] = a;
    atomicAdd(&sh[__float_as_uint(a) >> 19], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[(size_t)blockIdx.y * kHistBins + i], sh[i]);
}

size_t debug_median_workspace_bytes(int planes, int n) {
  return align_up((size_t)planes * kHistBins * sizeof(unsigned)) + align_up((size_t)planes * sizeof(MedInfo)) +
         align_up((size_t)planes * n * sizeof(unsigned)) + align_up((size_t)planes * sizeof(unsigned)) +
         align_up((size_t)planes * 2 * kMedH * sizeof(unsigned));
}

int debug_median_run(const float2* z, int planes, int n, float* amps, float* med, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  if (ws_bytes < debug_median_workspace_bytes(planes, n)) return 1;
  char* w = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { char* p = w; w += align_up(bytes); return p; };
  auto* hist = reinterpret_cast<unsigned*>(take((size_t)planes * kHistBins * sizeof(unsigned)));
  auto* info = reinterpret_cast<MedInfo*>(take((size_t)planes * sizeof(MedInfo)));
  auto* cand = reinterpret_cast<unsigned*>(take((size_t)planes * n * sizeof(unsigned)));
  auto* cnt = reinterpret_cast<unsigned*>(take((size_t)planes * sizeof(unsigned)));
  auto* mh = reinterpret_cast<unsigned*>(take((size_t)planes * 2 * kMedH * sizeof(unsigned)));
  cudaMemsetAsync(hist, 0, (size_t)planes * kHistBins * sizeof(unsigned), st);
  cudaMemsetAsync(cnt, 0, (size_t)planes * sizeof(unsigned), st);
  k_debug_amp<<<dim3(32, planes), 256, 0, st>>>(z, amps, hist, (unsigned)n);
  k_med_bins<<<planes, 1024, 0, st>>>(hist, info, (unsigned)n);
  dim3 grid((unsigned)min((size_t)64, ((size_t)n / 4 + 255) / 256 + 1), planes);
  k_med_collect<<<grid, 256, 0, st>>>(amps, info, cand, cnt, (unsigned)n);
  launch_med_select(cand, cnt, info, mh, med, planes, (unsigned)n, 1.0, st);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2
