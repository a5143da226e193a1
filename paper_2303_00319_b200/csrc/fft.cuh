// Register-blocked Stockham FFT engine for the log-Gabor filter bank.
//
// Fast path (N = 32*G, G a power of two <= 128): a group of G threads owns
// one transform; every thread keeps 32 complex values in registers.  The
// first pass is a radix-32 butterfly entirely in registers, followed by one
// shared-memory exchange and a radix-G pass (two passes for G > 32), so a
// 1024-point transform costs a single shared-memory round trip.
//
// Data convention (both directions): thread t of the group holds element
// t + G*m in v[m], m = 0..31.  Shared buffers use the padded index pad32().
//
// Generic path: any N whose factors are 2, 3, 5 (the reference's own fixtures
// use 384 = 2^7*3 and 800 = 2^5*5^2).  The whole CTA cooperates on one
// transform held in shared memory (ping-pong Stockham passes).
//
// Only the forward transform (e^{-2 pi i nk/N}, numpy sign) is implemented;
// inverses use conj(FFT(conj(x))).
#pragma once
#include "common.cuh"

namespace r2 {

// cos / sin of 2*pi*j/32, j = 0..31
struct W32 {
  static constexpr float c[32] = {
    1.000000000e+00f, 9.807852804e-01f, 9.238795325e-01f, 8.314696123e-01f, 7.071067812e-01f,
    5.555702330e-01f, 3.826834324e-01f, 1.950903220e-01f, 0.0f, -1.950903220e-01f,
    -3.826834324e-01f, -5.555702330e-01f, -7.071067812e-01f, -8.314696123e-01f, -9.238795325e-01f,
    -9.807852804e-01f, -1.000000000e+00f, -9.807852804e-01f, -9.238795325e-01f, -8.314696123e-01f,
    -7.071067812e-01f, -5.555702330e-01f, -3.826834324e-01f, -1.950903220e-01f, 0.0f,
    1.950903220e-01f, 3.826834324e-01f, 5.555702330e-01f, 7.071067812e-01f, 8.314696123e-01f,
    9.238795325e-01f, 9.807852804e-01f};
  static constexpr float s[32] = {
    0.0f, 1.950903220e-01f, 3.826834324e-01f, 5.555702330e-01f, 7.071067812e-01f,
    8.314696123e-01f, 9.238795325e-01f, 9.807852804e-01f, 1.000000000e+00f, 9.807852804e-01f,
    9.238795325e-01f, 8.314696123e-01f, 7.071067812e-01f, 5.555702330e-01f, 3.826834324e-01f,
    1.950903220e-01f, 0.0f, -1.950903220e-01f, -3.826834324e-01f, -5.555702330e-01f,
    -7.071067812e-01f, -8.314696123e-01f, -9.238795325e-01f, -9.807852804e-01f, -1.000000000e+00f,
    -9.807852804e-01f, -9.238795325e-01f, -8.314696123e-01f, -7.071067812e-01f, -5.555702330e-01f,
    -3.826834324e-01f, -1.950903220e-01f};
};

// a * exp(-2 pi i J / 32) with J a compile-time constant
template <int J>
R2_DEV float2 tw32(float2 a) {
  constexpr int j = J & 31;
  if constexpr (j == 0) return a;
  else if constexpr (j == 8) return make_float2(a.y, -a.x);
  else if constexpr (j == 16) return make_float2(-a.x, -a.y);
  else if constexpr (j == 24) return make_float2(-a.y, a.x);
  else if constexpr ((j & 7) == 4) {
    constexpr float h = 7.071067812e-01f;
    constexpr float cc = W32::c[j] > 0 ? h : -h;
    constexpr float ss = W32::s[j] > 0 ? h : -h;
    return cmul_cs(a, cc, ss);
  } else {
    constexpr float cc = W32::c[j], ss = W32::s[j];
    return cmul_cs(a, cc, ss);
  }
}

// ---- in-register forward DFTs of radix 2..32 (natural order in/out) -------
template <int R> struct DFT;

template <> struct DFT<1> { R2_DEV static void run(float2*) {} };

template <> struct DFT<2> {
  R2_DEV static void run(float2* v) {
    float2 a = v[0], b = v[1];
    v[0] = cadd(a, b); v[1] = csub(a, b);
  }
};

template <> struct DFT<4> {
  R2_DEV static void run(float2* v) {
    float2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    float2 s13 = cadd(v[1], v[3]), d13 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(s02, s13); v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13); v[3] = csub(d02, d13);
  }
};

// DFT of R = R1*R2 by the two-dimensional (Cooley-Tukey) decomposition:
// n = R2*n1 + n2, k = k1 + R1*k2.
template <int R1, int R2>
struct DFT2D {
  static constexpr int R = R1 * R2;
  template <int N2, int K1>
  R2_DEV static float2 twid(float2 a) { return tw32<(N2 * K1 * (32 / R)) & 31>(a); }

  template <int N2>
  R2_DEV static void cols(const float2* v, float2* t) {
    float2 a[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) a[n1] = v[R2 * n1 + N2];
    DFT<R1>::run(a);
    t[N2 * R1 + 0] = a[0];
    if constexpr (R1 > 1) t[N2 * R1 + 1] = twid<N2, 1>(a[1]);
    if constexpr (R1 > 2) t[N2 * R1 + 2] = twid<N2, 2>(a[2]);
    if constexpr (R1 > 3) t[N2 * R1 + 3] = twid<N2, 3>(a[3]);
    static_assert(R1 <= 4, "R1 <= 4");
    if constexpr (N2 + 1 < R2) cols<N2 + 1>(v, t);
  }

  R2_DEV static void run(float2* v) {
    float2 t[R];
    cols<0>(v, t);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      float2 b[R2];
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) b[n2] = t[n2 * R1 + k1];
      DFT<R2>::run(b);
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) v[k1 + R1 * k2] = b[k2];
    }
  }
};

template <> struct DFT<8> { R2_DEV static void run(float2* v) { DFT2D<4, 2>::run(v); } };
template <> struct DFT<16> { R2_DEV static void run(float2* v) { DFT2D<4, 4>::run(v); } };
template <> struct DFT<32> { R2_DEV static void run(float2* v) { DFT2D<4, 8>::run(v); } };

// radix 3 / 5 for the generic path
template <> struct DFT<3> {
  R2_DEV static void run(float2* v) {
    constexpr float s3 = 8.660254038e-01f;
    float2 a = v[0], b = v[1], c = v[2];
    float2 sbc = cadd(b, c), dbc = csub(b, c);
    float2 m = make_float2(a.x - 0.5f * sbc.x, a.y - 0.5f * sbc.y);
    float2 r = make_float2(s3 * dbc.y, -s3 * dbc.x);   // -i*s3*(b-c)
    v[0] = cadd(a, sbc); v[1] = cadd(m, r); v[2] = csub(m, r);
  }
};

template <> struct DFT<5> {
  R2_DEV static void run(float2* v) {
    constexpr float c1 = 3.090169944e-01f, c2 = -8.090169944e-01f;
    constexpr float s1 = 9.510565163e-01f, s2 = 5.877852523e-01f;
    float2 x0 = v[0];
    float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    float2 m1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
    float2 m2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
    // -i * (s1*b1 + s2*b2) and -i * (s2*b1 - s1*b2)
    float2 n1 = make_float2(s1 * b1.y + s2 * b2.y, -(s1 * b1.x + s2 * b2.x));
    float2 n2 = make_float2(s2 * b1.y - s1 * b2.y, -(s2 * b1.x - s1 * b2.x));
    v[0] = cadd(x0, cadd(a1, a2));
    v[1] = cadd(m1, n1); v[4] = csub(m1, n1);
    v[2] = cadd(m2, n2); v[3] = csub(m2, n2);
  }
};

// ---- fast path --------------------------------------------------------------

// Twiddle r = 1..R-1 inputs of one butterfly by W_N^{r*e}, e = k*step.
// Powers come from a short recurrence refreshed from the table every 8
// steps.  The table values a butterfly needs (W^e and W^{8qe}) are loaded
// by tw_load before the pass's exchange, so their latency overlaps it.
template <int R>
struct TwPre {
  float2 w[(R + 7) / 8];   // [0] = W^e, [q] = W^{8qe}
};
template <int R, int N>
R2_DEV TwPre<R> tw_load(const float2* __restrict__ tw, int e) {
  TwPre<R> p;
  p.w[0] = __ldg(&tw[e]);
#pragma unroll
  for (int q = 1; q < (R + 7) / 8; ++q) p.w[q] = __ldg(&tw[(8 * q * e) & (N - 1)]);
  return p;
}
template <int R>
R2_DEV void apply_twiddles(float2* v, const TwPre<R>& p, int e) {
  if (e == 0) return;
  const float2 base = p.w[0];
  float2 w = base;
#pragma unroll
  for (int r = 1; r < R; ++r) {
    if (r > 1) {
      if ((r & 7) == 0) w = p.w[r / 8];
      else w = cmul(w, base);
    }
    v[r] = cmul(v[r], w);
  }
}

// One Stockham pass with radix R over stride Ns, each thread doing 32/R
// butterflies j = t + G*i.  Inputs come from buf; non-final passes write
// their outputs back to buf, the final pass leaves X[t + G*m] in v[m].
template <int G, int R, int NS, bool LAST, class Sync>
R2_DEV void stockham_pass(float2 (&v)[32], float2* buf, const float2* __restrict__ tw, int t, Sync& sync) {
  constexpr int N = 32 * G, PER = 32 / R, NR = N / R, STEP = N / (NS * R);
  TwPre<R> pre[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) pre[i] = tw_load<R, N>(tw, ((t + G * i) & (NS - 1)) * STEP);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = t + G * i;
#pragma unroll
    for (int r = 0; r < R; ++r) v[i * R + r] = buf[pad32(j + r * NR)];
  }
  sync();
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = t + G * i;
    const int k = j & (NS - 1);
    apply_twiddles<R>(&v[i * R], pre[i], k * STEP);
    DFT<R>::run(&v[i * R]);
  }
  if constexpr (!LAST) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = t + G * i;
      const int k = j & (NS - 1);
      const int o = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[pad32(o + r * NS)] = v[i * R + r];
    }
    sync();
  } else {
    float2 u[32];
#pragma unroll
    for (int i = 0; i < PER; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) u[i + PER * r] = v[i * R + r];
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = u[m];
  }
}

// Forward FFT of N = 32*G points; v[m] = x[t + G*m] in, X[t + G*m] out.
// buf: group-private padded scratch of padded_len(N) float2.
// tw:  table W_N^j = exp(-2 pi i j / N), j < N.
template <int G, class Sync>
R2_DEV void fft_fast(float2 (&v)[32], float2* buf, const float2* __restrict__ tw, int t, Sync& sync) {
  DFT<32>::run(v);
  if constexpr (G == 1) {
    return;
  } else {
#pragma unroll
    for (int r = 0; r < 32; ++r) buf[pad32(32 * t + r)] = v[r];
    sync();
    if constexpr (G <= 32) {
      stockham_pass<G, G, 32, true>(v, buf, tw, t, sync);
    } else {
      static_assert(G == 64 || G == 128, "G in {1..128}");
      stockham_pass<G, 32, 32, false>(v, buf, tw, t, sync);
      stockham_pass<G, G / 32, 1024, true>(v, buf, tw, t, sync);
    }
  }
}

// Synchronisation objects for a group of G threads.
struct SyncWarp {
  unsigned mask;
  R2_DEV void operator()() const { __syncwarp(mask); }
};
// lanes of the G-thread group (G <= 32) containing this thread
R2_DEV unsigned group_mask(int G) {
  if (G >= 32) return 0xffffffffu;
  const unsigned base = (threadIdx.x & 31) / G * G;
  return ((1u << G) - 1u) << base;
}
struct SyncNamed {
  int id, n;
  R2_DEV void operator()() const { named_sync(id, n); }
};
struct SyncBlock { R2_DEV void operator()() const { __syncthreads(); } };

// ---- generic path -----------------------------------------------------------

struct GenericPlan {
  int n_pass;
  int radix[16];
};

template <int R>
R2_DEV void generic_pass(const float2* src, float2* dst, int N, int Ns, const float2* __restrict__ tw,
                         int tid, int nth) {
  const int NR = N / R;
  const int step = N / (Ns * R);
  for (int j = tid; j < NR; j += nth) {
    const int k = j % Ns;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[pad32(j + r * NR)];
    if (k) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[(r * k * step) % N]));
    }
    DFT<R>::run(v);
    const int o = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[pad32(o + r * Ns)] = v[r];
  }
}

// One Stockham pass of any radix R (the prime factors above 5 of a generic
// length, ref: loggabor.py:162-185 takes any image size): thread per output,
// an R-term DFT of the twiddled inputs with W_R^m = W_N^(m N / R) from the
// same table.  O(N R) per pass, so lengths with large prime factors are
// slow but exact in the same sense as the radix-2/3/5 passes.
R2_DEV void generic_pass_any(const float2* src, float2* dst, int N, int Ns, int R, const float2* __restrict__ tw,
                             int tid, int nth) {
  const int NR = N / R;
  const int step = N / (Ns * R);
  const int wr = N / R;                 // W_R = W_N^wr
  for (int idx = tid; idx < N; idx += nth) {
    const int j = idx % NR, ro = idx / NR;
    const int k = j % Ns;
    float2 acc = make_float2(0.f, 0.f);
    int e_in = 0, e_out = 0;            // exponents of W_N, kept reduced mod N
    const int din = k * step, dout = (ro * wr) % N;
    for (int r = 0; r < R; ++r) {
      const float2 x = src[pad32(j + r * NR)];
      const int e = e_in + e_out >= N ? e_in + e_out - N : e_in + e_out;   // twiddle r k step + DFT r ro N / R
      const float2 w = __ldg(&tw[e]);
      acc.x = fmaf(x.x, w.x, fmaf(-x.y, w.y, acc.x));
      acc.y = fmaf(x.x, w.y, fmaf(x.y, w.x, acc.y));
      e_in += din;
      if (e_in >= N) e_in -= N;
      e_out += dout;
      if (e_out >= N) e_out -= N;
    }
    const int o = (j / Ns) * Ns * R + k;
    dst[pad32(o + ro * Ns)] = acc;
  }
}

// Block-cooperative forward FFT of buf (padded, natural order) in place.
R2_DEV void fft_generic(float2* buf, float2* scr, int N, const GenericPlan& plan,
                        const float2* __restrict__ tw, int tid, int nth) {
  float2* src = buf;
  float2* dst = scr;
  int Ns = 1;
  for (int p = 0; p < plan.n_pass; ++p) {
    const int R = plan.radix[p];
    switch (R) {
      case 2: generic_pass<2>(src, dst, N, Ns, tw, tid, nth); break;
      case 3: generic_pass<3>(src, dst, N, Ns, tw, tid, nth); break;
      case 4: generic_pass<4>(src, dst, N, Ns, tw, tid, nth); break;
      case 5: generic_pass<5>(src, dst, N, Ns, tw, tid, nth); break;
      case 8: generic_pass<8>(src, dst, N, Ns, tw, tid, nth); break;
      default: generic_pass_any(src, dst, N, Ns, R, tw, tid, nth); break;
    }
    __syncthreads();
    Ns *= R;
    float2* tmp = src; src = dst; dst = tmp;
  }
  if (src != buf) {
    for (int i = tid; i < N; i += nth) buf[pad32(i)] = src[pad32(i)];
    __syncthreads();
  }
}

}  // namespace r2
