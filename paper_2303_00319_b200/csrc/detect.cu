// FAST keypoints on the moment maps, exact to the reference.
//
// Replaces ref: pkg/src/rift2/detector.py:50-155:
//   _normalize (:80-84), _fast_score (:50-77), detect_fast (:87-113),
//   _merge_within_radius (:116-137), detect_keypoints (:140-155).
//
// Exactness: the reference scores d_j = n_j - n_c on the min-max normalised
// map n.  Normalisation fl(fl(v - lo) / fl(hi - lo)) and fl(a - c) are both
// monotone non-decreasing, so max_k min_arc fl(n_j - n_c) equals
// fl(n(max_k min_arc v_j) - n(v_c)) bit for bit.  The arc min/max therefore
// run on the raw map values (float32 for the GPU's own maps) and only three
// float64 operations per pixel touch the normalised values.
//
// Kernels: k_init -> k_minmax -> k_fast_nms (score + 3x3 NMS + margin +
// candidate keys) -> k_sel_* (multi-CTA top max_points of the (-score, y, x,
// kind) keys: histogram, threshold bin, gather, rank) -> k_merge_suppress (2-px greedy merge of
// corners and edges as a parallel priority MIS, cap).
#include <cfloat>

#include "detect.h"
#include "sort.cuh"

namespace r2 {

namespace {

constexpr int kTile = 32;                 // score tile width
constexpr int kTileY = 64;                // score tile height (halves the border ring per pixel)
constexpr int kHalo = 4;                  // 3 for the ring + 1 for NMS
constexpr int kIn = kTile + 2 * kHalo;    // 40
constexpr int kInY = kTileY + 2 * kHalo;  // 72
constexpr int kSc = kTile + 2;            // 34
constexpr int kScY = kTileY + 2;          // 66
constexpr int kMaxNbr = 32;

// Bresenham circle of radius 3 (ref: detector.py:21-26, _CIRCLE) is spelled
// out at compile time in fast_score, so the ring loads use immediate offsets

R2_DEV unsigned long long ord_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
R2_DEV double ord_val(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// plane = image * nm + map; map 0 = moment_min (corners), 1 = moment_max (edges)
template <class T>
R2_DEV const T* plane_ptr(const T* mins, const T* maxs, int plane, int nm, size_t n) {
  const int b = plane / nm, m = plane % nm;
  return (m == 0 ? mins : maxs) + (size_t)b * n;
}

__global__ void k_init(unsigned long long* mm, unsigned* cnt, int planes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < planes) { mm[2 * i] = ~0ull; mm[2 * i + 1] = 0ull; cnt[i] = 0; }
}

template <class T>
__global__ void __launch_bounds__(256) k_minmax(const T* __restrict__ mins, const T* __restrict__ maxs, int nm,
                                                size_t n, unsigned long long* mm) {
  const int plane = blockIdx.y;
  const T* p = plane_ptr(mins, maxs, plane, nm, n);
  unsigned long long lo = ~0ull, hi = 0ull;
  if constexpr (sizeof(T) == 4) {
    // float maps: float4 loads and float min / max; only the warp results
    // become ordered double keys (the conversion is exact and monotone)
    float flo = FLT_MAX, fhi = -FLT_MAX;
    const size_t n4 = ((size_t)reinterpret_cast<uintptr_t>(p) & 15) == 0 ? n / 4 : 0;
    const float4* p4 = reinterpret_cast<const float4*>(p);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      const float4 v = __ldg(&p4[i]);
      flo = fminf(flo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
      fhi = fmaxf(fhi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (size_t i = 4 * n4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      flo = fminf(flo, p[i]);
      fhi = fmaxf(fhi, p[i]);
    }
    if (flo <= fhi) { lo = ord_key((double)flo); hi = ord_key((double)fhi); }
  } else {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const unsigned long long k = ord_key((double)p[i]);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, off);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, off);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[2 * plane], lo);
    atomicMax(&mm[2 * plane + 1], hi);
  }
}

R2_DEV float min3(float a, float b, float c) { return fminf(fminf(a, b), c); }   // FMNMX3
R2_DEV float max3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
R2_DEV double min3(double a, double b, double c) { return fmin(fmin(a, b), c); }
R2_DEV double max3(double a, double b, double c) { return fmax(fmax(a, b), c); }

// Largest threshold at which some 9-arc of the ring is brighter (A) /
// darker (B) than the centre, on raw values: A = max_k min_{j<9} v[k+j],
// B = min_k max_{j<9} v[k+j].  Windows of 3, then 3 windows of 3.
template <class T>
R2_DEV void arc_extrema(const T (&v)[16], T& A, T& B) {
  T m3[16], M3[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    m3[k] = min3(v[k], v[(k + 1) & 15], v[(k + 2) & 15]);
    M3[k] = max3(v[k], v[(k + 1) & 15], v[(k + 2) & 15]);
  }
  T m9[16], M9[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    m9[k] = min3(m3[k], m3[(k + 3) & 15], m3[(k + 6) & 15]);
    M9[k] = max3(M3[k], M3[(k + 3) & 15], M3[(k + 6) & 15]);
  }
  T a = max3(m9[0], m9[1], m9[2]), b = min3(M9[0], M9[1], M9[2]);
#pragma unroll
  for (int k = 3; k < 15; k += 2) { a = max3(a, m9[k], m9[k + 1]); b = min3(b, M9[k], M9[k + 1]); }
  A = fmax(a, m9[15]);
  B = fmin(b, M9[15]);
}

// (x - lo) / span in float64, correctly rounded, from y = RN(1 / span):
// q = RN(d y), r = d - span q (exact by fma), RN(q + r y) = RN(d / span)
// (Markstein's theorem; d >= 0, span > 0, no under/overflow in this range).
R2_DEV double div_span(double x, double lo, double span, double y) {
  const double d = x - lo;
  const double q = d * y;
  const double r = fma(-q, span, d);
  return fma(r, y, q);
}

// FAST score of the pixel at staged position (cy, cx) (ref: detector.py:50-84
// through the monotone normalisation, see the file header)
template <class T>
R2_DEV double fast_score(const T (*sv)[kIn + 1], int cy, int cx, double lo, double span, double rspan) {
  constexpr int dx[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
  constexpr int dy[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};
  T v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = sv[cy + dy[k]][cx + dx[k]];
  T A, B;
  arc_extrema(v, A, B);
  const T c = sv[cy][cx];
  // ref: max(max(na - nc, nc - nb), 0) with n = (v - lo) / span; a side
  // whose raw extreme does not beat the centre contributes <= 0: skipped
  double s = 0.0;
  if (A > c || B < c) {
    const double nc = div_span((double)c, lo, span, rspan);
    if (A > c) s = fmax(s, div_span((double)A, lo, span, rspan) - nc);
    if (B < c) s = fmax(s, nc - div_span((double)B, lo, span, rspan));
  }
  return s;
}

// score of score-tile position (sy, sx) = image pixel (y, x): -inf outside the
// image (never wins the NMS), 0 in the 3-pixel frame (ref: detector.py:63-76)
template <class T>
R2_DEV double tile_score(const T (*sv)[kIn + 1], int sy, int sx, int y, int x, int H, int W, bool inner, double lo,
                         double span, double rspan) {
  if (!inner) {
    if (y < 0 || y >= H || x < 0 || x >= W) return -DBL_MAX;
    if (y < 3 || y >= H - 3 || x < 3 || x >= W - 3) return 0.0;
  }
  return fast_score(sv, sy + kHalo - 1, sx + kHalo - 1, lo, span, rspan);
}

template <class T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 6 : 1) k_fast_nms(const T* __restrict__ mins, const T* __restrict__ maxs, int H, int W,
                                                  const unsigned long long* __restrict__ mm, double thr,
                                                  int margin, int nm, K128* __restrict__ cand,
                                                  unsigned* __restrict__ cnt, size_t cap) {
  __shared__ __align__(16) T sv[kInY][kIn + 1];
  __shared__ double ss[kScY][kSc + 1];
  const int plane = blockIdx.z;
  const int kind = nm == 2 ? (plane & 1) : 0;
  const T* p = plane_ptr(mins, maxs, plane, nm, (size_t)H * W);
  const double lo = ord_val(mm[2 * plane]);
  const double hi = ord_val(mm[2 * plane + 1]);
  const double span = hi - lo;
  if (!(span > 0)) return;   // normalised map is all zeros: no keypoints
  const double rspan = 1.0 / span;
  const int ty0 = blockIdx.y * kTileY, tx0 = blockIdx.x * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tile-uniform: the staged input lies inside the image / every scored
  // pixel is at least 3 pixels from the border
  const bool in_img = ty0 - kHalo >= 0 && ty0 + kTileY + kHalo <= H && tx0 - kHalo >= 0 && tx0 + kTile + kHalo <= W;
  const bool inner = ty0 - 1 >= 3 && ty0 + kTileY + 1 <= H - 3 && tx0 - 1 >= 3 && tx0 + kTile + 1 <= W - 3;
  if (sizeof(T) == 4 && in_img && (W & 3) == 0) {
    // 40 x 40 floats as 10 float4 per row (the row start tx0 - 4 is 16-byte aligned)
    for (int i = threadIdx.x; i < kInY * (kIn / 4); i += 256) {
      const int r = i / (kIn / 4), q = i - r * (kIn / 4);
      const float4 f = __ldg(reinterpret_cast<const float4*>(p + (size_t)(ty0 - kHalo + r) * W + tx0 - kHalo) + q);
      T* d = &sv[r][4 * q];
      d[0] = f.x; d[1] = f.y; d[2] = f.z; d[3] = f.w;
    }
  } else {
    for (int r = warp; r < kInY; r += 8) {
      const int yy = ty0 - kHalo + r;
      const bool row_in = yy >= 0 && yy < H;
      const T* prow = p + (size_t)(row_in ? yy : 0) * W;
      for (int cx = lane; cx < kIn; cx += 32) {
        const int xx = tx0 - kHalo + cx;
        sv[r][cx] = (row_in && xx >= 0 && xx < W) ? prow[xx] : T(0);
      }
    }
  }
  __syncthreads();
  // interior 32 x 32 scores: warp = row group, lane = column
#pragma unroll 1
  for (int r = warp; r < kTileY; r += 8)
    ss[r + 1][lane + 1] = tile_score(sv, r + 1, lane + 1, ty0 + r, tx0 + lane, H, W, inner, lo, span, rspan);
  // the one-pixel border ring of the score tile (196 positions)
  if (threadIdx.x < 2 * kSc + 2 * kTileY) {
    int sy, sx;
    const int i = threadIdx.x;
    if (i < kSc) { sy = 0; sx = i; }
    else if (i < 2 * kSc) { sy = kScY - 1; sx = i - kSc; }
    else if (i < 2 * kSc + kTileY) { sy = 1 + i - 2 * kSc; sx = 0; }
    else { sy = 1 + i - 2 * kSc - kTileY; sx = kSc - 1; }
    ss[sy][sx] = tile_score(sv, sy, sx, ty0 - 1 + sy, tx0 - 1 + sx, H, W, false, lo, span, rspan);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTileY * kTile; i += blockDim.x) {
    const int ly = i >> 5, lx = i & 31;
    const int y = ty0 + ly, x = tx0 + lx;
    bool keep = false;
    double s = 0.0;
    if (y < H && x < W) {
      s = ss[ly + 1][lx + 1];
      keep = s > thr && x >= margin && x <= W - 1 - margin && y >= margin && y <= H - 1 - margin;
      if (keep) {
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) keep = keep && s >= ss[ly + dy][lx + dx];
      }
    }
    const unsigned slot = agg_inc(&cnt[plane], keep);
    if (keep && slot < cap) {
      K128 k;
      k.hi = ~(unsigned long long)__double_as_longlong(s);
      k.lo = ((unsigned long long)y << 32) | ((unsigned long long)x << 8) | (unsigned long long)kind;
      cand[(size_t)plane * cap + slot] = k;
    }
  }
}

// ---- multi-CTA top-K selection -------------------------------------------
// Keys are (-score, y, x, kind) with the score's float64 bits in `hi`, so a
// monotone log-scale bin of the score orders them coarsely.  A histogram of
// all candidates finds the bin holding the K-th key (the threshold bin);
// keys of that bin and above are scattered into per-bin buckets at offsets
// from a scan of the histogram (higher bins first), and each key's final
// position is its bucket offset plus its rank among the keys of its own
// bucket.  Keys are unique (pixel + kind), so positions are a permutation
// and the first K equal the full sort's first K.
constexpr int kSelBins = 4096;
constexpr int kSelCtas = 32;                    // CTAs per plane in the streaming passes

R2_DEV int sel_bin(const K128& k) {
  // score bits (sign 0): exponent + 7 mantissa bits; scores > threshold >= 2^-20
  const unsigned long long b = ~k.hi;
  const long long v = (long long)(b >> 45) - (long long)((1003ull << 7));
  return v < 0 ? 0 : (v >= kSelBins ? kSelBins - 1 : (int)v);
}

__global__ void __launch_bounds__(256) k_sel_hist(const K128* __restrict__ cand, const unsigned* __restrict__ cnt,
                                                  size_t cap, unsigned* __restrict__ ghist) {
  __shared__ unsigned h[kSelBins];
  const int plane = blockIdx.y;
  const int n = (int)min((size_t)cnt[plane], cap);
  for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const K128* c = cand + (size_t)plane * cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&h[sel_bin(c[i])], 1u);
  __syncthreads();
  unsigned* g = ghist + (size_t)plane * kSelBins;
  for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
    if (h[i]) atomicAdd(&g[i], h[i]);
}

// per plane: threshold bin b* (the bin holding the K-th largest score; 0 when
// there are at most K candidates), bucket offsets of the bins >= b* (keys in
// higher bins first) and the kept-set size
__global__ void __launch_bounds__(1024) k_sel_thresh(const unsigned* __restrict__ cnt, size_t cap, int K,
                                                     const unsigned* __restrict__ ghist, int* __restrict__ bstar,
                                                     unsigned* __restrict__ bbase, unsigned* __restrict__ setn) {
  __shared__ unsigned part[1024];
  __shared__ int s_b;
  const int plane = blockIdx.x;
  const int n = (int)min((size_t)cnt[plane], cap);
  const unsigned* g = ghist + (size_t)plane * kSelBins;
  unsigned* bb = bbase + (size_t)plane * kSelBins;
  constexpr int per = kSelBins / 1024;          // bins per thread, thread 0 = highest bins
  const int b0 = kSelBins - per * (threadIdx.x + 1);
  unsigned s = 0;
  for (int i = 0; i < per; ++i) s += g[b0 + i];
  part[threadIdx.x] = s;
  if (threadIdx.x == 0) s_b = 0;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {    // inclusive scan from the top bins down
    const unsigned add = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += add;
    __syncthreads();
  }
  const unsigned above = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  unsigned run = above;
  for (int i = per - 1; i >= 0; --i) {          // highest bin of this thread first
    bb[b0 + i] = run;
    const unsigned nxt = run + g[b0 + i];
    if (n > K && run < (unsigned)K && nxt >= (unsigned)K) s_b = b0 + i;
    run = nxt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int bs = s_b;
    bstar[plane] = bs;
    setn[plane] = n <= K ? (unsigned)n : bb[bs] + g[bs];
  }
}

__global__ void __launch_bounds__(256) k_sel_scatter(const K128* __restrict__ cand, const unsigned* __restrict__ cnt,
                                                     size_t cap, const int* __restrict__ bstar,
                                                     const unsigned* __restrict__ bbase, unsigned* __restrict__ bfill,
                                                     K128* __restrict__ set) {
  const int plane = blockIdx.y;
  const int n = (int)min((size_t)cnt[plane], cap);
  const int bs = bstar[plane];
  const K128* c = cand + (size_t)plane * cap;
  const unsigned* bb = bbase + (size_t)plane * kSelBins;
  unsigned* bf = bfill + (size_t)plane * kSelBins;
  K128* o = set + (size_t)plane * cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const K128 k = c[i];
    const int bin = sel_bin(k);
    if (bin >= bs) o[bb[bin] + atomicAdd(&bf[bin], 1u)] = k;
  }
}

__global__ void __launch_bounds__(256) k_sel_rank(const K128* __restrict__ set, const unsigned* __restrict__ setn,
                                                  const unsigned* __restrict__ bbase,
                                                  const unsigned* __restrict__ ghist, size_t cap, int K,
                                                  K128* __restrict__ sorted, unsigned* __restrict__ nsel) {
  const int plane = blockIdx.y;
  const int n = (int)min((size_t)setn[plane], cap);
  const K128* s = set + (size_t)plane * cap;
  const unsigned* bb = bbase + (size_t)plane * kSelBins;
  const unsigned* g = ghist + (size_t)plane * kSelBins;
  if (blockIdx.x == 0 && threadIdx.x == 0) nsel[plane] = (unsigned)min(n, K);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const K128 mine = s[i];
    const int bin = sel_bin(mine);
    const unsigned lo = bb[bin], hi = lo + g[bin];
    if (lo >= (unsigned)K) continue;               // the whole bucket lies past K
    unsigned pos = lo;
    for (unsigned j = lo; j < hi; ++j) pos += k_less(s[j], mine) ? 1u : 0u;
    if (pos < (unsigned)K) sorted[(size_t)plane * K + pos] = mine;
  }
}

R2_DEV void write_kp(const K128& k, int idx, const DetectArgs& a, int b) {
  const size_t o = (size_t)b * a.max_points + idx;
  a.kp_y[o] = (int32_t)(k.lo >> 32);
  a.kp_x[o] = (int32_t)((k.lo >> 8) & 0xffffffull);
  a.kp_kind[o] = (uint8_t)(k.lo & 0xffull);
  a.kp_resp[o] = __longlong_as_double((long long)~k.hi);
}

__global__ void __launch_bounds__(1024) k_emit_single(const K128* __restrict__ sorted, const unsigned* __restrict__ nsel,
                                                      DetectArgs a) {
  const int b = blockIdx.x;
  const int m = nsel[b];
  for (int i = threadIdx.x; i < m; i += blockDim.x) write_kp(sorted[(size_t)b * a.max_points + i], i, a, b);
  if (threadIdx.x == 0) a.kp_count[b] = m;
}

R2_DEV unsigned hash_pix(unsigned p, unsigned mask) { return (p * 2654435761u) & mask; }

// Greedy 2-px suppression (ref: detector.py:116-137) as a priority MIS:
// a point is accepted once every higher-priority neighbour is rejected and
// rejected as soon as one of them is accepted; rounds repeat to a fixpoint,
// which equals the sequential greedy walk.  Three kernels: placement of
// every key in the merged (corners + edges) order plus a pixel hash, the
// neighbour lists, and the MIS rounds with the ordered compaction (one CTA
// per image).

// merged position of each key (binary search in the other list; a corner
// precedes an equal edge key, as in a merge taking ties from the first
// list) and its pixel -> position hash entry
__global__ void __launch_bounds__(256) k_merge_place(const K128* __restrict__ sorted, const unsigned* __restrict__ nsel,
                                                     K128* __restrict__ merged, int* __restrict__ hkey,
                                                     int* __restrict__ hval, int tsz, int W, int K) {
  const int b = blockIdx.y;
  const int nc = nsel[2 * b], ne = nsel[2 * b + 1];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nc + ne) return;
  const K128* corners = sorted + (size_t)(2 * b) * K;
  const K128* edges = sorted + (size_t)(2 * b + 1) * K;
  const bool is_c = e < nc;
  const int i = is_c ? e : e - nc;
  const K128 k = is_c ? corners[i] : edges[i];
  const K128* other = is_c ? edges : corners;
  int lo = 0, hi = is_c ? ne : nc;
  while (lo < hi) {                               // first other key not before k
    const int m = (lo + hi) >> 1;
    if (is_c ? k_less(other[m], k) : k_leq(other[m], k)) lo = m + 1; else hi = m;
  }
  const int pos = i + lo;
  merged[(size_t)b * 2 * K + pos] = k;
  const int pix = (int)(k.lo >> 32) * W + (int)((k.lo >> 8) & 0xffffffull);
  int* hk = hkey + (size_t)b * tsz;
  const unsigned mask = (unsigned)tsz - 1;
  unsigned h = hash_pix((unsigned)pix, mask);
  while (atomicCAS(&hk[h], -1, pix) != -1) h = (h + 1) & mask;
  hval[(size_t)b * tsz + h] = pos;
}

// higher-priority keys within distance 2 of each key (-1 terminated)
__global__ void __launch_bounds__(256) k_merge_nbr(const unsigned* __restrict__ nsel, const K128* __restrict__ merged,
                                                   const int* __restrict__ hkey, const int* __restrict__ hval,
                                                   int tsz, int* __restrict__ nbr, int W, int K) {
  const int b = blockIdx.y;
  const int n = nsel[2 * b] + nsel[2 * b + 1];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int* hk = hkey + (size_t)b * tsz;
  const int* hv = hval + (size_t)b * tsz;
  int* nb = nbr + ((size_t)b * 2 * K + i) * kMaxNbr;
  const unsigned mask = (unsigned)tsz - 1;
  const K128 k = merged[(size_t)b * 2 * K + i];
  const int y = (int)(k.lo >> 32), x = (int)((k.lo >> 8) & 0xffffffull);
  int cntn = 0;
  for (int dy = -2; dy <= 2; ++dy)
    for (int dx = -2; dx <= 2; ++dx) {
      if (dx * dx + dy * dy > 4) continue;
      const int yy = y + dy, xx = x + dx;
      if (yy < 0 || xx < 0 || xx >= W) continue;
      const int pix = yy * W + xx;
      unsigned h = hash_pix((unsigned)pix, mask);
      int key;
      while ((key = hk[h]) != -1) {
        if (key == pix) {
          const int j = hv[h];
          if (j < i && cntn < kMaxNbr) nb[cntn++] = j;
        }
        h = (h + 1) & mask;
      }
    }
  if (cntn < kMaxNbr) nb[cntn] = -1;
}

__global__ void __launch_bounds__(1024) k_merge_mis(const unsigned* __restrict__ nsel, const K128* __restrict__ merged,
                                                    const int* __restrict__ nbr, DetectArgs a) {
  extern __shared__ unsigned char s_status[];   // 0 undecided, 1 accepted, 2 rejected
  __shared__ int s_flag;
  __shared__ int s_base;
  __shared__ int s_warp[32];
  const int b = blockIdx.x;
  const int K = a.max_points;
  const int n = nsel[2 * b] + nsel[2 * b + 1];
  const K128* mg = merged + (size_t)b * 2 * K;
  const int* nb = nbr + (size_t)b * 2 * K * kMaxNbr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_status[i] = nb[(size_t)i * kMaxNbr] == -1 ? 1 : 0;
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (s_status[i] != 0) continue;
      bool all_rej = true, any_acc = false;
      for (int q = 0; q < kMaxNbr; ++q) {
        const int j = nb[(size_t)i * kMaxNbr + q];
        if (j < 0) break;
        const unsigned char st = ((volatile unsigned char*)s_status)[j];
        if (st == 1) { any_acc = true; break; }
        if (st != 2) all_rej = false;
      }
      if (any_acc) s_status[i] = 2;
      else if (all_rej) s_status[i] = 1;
      else s_flag = 1;
    }
    __syncthreads();
    if (!s_flag) break;
    __syncthreads();
  }
  // ordered compaction of the accepted points, capped at K
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool acc = i < n && s_status[i] == 1;
    const unsigned bal = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const int t = s_warp[w]; s_warp[w] = run; run += t; }
      s_flag = run;
    }
    __syncthreads();
    if (acc) {
      const int pos = s_base + s_warp[wid] + __popc(bal & ((1u << lane) - 1u));
      if (pos < K) write_kp(mg[i], pos, a, b);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += s_flag;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.kp_count[b] = min(s_base, K);
}

struct DetectPlan {
  int P, K, tsz;
  size_t cap;
  size_t off_mm, off_cnt, off_nsel, off_cand, off_sorted, off_tmp, off_merged, off_hk, off_hv, off_nbr;
  size_t off_ghist, off_bstar, off_setcnt, off_set, off_bbase, off_bfill, total;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

DetectPlan plan_detect(int B, int H, int W, int K) {
  DetectPlan p{};
  p.P = 2 * B;
  p.K = K > 0 ? K : 1;
  p.cap = (size_t)H * W;
  int t = 1024;
  while (t < 4 * p.K) t <<= 1;
  p.tsz = t;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = al(off + bytes); return o; };
  p.off_mm = take((size_t)p.P * 2 * sizeof(unsigned long long));
  p.off_cnt = take((size_t)p.P * sizeof(unsigned));
  p.off_nsel = take((size_t)p.P * sizeof(unsigned));
  p.off_cand = take((size_t)p.P * p.cap * sizeof(K128));
  p.off_sorted = take((size_t)p.P * p.K * sizeof(K128));
  p.off_tmp = take((size_t)p.P * p.K * sizeof(K128));
  p.off_merged = take((size_t)B * 2 * p.K * sizeof(K128));
  p.off_hk = take((size_t)B * p.tsz * sizeof(int));
  p.off_hv = take((size_t)B * p.tsz * sizeof(int));
  p.off_nbr = take((size_t)B * 2 * p.K * kMaxNbr * sizeof(int));
  p.off_ghist = take((size_t)p.P * kSelBins * sizeof(unsigned));
  p.off_bstar = take((size_t)p.P * sizeof(int));
  p.off_setcnt = take((size_t)p.P * sizeof(unsigned));
  p.off_set = take((size_t)p.P * p.cap * sizeof(K128));
  p.off_bbase = take((size_t)p.P * kSelBins * sizeof(unsigned));
  p.off_bfill = take((size_t)p.P * kSelBins * sizeof(unsigned));
  p.total = off;
  return p;
}

template <class T>
int detect_impl(const T* mins, const T* maxs, const DetectArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  const DetectPlan p = plan_detect(a.B, a.H, a.W, a.max_points);
  if (ws_bytes < p.total) return 1;
  char* w = static_cast<char*>(ws);
  auto* mm = reinterpret_cast<unsigned long long*>(w + p.off_mm);
  auto* cnt = reinterpret_cast<unsigned*>(w + p.off_cnt);
  auto* nsel = reinterpret_cast<unsigned*>(w + p.off_nsel);
  auto* cand = reinterpret_cast<K128*>(w + p.off_cand);
  auto* sorted = reinterpret_cast<K128*>(w + p.off_sorted);
  auto* tmp = reinterpret_cast<K128*>(w + p.off_tmp);
  auto* merged = reinterpret_cast<K128*>(w + p.off_merged);
  auto* hk = reinterpret_cast<int*>(w + p.off_hk);
  auto* hv = reinterpret_cast<int*>(w + p.off_hv);
  auto* nbr = reinterpret_cast<int*>(w + p.off_nbr);
  const int nm = a.single_map ? 1 : 2;
  const int planes = a.B * nm;
  if (a.max_points == 0) {
    cudaMemsetAsync(a.kp_count, 0, sizeof(int32_t) * a.B, st);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
  }
  k_init<<<(planes + 255) / 256, 256, 0, st>>>(mm, cnt, planes);
  const size_t n = (size_t)a.H * a.W;
  if (a.range) {
    // the filter bank already reduced the maps (same key format, same plane order)
    cudaMemcpyAsync(mm, a.range, (size_t)planes * 2 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st);
  } else {
    dim3 grid((unsigned)min((size_t)64, (n + 1023) / 1024), planes);
    k_minmax<T><<<grid, 256, 0, st>>>(mins, maxs, nm, n, mm);
  }
  {
    dim3 grid((a.W + kTile - 1) / kTile, (a.H + kTileY - 1) / kTileY, planes);
    // 6 resident CTAs of ~30 KB static shared memory: ask for the full carveout
    static const bool carveout = cudaFuncSetAttribute(k_fast_nms<T>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                      cudaSharedmemCarveoutMaxShared) == cudaSuccess;
    (void)carveout;
    k_fast_nms<T><<<grid, 256, 0, st>>>(mins, maxs, a.H, a.W, mm, a.threshold, a.margin, nm, cand, cnt, p.cap);
  }
  {
    auto* ghist = reinterpret_cast<unsigned*>(w + p.off_ghist);
    auto* bstar = reinterpret_cast<int*>(w + p.off_bstar);
    auto* setn = reinterpret_cast<unsigned*>(w + p.off_setcnt);
    auto* set = reinterpret_cast<K128*>(w + p.off_set);
    auto* bbase = reinterpret_cast<unsigned*>(w + p.off_bbase);
    auto* bfill = reinterpret_cast<unsigned*>(w + p.off_bfill);
    (void)tmp;
    cudaMemsetAsync(ghist, 0, (size_t)planes * kSelBins * sizeof(unsigned), st);
    cudaMemsetAsync(bfill, 0, (size_t)planes * kSelBins * sizeof(unsigned), st);
    k_sel_hist<<<dim3(kSelCtas, planes), 256, 0, st>>>(cand, cnt, p.cap, ghist);
    k_sel_thresh<<<planes, 1024, 0, st>>>(cnt, p.cap, a.max_points, ghist, bstar, bbase, setn);
    k_sel_scatter<<<dim3(kSelCtas, planes), 256, 0, st>>>(cand, cnt, p.cap, bstar, bbase, bfill, set);
    const int rank_ctas = (int)min((size_t)64, ((size_t)2 * a.max_points + 255) / 256);
    k_sel_rank<<<dim3(rank_ctas, planes), 256, 0, st>>>(set, setn, bbase, ghist, p.cap, a.max_points, sorted, nsel);
  }
  if (a.single_map) {
    k_emit_single<<<a.B, 1024, 0, st>>>(sorted, nsel, a);
  } else {
    const size_t smem = (size_t)2 * a.max_points;
    const dim3 g2((2 * a.max_points + 255) / 256, a.B);
    cudaMemsetAsync(hk, 0xFF, (size_t)a.B * p.tsz * sizeof(int), st);   // empty slots = -1
    k_merge_place<<<g2, 256, 0, st>>>(sorted, nsel, merged, hk, hv, p.tsz, a.W, a.max_points);
    k_merge_nbr<<<g2, 256, 0, st>>>(nsel, merged, hk, hv, p.tsz, nbr, a.W, a.max_points);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_merge_mis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_merge_mis<<<a.B, 1024, smem, st>>>(nsel, merged, nbr, a);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

size_t detect_workspace_bytes(int B, int H, int W, int max_points) {
  return plan_detect(B, H, W, max_points).total;
}

int detect_run(const float* mins, const float* maxs, const DetectArgs& a, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  return detect_impl(mins, maxs, a, ws, ws_bytes, st);
}

int detect_run(const double* mins, const double* maxs, const DetectArgs& a, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  return detect_impl(mins, maxs, a, ws, ws_bytes, st);
}

}  // namespace r2
