// Single-CTA sort of 128-bit keys (ascending), used wherever the reference
// orders by a lexicographic tuple: keypoints by (-response, y, x, kind)
// (ref: detector.py:110,127,154) and matches by (dist, ref, tgt)
// (ref: matcher.py:143-146).  Keys are built so that unsigned (hi, lo)
// order equals the reference's tuple order, which makes the result
// independent of the sort's own stability.
#pragma once
#include "common.cuh"

namespace r2 {

struct K128 {
  unsigned long long hi, lo;
};

R2_DEV bool k_less(const K128& a, const K128& b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
R2_DEV bool k_leq(const K128& a, const K128& b) { return !k_less(b, a); }

constexpr int kSortChunk = 4096;   // keys per shared-memory bitonic chunk (64 KB)

// Bitonic sort of n <= kSortChunk keys held in shared memory (padded with max).
R2_DEV void bitonic_smem(K128* s, int n) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += blockDim.x) s[i] = K128{~0ull, ~0ull};
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const K128 a = s[i], b = s[p];
          const bool up = (i & k) == 0;
          if (up ? k_less(b, a) : k_less(a, b)) { s[i] = b; s[p] = a; }
        }
      }
      __syncthreads();
    }
  }
}

// Merge sorted a[0..na) and b[0..nb) into out, split evenly over the block
// (merge path).  Ties take from `a` first.
R2_DEV void merge_path_block(const K128* a, int na, const K128* b, int nb, K128* out) {
  const int total = na + nb;
  const int per = (total + blockDim.x - 1) / blockDim.x;
  const int d0 = min(total, (int)threadIdx.x * per);
  const int d1 = min(total, d0 + per);
  if (d0 >= d1) return;
  // find split i (+ j = d0 - i) with a[i-1] <= b[j] and b[j-1] < a[i]
  int lo = max(0, d0 - nb), hi = min(d0, na);
  while (lo < hi) {
    const int i = (lo + hi) >> 1;
    const int j = d0 - 1 - i;
    if (k_less(b[j], a[i])) hi = i; else lo = i + 1;
  }
  int i = lo, j = d0 - lo;
  for (int d = d0; d < d1; ++d) {
    const bool take_a = j >= nb || (i < na && k_leq(a[i], b[j]));
    out[d] = take_a ? a[i++] : b[j++];
  }
}

// Sort n keys in `data` (global memory) using `tmp` (n keys) as scratch and
// `s` (kSortChunk keys of shared memory).  Result ends up in `data`.
R2_DEV void sort_keys_block(K128* data, K128* tmp, int n, K128* s) {
  for (int c0 = 0; c0 < n; c0 += kSortChunk) {
    const int len = min(kSortChunk, n - c0);
    for (int i = threadIdx.x; i < len; i += blockDim.x) s[i] = data[c0 + i];
    __syncthreads();
    bitonic_smem(s, len);
    for (int i = threadIdx.x; i < len; i += blockDim.x) data[c0 + i] = s[i];
    __syncthreads();
  }
  K128* src = data;
  K128* dst = tmp;
  for (int w = kSortChunk; w < n; w <<= 1) {
    for (int s0 = 0; s0 < n; s0 += 2 * w) {
      const int na = min(w, n - s0);
      const int nb = max(0, min(w, n - s0 - w));
      merge_path_block(src + s0, na, src + s0 + na, nb, dst + s0);
    }
    __syncthreads();
    K128* t = src; src = dst; dst = t;
  }
  if (src != data) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) data[i] = src[i];
    __syncthreads();
  }
}

}  // namespace r2
