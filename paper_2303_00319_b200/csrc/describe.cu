// RIFT2 dominant-index descriptors (and the ring / plain baselines).
//
// Replaces ref: pkg/src/rift2/descriptor.py:85-254 and mim.py:58-136:
//   extract_patch (:85-125) with the rotated nearest-neighbour gather table
//   (_rotated_offsets :46-64, _gather_table :70-82), patch_histogram
//   (mim.py:58-66), dominant_indices (mim.py:69-91), recode / cyclic_shift
//   (mim.py:97-136), encode (:131-164), describe_rift2 (:179-216),
//   describe_ring (:219-236), describe_plain (:239-254).
//
// Descriptors are emitted as exact integer cell-histogram counts (the
// reference's float64 vector is counts / ||counts||, rebuilt bit-exactly by
// the host layer when the dataclass API is used).
//
//   k_desc_plan  one CTA per keypoint: base-patch cell counts (packed byte
//                counters per column thread, segmented warp reduction),
//                dominant index / runner-up, rotated-bbox skip test
//   k_desc_scan  per image: exclusive scan of descriptors per keypoint
//   k_desc_emit  one CTA per keypoint: recode (a per-cell permutation of the
//                base counts) or rotated gather + recode, fp16 rows out
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "describe.h"

namespace r2 {

namespace {

constexpr int kT = 256;
constexpr int kMaxCells = 16 * 16;
constexpr int kMaxDim = kMaxCells * 16;

struct KpPlan {
  int ndesc;
  int skipped;
  int pick[2];
};

struct GatherTables {
  const short2* off;     // [O][P*P] (dx, dy); angle index 0 unused
  const int4* bbox;      // [O] (dx_min, dx_max, dy_min, dy_max)
};

std::mutex g_mu;
std::unordered_map<long long, GatherTables> g_tables;

// Host: the reference's rotated sample offsets (float64, snapped cos/sin,
// nearest neighbour floor(u + 0.5)), ref: descriptor.py:46-82.
static double snap_h(double v) {
  if (std::fabs(v) < 1e-12) return 0.0;
  if (std::fabs(std::fabs(v) - 1.0) < 1e-12) return std::copysign(1.0, v);
  return v;
}

GatherTables gather_tables(int P, int O) {
  int dev = 0;
  cudaGetDevice(&dev);
  const long long key = ((long long)dev << 40) | ((long long)P << 16) | O;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_tables.find(key);
  if (it != g_tables.end()) return it->second;
  std::vector<short2> off((size_t)O * P * P);
  std::vector<int4> bbox(O);
  const double half = P / 2.0;
  for (int a = 0; a < O; ++a) {
    const double ang = a * (M_PI / O);
    const double c = snap_h(std::cos(ang)), s = snap_h(std::sin(ang));
    int4 bb = make_int4(1 << 30, -(1 << 30), 1 << 30, -(1 << 30));
    for (int i = 0; i < P; ++i) {
      const double v = i + 0.5 - half;
      for (int j = 0; j < P; ++j) {
        const double u = j + 0.5 - half;
        const int dx = (int)std::floor(c * u - s * v + 0.5);
        const int dy = (int)std::floor(s * u + c * v + 0.5);
        off[(size_t)a * P * P + i * P + j] = make_short2((short)dx, (short)dy);
        bb.x = std::min(bb.x, dx); bb.y = std::max(bb.y, dx);
        bb.z = std::min(bb.z, dy); bb.w = std::max(bb.w, dy);
      }
    }
    bbox[a] = bb;
  }
  GatherTables t{nullptr, nullptr};
  short2* d_off = nullptr;
  int4* d_bb = nullptr;
  if (cudaMalloc(&d_off, off.size() * sizeof(short2)) != cudaSuccess) return t;
  if (cudaMalloc(&d_bb, bbox.size() * sizeof(int4)) != cudaSuccess) return t;
  cudaMemcpy(d_off, off.data(), off.size() * sizeof(short2), cudaMemcpyHostToDevice);
  cudaMemcpy(d_bb, bbox.data(), bbox.size() * sizeof(int4), cudaMemcpyHostToDevice);
  t.off = d_off;
  t.bbox = d_bb;
  g_tables[key] = t;
  return t;
}

struct DescConst {
  int H, W, O, P, g, cs, cells, dim;
  double ratio;
  bool rotate;
  int mode;
  bool fast;           // cs is a power of two <= 32 and O <= 8
};

// Count per (cell, value) of a P x P sample grid read through `src(i, j)`
// (i = sample row, j = sample column) into smem cnt[cells * O].
template <class Src>
R2_DEV void cell_counts(const DescConst& c, Src src, unsigned* cnt) {
  for (int i = threadIdx.x; i < c.cells * c.O; i += kT) cnt[i] = 0;
  __syncthreads();
  const int ngrp = kT / c.P;
  const int grp = threadIdx.x / c.P, col = threadIdx.x % c.P;
  const bool active = grp < ngrp;
  for (int cr0 = 0; cr0 < c.g; cr0 += ngrp) {
    const int cr = cr0 + grp;
    const bool on = active && cr < c.g;
    unsigned long long acc = 0, acc2 = 0;
    if (on) {
      for (int r = 0; r < c.cs; ++r) {
        const int v = src(cr * c.cs + r, col);
        if (v >= 1 && v <= 8) acc += 1ull << (8 * (v - 1));
        else if (v > 8 && v <= 16) acc2 += 1ull << (8 * (v - 9));
      }
    }
    const int cell = cr * c.g + col / c.cs;
    if (c.fast) {
      // split into 16-bit fields and reduce across the cs column threads of the cell
      unsigned long long e = acc & 0x00ff00ff00ff00ffull, o = (acc >> 8) & 0x00ff00ff00ff00ffull;
      for (int m = 1; m < c.cs; m <<= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, m);
        o += __shfl_xor_sync(0xffffffffu, o, m);
      }
      if (on && (col % c.cs) == 0) {
        for (int v = 0; v < c.O; ++v) {
          const unsigned long long w = (v & 1) ? o : e;
          cnt[cell * c.O + v] = (unsigned)((w >> (16 * (v >> 1))) & 0xffffu);
        }
      }
    } else if (on) {
      for (int v = 0; v < c.O; ++v) {
        const unsigned n = v < 8 ? (unsigned)((acc >> (8 * v)) & 255u) : (unsigned)((acc2 >> (8 * (v - 8))) & 255u);
        if (n) atomicAdd(&cnt[cell * c.O + v], n);
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kT) k_desc_plan(const uint8_t* __restrict__ mim, DescribeArgs a, DescConst c,
                                                  GatherTables tab, KpPlan* __restrict__ plan,
                                                  unsigned short* __restrict__ base) {
  __shared__ unsigned cnt[kMaxDim];
  const int b = blockIdx.y, k = blockIdx.x;
  KpPlan* pl = plan + (size_t)b * a.kp_stride + k;
  if (k >= a.kp_count[b]) {
    if (threadIdx.x == 0) { pl->ndesc = 0; pl->skipped = 0; }
    return;
  }
  const int x = a.kp_x[(size_t)b * a.kp_stride + k], y = a.kp_y[(size_t)b * a.kp_stride + k];
  const int x0 = x + 1 - (c.P + 1) / 2, y0 = y + 1 - (c.P + 1) / 2;   // floor(kp + 1 - P/2)
  if (x0 < 0 || y0 < 0 || x0 + c.P > c.W || y0 + c.P > c.H) {
    if (threadIdx.x == 0) { pl->ndesc = 0; pl->skipped = 1; }
    return;
  }
  const uint8_t* m = mim + (size_t)b * c.H * c.W;
  cell_counts(c, [&](int i, int j) { return (int)__ldg(&m[(size_t)(y0 + i) * c.W + x0 + j]); }, cnt);
  unsigned short* bo = base + ((size_t)b * a.kp_stride + k) * c.cells * c.O;
  for (int i = threadIdx.x; i < c.cells * c.O; i += kT) bo[i] = (unsigned short)cnt[i];
  if (threadIdx.x < 32) {
    // patch histogram (ref: mim.py:58-66) = sum of the cell counts, warp-parallel
    unsigned hs[16];
    for (int v = 0; v < c.O; ++v) {
      unsigned s = 0;
      for (int q = threadIdx.x; q < c.cells; q += 32) s += cnt[q * c.O + v];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      hs[v] = s;
    }
    if (threadIdx.x != 0) return;
    KpPlan p{0, 0, {0, 0}};
    if (c.mode == 0) { p.ndesc = 1; p.pick[0] = 1; }
    else if (c.mode == 1) { p.ndesc = c.O; }
    else {
      // ref: mim.py:69-91 -- first argmax, runner-up if >= ratio * peak
      // (float64, inclusive), runner-up ties to the bin cyclically closest
      // after the peak.
      double hist[16];
      for (int v = 0; v < c.O; ++v) hist[v] = (double)hs[v];
      int pk = 0;
      for (int v = 1; v < c.O; ++v) if (hist[v] > hist[pk]) pk = v;
      double rv = -1.0;
      for (int v = 0; v < c.O; ++v) if (v != pk && hist[v] > rv) rv = hist[v];
      int picks[2] = {pk + 1, 0};
      int np = 1;
      if (rv >= c.ratio * hist[pk]) {
        int best = -1, bestd = 1 << 30;
        for (int v = 0; v < c.O; ++v) {
          if (v == pk || hist[v] != rv) continue;
          const int d = ((v - pk) % c.O + c.O) % c.O;
          if (d < bestd) { bestd = d; best = v; }
        }
        picks[1] = best + 1;
        np = 2;
      }
      for (int q = 0; q < np; ++q) {
        const int dom = picks[q];
        if (c.rotate && dom != 1) {
          const int4 bb = tab.bbox[dom - 1];
          if (x + bb.x < 0 || x + bb.y >= c.W || y + bb.z < 0 || y + bb.w >= c.H) { p.skipped++; continue; }
        }
        p.pick[p.ndesc++] = dom;
      }
    }
    *pl = p;
  }
}

__global__ void __launch_bounds__(1024) k_desc_scan(const KpPlan* __restrict__ plan, DescribeArgs a,
                                                    int* __restrict__ offs) {
  __shared__ int s_warp[32];
  __shared__ int s_base, s_skip, s_tot;
  const int b = blockIdx.x;
  const int n = a.kp_count[b];
  const KpPlan* pl = plan + (size_t)b * a.kp_stride;
  int* of = offs + (size_t)b * a.kp_stride;
  if (threadIdx.x == 0) { s_base = 0; s_skip = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const int v = i < n ? pl[i].ndesc : 0;
    if (i < n && pl[i].skipped) atomicAdd(&s_skip, pl[i].skipped);
    int incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const int t = s_warp[w]; s_warp[w] = run; run += t; }
      s_tot = run;
    }
    __syncthreads();
    if (i < n) of[i] = s_base + s_warp[wid] + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) s_base += s_tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) { a.count[b] = s_base; a.skipped[b] = s_skip; }
}

__global__ void __launch_bounds__(kT) k_desc_emit(const uint8_t* __restrict__ mim, DescribeArgs a, DescConst c,
                                                  GatherTables tab, const KpPlan* __restrict__ plan,
                                                  const unsigned short* __restrict__ base,
                                                  const int* __restrict__ offs) {
  __shared__ unsigned cnt[kMaxDim];
  __shared__ int s_sq;
  const int b = blockIdx.y, k = blockIdx.x;
  if (k >= a.kp_count[b]) return;
  const KpPlan pl = plan[(size_t)b * a.kp_stride + k];
  if (pl.ndesc == 0) return;
  const int x = a.kp_x[(size_t)b * a.kp_stride + k], y = a.kp_y[(size_t)b * a.kp_stride + k];
  const unsigned short* bi = base + ((size_t)b * a.kp_stride + k) * c.cells * c.O;
  const uint8_t* m = mim + (size_t)b * c.H * c.W;
  const int off0 = offs[(size_t)b * a.kp_stride + k];
  for (int j = 0; j < pl.ndesc; ++j) {
    const int slot = off0 + j;
    int variant, pivot;
    bool rotated = false;
    if (c.mode == 0) { variant = 1; pivot = 1; }
    else if (c.mode == 1) { variant = j + 1; pivot = j + 1; }
    else { variant = pl.pick[j]; pivot = variant; rotated = c.rotate && variant != 1; }
    if (rotated) {
      const short2* t = tab.off + (size_t)(variant - 1) * c.P * c.P;
      cell_counts(c, [&](int i, int jj) {
        const short2 d = __ldg(&t[i * c.P + jj]);
        return (int)__ldg(&m[(size_t)(y + d.y) * c.W + x + d.x]);
      }, cnt);
    } else {
      __syncthreads();
      for (int i = threadIdx.x; i < c.cells * c.O; i += kT) cnt[i] = bi[i];
      __syncthreads();
    }
    if (threadIdx.x == 0) s_sq = 0;
    __syncthreads();
    if (slot < a.cap) {
      __half* row = a.counts + ((size_t)b * a.cap + slot) * a.stride;
      int sq = 0;
      for (int i = threadIdx.x; i < a.stride; i += kT) {
        unsigned v = 0;
        if (i < c.dim) {
          // output bin (cell, w-1) holds input value v' with recode(v') = w:
          // v' = (w - 1 + pivot - 1) mod O + 1  (ref: mim.py:117-136)
          const int cell = i / c.O, w = i % c.O;
          const int src = (w + pivot - 1) % c.O;
          v = cnt[cell * c.O + src];
        }
        row[i] = __uint2half_rn(v);
        sq += (int)(v * v);
      }
      atomicAdd(&s_sq, sq);
      __syncthreads();
      if (threadIdx.x == 0) {
        const size_t o = (size_t)b * a.cap + slot;
        a.sqnorm[o] = s_sq;
        a.kp[o] = k;
        a.variant[o] = (uint8_t)variant;
      }
    }
    __syncthreads();
  }
}

struct DescPlanWs {
  size_t off_plan, off_base, off_offs, total;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

DescPlanWs plan_ws(int B, int S, int grid, int O) {
  DescPlanWs p{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = al(off + bytes); return o; };
  p.off_plan = take((size_t)B * S * sizeof(KpPlan));
  p.off_base = take((size_t)B * S * grid * grid * O * sizeof(unsigned short));
  p.off_offs = take((size_t)B * S * sizeof(int));
  p.total = off;
  return p;
}

}  // namespace

size_t describe_workspace_bytes(int B, int kp_stride, int grid, int O) {
  return plan_ws(B, kp_stride > 0 ? kp_stride : 1, grid, O).total;
}

int describe_run(const uint8_t* mim, const DescribeArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  const DescPlanWs p = plan_ws(a.B, a.kp_stride > 0 ? a.kp_stride : 1, a.grid, a.O);
  if (ws_bytes < p.total) return 1;
  DescConst c{};
  c.H = a.H; c.W = a.W; c.O = a.O; c.P = a.patch; c.g = a.grid; c.cs = a.patch / a.grid;
  c.cells = a.grid * a.grid; c.dim = c.cells * a.O;
  c.ratio = a.ratio; c.rotate = a.rotate; c.mode = a.mode;
  c.fast = (c.cs <= 32) && ((c.cs & (c.cs - 1)) == 0) && a.O <= 8;
  GatherTables tab = gather_tables(a.patch, a.O);
  if (!tab.off) return 3;
  char* w = static_cast<char*>(ws);
  auto* plan = reinterpret_cast<KpPlan*>(w + p.off_plan);
  auto* base = reinterpret_cast<unsigned short*>(w + p.off_base);
  auto* offs = reinterpret_cast<int*>(w + p.off_offs);
  if (a.kp_stride == 0) {
    cudaMemsetAsync(a.count, 0, sizeof(int32_t) * a.B, st);
    cudaMemsetAsync(a.skipped, 0, sizeof(int32_t) * a.B, st);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  dim3 grid(a.kp_stride, a.B);
  k_desc_plan<<<grid, kT, 0, st>>>(mim, a, c, tab, plan, base);
  k_desc_scan<<<a.B, 1024, 0, st>>>(plan, a, offs);
  k_desc_emit<<<grid, kT, 0, st>>>(mim, a, c, tab, plan, base, offs);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2
