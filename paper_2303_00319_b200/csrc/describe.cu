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
//   k_desc_main  one CTA per keypoint.  The MIM neighbourhood every sample of
//                the axis-aligned and rotated patches can touch is staged in
//                shared memory as bytes s = 5(v-1) (4 pixels per word op;
//                0xFF outside the image), so a sample counts as
//                acc += 1 << s into six 5-bit fields.  Four threads share a
//                cell (4 columns x cs rows each) and reduce with two shuffles.
//                With the larger workspace the axis-aligned counts come
//                instead from k_cell_sums (dense 16 x 16 window counts of
//                every pixel, 36 loads per keypoint) and only keypoints
//                with a rotated pick wait for the staged bytes.
//                Then dominant index / runner-up (every thread, from the
//                patch histogram), the rotated patch of each pick through a
//                host-built offset table, recode (a per-cell permutation), and
//                the rows written straight to their final, reference-ordered
//                slots: CTAs take keypoints in start order and find their
//                output offset by a decoupled look-back over the descriptor
//                counts the earlier keypoints publish.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "describe.h"
#include "tma.cuh"

namespace r2 {

namespace {

constexpr int kT = 160;   // 5 warps: 144 counting threads for the 6x6 grid of 16-px cells

// offsets are stored as uint16 dy*stride + dx + kOffBias: 8 bytes per four
// samples, so the four rotated angles' tables (72 KB at 96^2) mostly stay in L1
constexpr int kOffBias = 32768;
#ifndef R2_DESC_CARVE
#define R2_DESC_CARVE 100
#endif

#ifndef R2_DESC_SPREAD
#define R2_DESC_SPREAD 1
#endif
constexpr bool kDescSpread = R2_DESC_SPREAD;   // bank-aware sample order of the rotated tables
#ifndef R2_DESC_DENSE
#define R2_DESC_DENSE 1
#endif
constexpr bool kDescDense = R2_DESC_DENSE;     // axis-aligned patches from dense 16 x 16 cell sums

constexpr int kMaxOrientG = 16;   // the generic kernel's orientation limit (the C ABI's)

struct GatherTables {
  const uint16_t* soff;  // [O][P*P] dy*stride + dx + kOffBias into the staged region; angle 0 unused
  const int4* bbox;      // [O] (dx_min, dx_max, dy_min, dy_max)
  const double2* uv;     // [O][P*P] the reference's continuous offsets (ux, vy), float64
  int radius;            // max |offset| over all angles (and the axis crop)
  int stride;            // staged row length in bytes (multiple of 16)
  int4 hbbox[8];         // host copy of bbox
  double4 hbbf[kMaxOrientG];   // (ux_min, ux_max, vy_min, vy_max) per angle
};

std::mutex g_mu;
std::unordered_map<long long, GatherTables> g_tables;

// Host: the reference's rotated sample offsets (float64, snapped cos/sin,
// nearest neighbour floor(u + 0.5)), ref: descriptor.py:46-82.
double snap_h(double v) {
  if (std::fabs(v) < 1e-12) return 0.0;
  if (std::fabs(std::fabs(v) - 1.0) < 1e-12) return std::copysign(1.0, v);
  return v;
}

// Bank-aware order of the rotated samples.  k_desc_main's thread (cell, sub)
// reads 16 rows x 4 samples of its cell through the table, one byte gather per
// warp per (row, sample) slot; a cell's counts do not depend on which of its
// threads reads which sample, so each cell's 256 samples are dealt to its
// slots greedily such that the 32 lanes of a slot fall into distinct
// shared-memory banks (or the same word), over the four byte alignments the
// keypoint column can have.  In raster order a slot costs 2.65 wavefronts on
// average at 96^2 / 6 orientations; dealt this way 1.2.
void spread_banks(uint16_t* t, int P, int stride, int radius) {
  constexpr int CS = 16, TPC = CS / 4;
  const int g = P / CS, nthr = g * g * TPC;
  const int base = radius * stride + radius - kOffBias;   // byte address of the keypoint pixel (column shift 0)
  const int nwords = ((2 * radius + 2) * stride + 64) / 4;
  std::vector<uint16_t> out((size_t)P * P);
  std::vector<uint8_t> present(4 * (size_t)nwords);
  std::vector<int> touched;
  for (int w0 = 0; w0 < nthr; w0 += 32) {
    const int w1 = std::min(nthr, w0 + 32);
    const int c0 = w0 / TPC, c1 = (w1 - 1) / TPC;
    std::vector<std::vector<uint16_t>> pool(c1 - c0 + 1);
    for (int c = c0; c <= c1; ++c)
      for (int i = 0; i < CS; ++i)
        for (int j = 0; j < CS; ++j) pool[c - c0].push_back(t[((c / g) * CS + i) * P + (c % g) * CS + j]);
    for (int slot = 0; slot < CS * 4; ++slot) {
      int cnt[4][32] = {}, mx[4] = {};
      for (int tid = w0; tid < w1; ++tid) {
        auto& pl = pool[tid / TPC - c0];
        int best = 0, best_cost = 1 << 30;
        for (int q = 0; q < (int)pl.size(); ++q) {
          int cost = 0;
          for (int d = 0; d < 4; ++d) {
            const int wd = (base + pl[q] + d) >> 2, bk = wd & 31;
            const int n = cnt[d][bk] + (present[(size_t)d * nwords + wd] ? 0 : 1);
            cost += 100 * (std::max(n, mx[d]) - mx[d]) + n;
          }
          if (cost < best_cost) { best_cost = cost; best = q; }
        }
        const uint16_t v = pl[best];
        pl.erase(pl.begin() + best);
        for (int d = 0; d < 4; ++d) {
          const int wd = (base + v + d) >> 2, bk = wd & 31;
          uint8_t& p = present[(size_t)d * nwords + wd];
          if (!p) { p = 1; touched.push_back(d * nwords + wd); mx[d] = std::max(mx[d], ++cnt[d][bk]); }
        }
        const int cell = tid / TPC, sub = tid % TPC, r = slot / 4, k = slot % 4;
        out[((cell / g) * CS + r) * P + (cell % g) * CS + 4 * sub + k] = v;
      }
      for (int i : touched) present[i] = 0;
      touched.clear();
    }
  }
  std::copy(out.begin(), out.end(), t);
}

GatherTables gather_tables(int P, int O) {
  int dev = 0;
  cudaGetDevice(&dev);
  const long long key = ((long long)dev << 40) | ((long long)P << 16) | O;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_tables.find(key);
  if (it != g_tables.end()) return it->second;
  std::vector<int2> off((size_t)O * P * P);
  std::vector<double2> uv((size_t)O * P * P);
  std::vector<double4> bbf(O);
  std::vector<int4> bbox(O);
  const double half = P / 2.0;
  int radius = (P + 1) / 2;   // axis crop spans [x + 1 - (P+1)/2, x + P - (P+1)/2]
  for (int a = 0; a < O; ++a) {
    const double ang = a * (M_PI / O);
    const double c = snap_h(std::cos(ang)), s = snap_h(std::sin(ang));
    int4 bb = make_int4(1 << 30, -(1 << 30), 1 << 30, -(1 << 30));
    double4 bf = make_double4(1e300, -1e300, 1e300, -1e300);
    for (int i = 0; i < P; ++i) {
      const double v = i + 0.5 - half;
      for (int j = 0; j < P; ++j) {
        const double u = j + 0.5 - half;
        const double ux = c * u - s * v, vy = s * u + c * v;   // ref: descriptor.py:61-62
        uv[(size_t)a * P * P + i * P + j] = make_double2(ux, vy);
        bf.x = std::min(bf.x, ux); bf.y = std::max(bf.y, ux);
        bf.z = std::min(bf.z, vy); bf.w = std::max(bf.w, vy);
        const int dx = (int)std::floor(ux + 0.5);
        const int dy = (int)std::floor(vy + 0.5);
        off[(size_t)a * P * P + i * P + j] = make_int2(dx, dy);
        bb.x = std::min(bb.x, dx); bb.y = std::max(bb.y, dx);
        bb.z = std::min(bb.z, dy); bb.w = std::max(bb.w, dy);
      }
    }
    bbox[a] = bb;
    bbf[a] = bf;
    radius = std::max({radius, -bb.x, bb.y, -bb.z, bb.w});
  }
  // staged row pitch: 2R+1 bytes from a 16-aligned start (+15; TMA box x
  // coordinates must be 16-byte aligned), one spare word for the funnel-shift
  // reads (+4), rounded to 16 bytes for the TMA box
  const int stride = ((2 * radius + 1 + 15 + 4 + 15) / 16) * 16;
  GatherTables t{nullptr, nullptr, nullptr, radius, stride, {}, {}};
  for (int a = 0; a < O && a < 8; ++a) t.hbbox[a] = bbox[a];
  for (int a = 0; a < O && a < kMaxOrientG; ++a) t.hbbf[a] = bbf[a];
  double2* d_uv = nullptr;
  if (cudaMalloc(&d_uv, uv.size() * sizeof(double2)) != cudaSuccess) return t;
  cudaMemcpy(d_uv, uv.data(), uv.size() * sizeof(double2), cudaMemcpyHostToDevice);
  t.uv = d_uv;                                   // the generic kernel's tables
  // biased 16-bit offsets: a thread's four samples of a row are one 8-byte load
  std::vector<uint16_t> soff(off.size());
  bool fits = true;
  for (size_t i = 0; i < off.size(); ++i) {
    const int v = off[i].y * stride + off[i].x + kOffBias;
    if (v < 0 || v > 65535) { fits = false; break; }   // large patches: the generic kernel only
    soff[i] = (uint16_t)v;
  }
  if (!fits) { g_tables[key] = t; return t; }
  if (kDescSpread && P % 16 == 0)
    for (int a = 1; a < O; ++a) spread_banks(soff.data() + (size_t)a * P * P, P, stride, radius);
  uint16_t* d_off = nullptr;
  int4* d_bb = nullptr;
  if (cudaMalloc(&d_off, soff.size() * sizeof(uint16_t)) != cudaSuccess) return t;
  if (cudaMalloc(&d_bb, bbox.size() * sizeof(int4)) != cudaSuccess) return t;
  cudaMemcpy(d_off, soff.data(), soff.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
  cudaMemcpy(d_bb, bbox.data(), bbox.size() * sizeof(int4), cudaMemcpyHostToDevice);
  t.soff = d_off;
  t.bbox = d_bb;
  g_tables[key] = t;
  return t;
}

struct DescConst {
  int H, W, O, P, g, cs, cells, dim, per;
  double ratio;
  bool rotate;
  int mode;
  int R, stride, rows;   // staging radius, staged row bytes, staged rows (2R+1)
  int tma;               // stage the neighbourhood with one TMA box load
  int preshift;          // the TMA source already holds shift bytes 5(v-1) (k_mim_shift)
  const uint2* dense;    // 16 x 16 cell sums of every pixel (k_cell_sums), or nullptr: count the axis patch
  int4 bbox[8];          // per-angle rotated-patch bounding boxes (dx_min, dx_max, dy_min, dy_max)
};

// six 5-bit counters (<= 31 samples) -> 10-bit fields: values 1,3,5 into e, 2,4,6 into o
R2_DEV void widen(uint32_t acc, uint32_t& e, uint32_t& o) {
  e += (acc & 31u) | ((acc >> 10) & 31u) << 10 | ((acc >> 20) & 31u) << 20;
  o += ((acc >> 5) & 31u) | ((acc >> 15) & 31u) << 10 | ((acc >> 25) & 31u) << 20;
}

// reduce the 4 threads of a cell, write its O counts and add their squares
// to the descriptor's squared norm (recode only permutes bins)
// The patch histogram and the squared norm are reduced per warp (the
// histogram as three words of two 16-bit counts: <= 9,216 per value) and
// added to shared memory by one lane, instead of per-cell atomics on the same
// few addresses.  Every lane of the warp calls this.
template <int OT>
R2_DEV void reduce_cell(uint32_t e, uint32_t o, bool writer, unsigned* out, int O_rt, int* sq,
                        unsigned* hist = nullptr) {
  const int O = OT ? OT : O_rt;
  e += __shfl_xor_sync(0xffffffffu, e, 1);
  o += __shfl_xor_sync(0xffffffffu, o, 1);
  e += __shfl_xor_sync(0xffffffffu, e, 2);
  o += __shfl_xor_sync(0xffffffffu, o, 2);
  int q = 0;
  uint32_t h01 = 0, h23 = 0, h45 = 0;
  if (writer) {
#pragma unroll
    for (int v = 0; v < (OT ? OT : 8); ++v) {
      if (!OT && v >= O) break;
      const unsigned n = (((v & 1) ? o : e) >> (10 * (v >> 1))) & 1023u;
      out[v] = n;
      q += (int)(n * n);
    }
    // 16-bit packed histogram words: value v in word v / 2, half v % 2
    h01 = (e & 1023u) | (o & 1023u) << 16;
    h23 = ((e >> 10) & 1023u) | ((o >> 10) & 1023u) << 16;
    h45 = ((e >> 20) & 1023u) | ((o >> 20) & 1023u) << 16;
  }
  q = __reduce_add_sync(0xffffffffu, q);
  if (hist) {
    h01 = __reduce_add_sync(0xffffffffu, h01);
    h23 = __reduce_add_sync(0xffffffffu, h23);
    h45 = __reduce_add_sync(0xffffffffu, h45);
  }
  if ((threadIdx.x & 31) == 0) {
    if (q) atomicAdd(sq, q);
    if (hist) {
      if (h01) atomicAdd(&hist[0], h01);
      if (h23) atomicAdd(&hist[1], h23);
      if (h45) atomicAdd(&hist[2], h45);
    }
  }
}

// 1 << s for a staged shift byte; PTX shl clamps shifts >= 32 to a zero
// result, so out-of-image bytes (0xFF, or the garbage of a zero-filled TMA
// word) count nothing -- and they are never sampled by an emitted descriptor
R2_DEV uint32_t one_hot(uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(s));
  return r;
}

// axis-aligned patch: thread = (cell, quarter); 4 columns x CS rows per thread.
// OT / GT: orientation count and grid fixed at compile time (0 = runtime)
template <int CS, int OT, int GT>
R2_DEV void count_axis(const DescConst& c, const uint8_t* sreg, int off0, unsigned* cnt, int* sq, unsigned* hist) {
  const int tpc = CS / 4;                       // threads per cell
  const int g = GT ? GT : c.g, O = OT ? OT : c.O;
  const int t = threadIdx.x;
  const bool on = t < g * g * tpc;
  const int cell = on ? t / tpc : 0, sub = t % tpc;
  const int cr = cell / g, cc = cell % g;
  uint32_t e = 0, o = 0;
  if (on) {
    const int col = off0 + cc * CS + 4 * sub;   // byte offset of this thread's 4 columns within a row
    const int wbase = col >> 2, sh = (col & 3) * 8;
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(sreg) + (cr * CS) * (c.stride >> 2) + wbase;
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < CS; ++r) {
      const uint32_t* p = rw + r * (c.stride >> 2);
      const uint32_t w = __funnelshift_r(p[0], p[1], sh);
      acc += one_hot(w & 255u) + one_hot((w >> 8) & 255u) + one_hot((w >> 16) & 255u) + one_hot(w >> 24);
      if (r % 7 == 6 || r == CS - 1) { widen(acc, e, o); acc = 0; }   // 4 samples/row: <= 28 per field
    }
  }
  reduce_cell<OT>(e, o, on && sub == 0, cnt + cell * O, O, sq, hist);
}

// axis-aligned patch from the dense cell sums: cell (cr, cc) of the patch at
// (x0, y0) is the 16 x 16 window anchored at (x0 + 16 cc, y0 + 16 cr), whose
// per-value counts k_cell_sums left as two words of 10-bit fields (the e / o
// format of reduce_cell).  One thread per cell; warps 0 and 1 call this.
template <int OT, int GT>
R2_DEV void count_axis_dense(const DescConst& c, const uint2* __restrict__ cells, int x0, int y0, unsigned* cnt,
                             int* sq, unsigned* hist) {
  const int g = GT ? GT : c.g, O = OT ? OT : c.O;
  const int t = threadIdx.x;
  const bool on = t < g * g;
  int q = 0;
  uint32_t h01 = 0, h23 = 0, h45 = 0;
  if (on) {
    const int cr = t / g, cc = t % g;
    const uint2 w = __ldg(cells + (size_t)(y0 + 16 * cr) * c.W + x0 + 16 * cc);
    const uint32_t e = w.x, o = w.y;
#pragma unroll
    for (int v = 0; v < (OT ? OT : 8); ++v) {
      if (!OT && v >= O) break;
      const unsigned n = (((v & 1) ? o : e) >> (10 * (v >> 1))) & 1023u;
      cnt[t * O + v] = n;
      q += (int)(n * n);
    }
    h01 = (e & 1023u) | (o & 1023u) << 16;
    h23 = ((e >> 10) & 1023u) | ((o >> 10) & 1023u) << 16;
    h45 = ((e >> 20) & 1023u) | ((o >> 20) & 1023u) << 16;
  }
  q = __reduce_add_sync(0xffffffffu, q);
  h01 = __reduce_add_sync(0xffffffffu, h01);
  h23 = __reduce_add_sync(0xffffffffu, h23);
  h45 = __reduce_add_sync(0xffffffffu, h45);
  if ((t & 31) == 0) {
    if (q) atomicAdd(sq, q);
    if (h01) atomicAdd(&hist[0], h01);
    if (h23) atomicAdd(&hist[1], h23);
    if (h45) atomicAdd(&hist[2], h45);
  }
}

// rotated patch of angle table t: sample (i, j) at ctr + t[i*P + j]
template <int CS, int OT, int GT>
R2_DEV void count_rotated(const DescConst& c, const uint8_t* ctr, const uint16_t* __restrict__ t, unsigned* cnt,
                          int* sq) {
  const int tpc = CS / 4;
  const int g = GT ? GT : c.g, O = OT ? OT : c.O, P = GT ? GT * CS : c.P;
  const int tid = threadIdx.x;
  const bool on = tid < g * g * tpc;
  const int cell = on ? tid / tpc : 0, sub = tid % tpc;
  const int cr = cell / g, cc = cell % g;
  uint32_t e = 0, o = 0;
  if (on) {
    const uint2* tr = reinterpret_cast<const uint2*>(t + (cr * CS) * P + cc * CS + 4 * sub);
    const uint8_t* cb = ctr - kOffBias;
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < CS; ++r) {
      const uint2 a = __ldg(tr + r * (P / 4));
      acc += one_hot(cb[a.x & 0xffffu]) + one_hot(cb[a.x >> 16]) + one_hot(cb[a.y & 0xffffu]) + one_hot(cb[a.y >> 16]);
      if (r % 7 == 6 || r == CS - 1) { widen(acc, e, o); acc = 0; }
    }
  }
  reduce_cell<OT>(e, o, on && sub == 0, cnt + cell * O, O, sq);
}

// write one descriptor row: output bin (cell, w-1) holds the count of the
// input value v with recode(v) = w, i.e. v = (w - 1 + pivot - 1) mod O + 1
// (ref: mim.py:117-136)
template <int OT, int GT>
R2_DEV void emit_row(const DescribeArgs& a, const DescConst& c, const unsigned* cnt, int pivot, __half* row) {
  const int O = OT ? OT : c.O, dim = GT ? GT * GT * O : c.dim;
  for (int i = threadIdx.x; i < a.stride; i += kT) {
    unsigned v = 0;
    if (i < dim) {
      const int cell = i / O, w = i % O;
      const int u = w + pivot - 1;
      v = cnt[cell * O + (u >= O ? u - O : u)];
    }
    row[i] = __uint2half_rn(v);
  }
}

// 90-degree pick: with cos/sin snapped to (0, 1) the rotated sample (i, j)
// reads the axis-patch pixel (j, P-1-i) (ref: descriptor.py:46-82, P even), so
// rotated cell (R, C) is axis cell (C, g-1-R): a permutation of the axis
// counts, no gather
template <int OT, int GT>
R2_DEV void emit_row_rot90(const DescribeArgs& a, const DescConst& c, const unsigned* cnt, int pivot, __half* row) {
  const int O = OT ? OT : c.O, g = GT ? GT : c.g, dim = g * g * O;
  for (int i = threadIdx.x; i < a.stride; i += kT) {
    unsigned v = 0;
    if (i < dim) {
      const int cell = i / O, w = i % O;
      const int R = cell / g, C = cell % g;
      const int u = w + pivot - 1;
      v = cnt[(C * g + (g - 1 - R)) * O + (u >= O ? u - O : u)];
    }
    row[i] = __uint2half_rn(v);
  }
}

// decoupled look-back words: status in bits 63..62 (0 = not yet, 1 = this
// keypoint's descriptor count, 2 = inclusive prefix), value in bits 31..0
constexpr unsigned long long kChainAgg = 1, kChainPrefix = 2;
R2_DEV void chain_publish(unsigned long long* w, unsigned long long status, unsigned v) {
  atomicExch(w, (status << 62) | v);
}
R2_DEV unsigned long long chain_read(const unsigned long long* w) {
  return *reinterpret_cast<const volatile unsigned long long*>(w);
}

template <int CS, int OT, int GT>
__global__ void __launch_bounds__(kT) k_desc_main(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ mim, DescribeArgs a,
                                                  DescConst c, GatherTables tab,
                                                  unsigned long long* __restrict__ chain,
                                                  unsigned* __restrict__ ticket) {
  extern __shared__ __align__(128) uint32_t s_raw[];
  __shared__ uint64_t s_bar;
  // staged bytes (c.rows x c.stride, 128-byte aligned for the TMA box), then cnt
  uint32_t* s_dyn = s_raw + ((128u - (smem_u32(s_raw) & 127u)) & 127u) / 4;
  uint8_t* sreg = reinterpret_cast<uint8_t*>(s_dyn);
  // count buffers: axis patch, first and second rotated pick, [cells * O] each
  const int O = OT ? OT : c.O, cells = GT ? GT * GT : c.cells;
  unsigned* cnt = s_dyn + (c.rows * c.stride) / 4;
  unsigned* cnt_rot[2] = {cnt + cells * O, cnt + 2 * cells * O};
  __shared__ int s_sq[3];
  __shared__ unsigned s_hist[8];                  // axis-patch histogram (ref: mim.py:58-66)
  __shared__ int s_k;
  __shared__ unsigned s_excl;
  const int b = blockIdx.y;
  // mode 3 is the reference pipeline's ring mode (ref: pipeline.py:53-64):
  // the reference side (even blocks) ring, the target side (odd blocks) plain
  const int mode = c.mode == 3 ? ((b & 1) ? 0 : 1) : c.mode;
  // keypoints are taken in CTA start order (a per-image ticket), so every
  // keypoint before this one belongs to a CTA that has already started: the
  // look-back below only waits on running CTAs
  if (threadIdx.x == 0) s_k = (int)atomicAdd(&ticket[b], 1u);
  __syncthreads();
  const int k = s_k;
  if (k >= min(a.kp_count[b], a.kp_stride)) return;   // no live keypoint follows
  unsigned long long* lb = chain + (size_t)b * a.kp_stride;
  const int x = a.kp_x[(size_t)b * a.kp_stride + k], y = a.kp_y[(size_t)b * a.kp_stride + k];
  const int x0 = x + 1 - (c.P + 1) / 2, y0 = y + 1 - (c.P + 1) / 2;   // floor(kp + 1 - P/2)
  if (x0 < 0 || y0 < 0 || x0 + c.P > c.W || y0 + c.P > c.H) {
    if (threadIdx.x == 0) {                       // skipped (ref: descriptor.py:196-198): no rows
      chain_publish(&lb[k], kChainAgg, 0u);
      atomicAdd(&a.skipped[b], 1);
    }
    return;
  }
  const uint8_t* m = mim + (size_t)b * c.H * c.W;
  // ---- stage rows y-R..y+R, word-aligned columns from ax0, as shift bytes 5(v-1)
  const int ax0 = (x - c.R) & (c.tma ? ~15 : ~3);   // floor to 16 (TMA) / 4 bytes
  const int wpr = c.stride / 4;
  const bool word_ok = (c.W & 3) == 0;
  uint32_t* sw = s_dyn;
  const bool inside = word_ok && y - c.R >= 0 && y + c.R < c.H && ax0 >= 0 && ax0 + 4 * wpr <= c.W;
  if (c.tma) {
    // one TMA box (zero fill left/right of the image, neighbouring images'
    // rows above/below; W % 16 == 0 and a 16-aligned start, so out-of-image
    // bytes form whole words and the per-word transform cannot borrow into
    // an image byte), then an in-place shift-byte transform
    if (threadIdx.x == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(&tmap) : "memory");
      mbar_init(&s_bar, 1);
      mbar_fence_init();
      mbar_expect_tx(&s_bar, (uint32_t)(c.rows * c.stride));
      tma_load_2d(sw, &tmap, ax0, b * c.H + y - c.R, &s_bar);
    }
    if (threadIdx.x < 8) s_hist[threadIdx.x] = 0;
    if (threadIdx.x == 0) { s_sq[0] = 0; s_sq[1] = 0; s_sq[2] = 0; }
    __syncthreads();
    // (with the dense cell sums the staged bytes are only needed by rotated
    // picks: waited for below, once the picks are known)
    if (!c.dense) mbar_wait(&s_bar, 0);
    uint4* q4 = reinterpret_cast<uint4*>(sw);
    if (!c.preshift)
    for (int i = threadIdx.x; i < c.rows * c.stride / 16; i += kT) {
      uint4 w = q4[i];
      w.x = w.x * 5u - 0x05050505u;
      w.y = w.y * 5u - 0x05050505u;
      w.z = w.z * 5u - 0x05050505u;
      w.w = w.w * 5u - 0x05050505u;
      q4[i] = w;
    }
  } else if (inside) {
    // common case: one aligned word load + one multiply-add per 4 pixels
    const uint32_t* src0 = reinterpret_cast<const uint32_t*>(m + (size_t)(y - c.R) * c.W + ax0);
    const int wrow = c.W >> 2;
    for (int r = threadIdx.x >> 5; r < c.rows; r += kT / 32) {
      const uint32_t* src = src0 + r * wrow;
      uint32_t* dst = sw + r * wpr;
      for (int wq = threadIdx.x & 31; wq < wpr; wq += 32) dst[wq] = __ldg(src + wq) * 5u - 0x05050505u;
    }
  } else for (int r = threadIdx.x >> 5; r < c.rows; r += kT / 32) {
    const int gy = y - c.R + r;
    const bool row_in = gy >= 0 && gy < c.H;
    const uint8_t* row = m + (size_t)(row_in ? gy : 0) * c.W;
    for (int wq = threadIdx.x & 31; wq < wpr; wq += 32) {
      const int gx = ax0 + 4 * wq;
      uint32_t v = 0xffffffffu;
      if (row_in) {
        if (word_ok && gx >= 0 && gx + 3 < c.W) {
          v = __ldg(reinterpret_cast<const uint32_t*>(row + gx)) * 5u - 0x05050505u;
        } else {
          v = 0;
          for (int e = 0; e < 4; ++e) {
            const int xx = gx + e;
            const uint32_t s = (xx >= 0 && xx < c.W) ? (uint32_t)(5 * (row[xx] - 1)) & 255u : 255u;
            v |= s << (8 * e);
          }
        }
      }
      sw[r * wpr + wq] = v;
    }
  }
  if (!c.tma && threadIdx.x < 8) s_hist[threadIdx.x] = 0;
  if (!c.tma && threadIdx.x == 0) { s_sq[0] = 0; s_sq[1] = 0; s_sq[2] = 0; }
  __syncthreads();
  const int bx = x - ax0;                         // keypoint column within a staged row
  const uint8_t* ctr = sreg + c.R * c.stride + bx;   // keypoint pixel
  // ---- axis-aligned patch
  if (c.dense) {
    if (threadIdx.x < 64) count_axis_dense<OT, GT>(c, c.dense + (size_t)b * c.H * c.W, x0, y0, cnt, &s_sq[0], s_hist);
  } else {
    count_axis<CS, OT, GT>(c, sreg + (c.R + y0 - y) * c.stride, bx + x0 - x, cnt, &s_sq[0], s_hist);
  }
  __syncthreads();
  // ---- dominant index / runner-up (ref: mim.py:69-91), computed by every
  // thread from the 6-bin patch histogram (no extra barrier)
  constexpr int kMaxPick = OT ? (OT > 2 ? OT : 2) : 8;
  int pick[kMaxPick];
  int np = 0;
  {
    unsigned hs[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) hs[v] = v < O ? (s_hist[v >> 1] >> (16 * (v & 1))) & 0xffffu : 0u;
    int skip = 0;
    if (mode == 0) { pick[np++] = 1; }
    else if (mode == 1) {
#pragma unroll
      for (int v = 1; v <= kMaxPick; ++v) if (v <= O) pick[np++] = v;
    } else {
      // first argmax; runner-up if >= ratio * peak (float64, inclusive);
      // runner-up ties go to the bin cyclically closest after the peak
      int pk = 0;
#pragma unroll
      for (int v = 1; v < 8; ++v) if (v < O && hs[v] > hs[pk]) pk = v;
      // (counts are integers: only the ratio test needs float64)
      int rv = -1;
#pragma unroll
      for (int v = 0; v < 8; ++v) if (v < O && v != pk && (int)hs[v] > rv) rv = (int)hs[v];
      int picks[2] = {pk + 1, 0}, cand = 1;
      if (rv >= 0 && (double)rv >= c.ratio * (double)hs[pk]) {
        int best = -1, bestd = 1 << 30;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          if (v >= O || v == pk || (int)hs[v] != rv) continue;
          const int d = v > pk ? v - pk : v - pk + O;
          if (d < bestd) { bestd = d; best = v; }
        }
        picks[1] = best + 1;
        cand = 2;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (q >= cand) break;
        const int dom = picks[q];
        if (c.rotate && dom != 1) {
          const int4 bb = c.bbox[dom - 1];
          if (x + bb.x < 0 || x + bb.y >= c.W || y + bb.z < 0 || y + bb.w >= c.H) { ++skip; continue; }
        }
        pick[np++] = dom;
      }
    }
    if (threadIdx.x == 0) {
      chain_publish(&lb[k], kChainAgg, (unsigned)np);   // successors may look back through us now
      if (skip) atomicAdd(&a.skipped[b], skip);
      if (np) atomicAdd(&a.count[b], np);
    }
  }
  // count the rotated picks (at most two) into their own buffers
  const bool rot_mode = mode == 2 && c.rotate;
  const int dom90 = (O % 2 == 0 && c.P % 2 == 0) ? O / 2 + 1 : -1;
  int nrot = 0;
  bool need_rot = false;
#pragma unroll
  for (int q = 0; q < kMaxPick; ++q)
    if (q < np && rot_mode && pick[q] != 1 && pick[q] != dom90) need_rot = true;
  // the staged neighbourhood: every thread that gathers from it waits for the
  // TMA box; a keypoint with no rotated pick never reads it, and thread 0
  // alone sees the load land before the CTA gives its shared memory back
  if (c.dense && need_rot) mbar_wait(&s_bar, 0);
#pragma unroll
  for (int q = 0; q < kMaxPick; ++q) {
    if (q >= np) break;
    const int dom = pick[q];
    if (rot_mode && dom != 1 && dom != dom90) {
      count_rotated<CS, OT, GT>(c, ctr, tab.soff + (size_t)(dom - 1) * c.P * c.P, cnt_rot[nrot], &s_sq[1 + nrot]);
      ++nrot;
    }
  }
  // output position: exclusive prefix of the descriptor counts of the keypoints
  // before this one (decoupled look-back over their published counts)
  if (threadIdx.x < 32) {
    // warp-wide look-back: 32 predecessors per step; stop at the nearest
    // inclusive prefix, add the counts after it
    const unsigned lane = threadIdx.x;
    unsigned excl = 0;
    for (int base = k - 1; base >= 0; base -= 32) {
      const int j = base - (int)lane;
      unsigned long long f = 2ull << 62;          // before keypoint 0: prefix 0
      if (j >= 0) do { f = chain_read(&lb[j]); } while ((f >> 62) == 0);
      const unsigned pre = __ballot_sync(0xffffffffu, (f >> 62) == kChainPrefix);
      const int stop = pre ? __ffs(pre) - 1 : 32;   // nearest prefix: the lowest lane
      unsigned v = (int)lane <= stop ? (unsigned)f : 0u;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      excl += v;
      if (pre) break;
    }
    if (lane == 0) {
      chain_publish(&lb[k], kChainPrefix, excl + (unsigned)np);
      s_excl = excl;
    }
  }
  __syncthreads();
  // rows straight into their final slots, in pick order (ref: descriptor.py:199-216)
  const unsigned excl = s_excl;
  int r = 0;
#pragma unroll
  for (int q = 0; q < kMaxPick; ++q) {
    if (q >= np) break;
    const int dom = pick[q];
    const unsigned dst = excl + q;
    const bool rotated = rot_mode && dom != 1 && dom != dom90;
    if (dst < (unsigned)a.cap) {
      const size_t o = (size_t)b * a.cap + dst;
      __half* row = a.counts + o * a.stride;
      const int var = mode == 0 ? 1 : dom;
      if (rot_mode && dom == dom90) emit_row_rot90<OT, GT>(a, c, cnt, dom, row);
      else emit_row<OT, GT>(a, c, rotated ? cnt_rot[r] : cnt, var, row);
      if (threadIdx.x == 0) {
        a.sqnorm[o] = rotated ? s_sq[1 + r] : s_sq[0];
        a.kp[o] = k;
        a.variant[o] = (uint8_t)var;
      }
    }
    if (rotated) ++r;
  }
  if (c.dense && !need_rot && threadIdx.x == 0) mbar_wait(&s_bar, 0);
}

// ---------------------------------------------------------------------------
// Generic descriptor kernel: any orientation count (<= 16), any cell size,
// and keypoints with fractional coordinates (ref: descriptor.py:85-125: the
// axis crop at floor(x + 1 - P/2), rotated samples at floor(x + ux + 0.5)
// in float64 from the continuous offsets; integer keypoints take the
// reference's integer table path floor(ux + 0.5) + x).  One CTA per
// keypoint, straight from the global index map, counts by shared-memory
// atomics: the BASELINE configuration (6 orientations, 16-px cells, integer
// keypoints from the detector) runs on k_desc_main; this covers the rest of
// the reference's parameter space exactly.
struct DescConstG {
  int H, W, O, P, g, cs, cells, dim;
  double ratio;
  bool rotate;
  int mode;
  double4 bbf[kMaxOrientG];   // continuous offset bounds per angle
};

constexpr int kTG = 256;

R2_DEV void count_patch_g(const uint8_t* m, const DescConstG& c, const DescribeArgs& a, int y0, int x0,
                          const double2* uv, double xd, double yd, bool integral, unsigned* cnt) {
  const int P = c.P;
  for (int idx = threadIdx.x; idx < P * P; idx += kTG) {
    const int i = idx / P, j = idx - i * P;
    int sy, sx;
    if (!uv) {
      sy = y0 + i;
      sx = x0 + j;
    } else {
      const double2 o = __ldg(&uv[idx]);
      if (integral) {
        sx = (int)xd + (int)floor(o.x + 0.5);
        sy = (int)yd + (int)floor(o.y + 0.5);
      } else {
        sx = (int)floor(__dadd_rn(__dadd_rn(xd, o.x), 0.5));
        sy = (int)floor(__dadd_rn(__dadd_rn(yd, o.y), 0.5));
      }
    }
    const int v = m[(size_t)sy * c.W + sx];   // 1..O; anything else counts nothing
    const int cell = (i / c.cs) * c.g + j / c.cs;
    if (v >= 1 && v <= c.O) atomicAdd(&cnt[cell * c.O + v - 1], 1u);
  }
}

// bounds of a rotated patch (monotone in the offset: the extreme samples
// come from the extreme offsets), ref: descriptor.py:118-125
R2_DEV bool rotated_inside(const DescConstG& c, int ang, double xd, double yd, bool integral) {
  const double4 b = c.bbf[ang];
  int x_lo, x_hi, y_lo, y_hi;
  if (integral) {
    x_lo = (int)xd + (int)floor(b.x + 0.5); x_hi = (int)xd + (int)floor(b.y + 0.5);
    y_lo = (int)yd + (int)floor(b.z + 0.5); y_hi = (int)yd + (int)floor(b.w + 0.5);
  } else {
    x_lo = (int)floor(__dadd_rn(__dadd_rn(xd, b.x), 0.5)); x_hi = (int)floor(__dadd_rn(__dadd_rn(xd, b.y), 0.5));
    y_lo = (int)floor(__dadd_rn(__dadd_rn(yd, b.z), 0.5)); y_hi = (int)floor(__dadd_rn(__dadd_rn(yd, b.w), 0.5));
  }
  return x_lo >= 0 && x_hi < c.W && y_lo >= 0 && y_hi < c.H;
}

template <bool FKP>
__global__ void __launch_bounds__(kTG) k_desc_generic(const uint8_t* __restrict__ mim, DescribeArgs a, DescConstG c,
                                                      const double2* __restrict__ uv,
                                                      unsigned long long* __restrict__ chain,
                                                      unsigned* __restrict__ ticket) {
  extern __shared__ unsigned s_cnt[];           // [3][cells * O]: axis patch, rotated picks 0 and 1
  __shared__ unsigned s_hist[kMaxOrientG];
  __shared__ int s_pick[kMaxOrientG];
  __shared__ int s_np, s_k;
  __shared__ unsigned s_excl;
  const int b = blockIdx.y;
  const int mode = c.mode == 3 ? ((b & 1) ? 0 : 1) : c.mode;   // see k_desc_main
  if (threadIdx.x == 0) s_k = (int)atomicAdd(&ticket[b], 1u);
  __syncthreads();
  const int k = s_k;
  if (k >= min(a.kp_count[b], a.kp_stride)) return;
  unsigned long long* lb = chain + (size_t)b * a.kp_stride;
  const size_t ki = (size_t)b * a.kp_stride + k;
  const double xd = FKP ? a.kp_xd[ki] : (double)a.kp_x[ki];
  const double yd = FKP ? a.kp_yd[ki] : (double)a.kp_y[ki];
  const bool integral = !FKP || (xd == floor(xd) && yd == floor(yd));
  const int x0 = (int)floor(xd + 1.0 - c.P / 2.0), y0 = (int)floor(yd + 1.0 - c.P / 2.0);
  if (x0 < 0 || y0 < 0 || x0 + c.P > c.W || y0 + c.P > c.H) {
    if (threadIdx.x == 0) {
      chain_publish(&lb[k], kChainAgg, 0u);
      atomicAdd(&a.skipped[b], 1);
    }
    return;
  }
  const int nb = c.cells * c.O;
  const uint8_t* m = mim + (size_t)b * c.H * c.W;
  for (int i = threadIdx.x; i < 3 * nb; i += kTG) s_cnt[i] = 0;
  __syncthreads();
  count_patch_g(m, c, a, y0, x0, nullptr, xd, yd, integral, s_cnt);
  __syncthreads();
  if (threadIdx.x < c.O) {                       // patch histogram (ref: mim.py:58-66)
    unsigned h = 0;
    for (int q = 0; q < c.cells; ++q) h += s_cnt[q * c.O + threadIdx.x];
    s_hist[threadIdx.x] = h;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int np = 0, skip = 0;
    if (mode == 0) s_pick[np++] = 1;
    else if (mode == 1) { for (int v = 1; v <= c.O; ++v) s_pick[np++] = v; }
    else {
      // ref: mim.py:69-91 (first argmax; runner-up >= ratio * peak, cyclic tie rule)
      int pk = 0;
      for (int v = 1; v < c.O; ++v) if (s_hist[v] > s_hist[pk]) pk = v;
      double rv = -1.0;
      for (int v = 0; v < c.O; ++v) if (v != pk && (double)s_hist[v] > rv) rv = (double)s_hist[v];
      int picks[2] = {pk + 1, 0}, cand = 1;
      if (rv >= c.ratio * (double)s_hist[pk]) {
        int best = -1, bestd = 1 << 30;
        for (int v = 0; v < c.O; ++v) {
          if (v == pk || (double)s_hist[v] != rv) continue;
          const int d = v > pk ? v - pk : v - pk + c.O;
          if (d < bestd) { bestd = d; best = v; }
        }
        picks[1] = best + 1;
        cand = 2;
      }
      for (int q = 0; q < cand; ++q) {
        const int dom = picks[q];
        if (c.rotate && dom != 1 && !rotated_inside(c, dom - 1, xd, yd, integral)) { ++skip; continue; }
        s_pick[np++] = dom;
      }
    }
    s_np = np;
    chain_publish(&lb[k], kChainAgg, (unsigned)np);
    if (skip) atomicAdd(&a.skipped[b], skip);
    if (np) atomicAdd(&a.count[b], np);
  }
  __syncthreads();
  const int np = s_np;
  const bool rot_mode = mode == 2 && c.rotate;
  int nrot = 0;
  for (int q = 0; q < np && q < 2; ++q) {
    const int dom = s_pick[q];
    if (rot_mode && dom != 1) {
      count_patch_g(m, c, a, y0, x0, uv + (size_t)(dom - 1) * c.P * c.P, xd, yd, integral, s_cnt + (1 + nrot) * nb);
      ++nrot;
    }
  }
  // output offset: decoupled look-back over the earlier keypoints' counts (as k_desc_main)
  if (threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    unsigned excl = 0;
    for (int base = k - 1; base >= 0; base -= 32) {
      const int j = base - (int)lane;
      unsigned long long f = 2ull << 62;
      if (j >= 0) do { f = chain_read(&lb[j]); } while ((f >> 62) == 0);
      const unsigned pre = __ballot_sync(0xffffffffu, (f >> 62) == kChainPrefix);
      const int stop = pre ? __ffs(pre) - 1 : 32;
      unsigned v = (int)lane <= stop ? (unsigned)f : 0u;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      excl += v;
      if (pre) break;
    }
    if (lane == 0) {
      chain_publish(&lb[k], kChainPrefix, excl + (unsigned)np);
      s_excl = excl;
    }
  }
  __syncthreads();
  const unsigned excl = s_excl;
  int r = 0;
  for (int q = 0; q < np; ++q) {
    const int dom = s_pick[q];
    const bool rotated = rot_mode && dom != 1;
    const unsigned* src = rotated ? s_cnt + (1 + r) * nb : s_cnt;
    const int var = mode == 0 ? 1 : dom;
    const unsigned dst = excl + q;
    if (dst < (unsigned)a.cap) {
      const size_t o = (size_t)b * a.cap + dst;
      __half* row = a.counts + o * a.stride;
      // recode (ref: mim.py:117-136): output bin (cell, w) <- value (w + var - 1) mod O
      for (int i = threadIdx.x; i < a.stride; i += kTG) {
        unsigned v = 0;
        if (i < c.dim) {
          const int cell = i / c.O, w = i % c.O;
          const int u = w + var - 1;
          v = src[cell * c.O + (u >= c.O ? u - c.O : u)];
        }
        row[i] = __uint2half_rn(v);
      }
      if (threadIdx.x == 0) {
        int sq = 0;
        for (int i = 0; i < nb; ++i) sq += (int)(src[i] * src[i]);
        a.sqnorm[o] = sq;
        a.kp[o] = k;
        a.variant[o] = (uint8_t)var;
      }
    }
    if (rotated) ++r;
  }
}

// Dense 16 x 16 cell sums: out[y][x] = per-value counts of the window
// [y, y+16) x [x, x+16) of the index map, as two words of 10-bit fields
// (values 1, 3, 5 in .x, values 2, 4, 6 in .y: the e / o words of
// reduce_cell).  The axis-aligned patch of a keypoint is 36 such windows, so
// k_desc_main reads 36 words instead of counting 9,216 pixels (the
// keypoints' patches overlap ~44-fold at 5,000 keypoints per 1024^2 image).
// Separable running sums per 64 x 64 tile over the shift-byte copy: two
// threads per staged row slide a 16-wide window along x (5-bit fields), then
// two threads per column slide 16 rows down (widened to the 10-bit fields).
// Windows that leave the image are never read (ref: descriptor.py:196-198
// skips those keypoints).
constexpr int kCsT = 64, kCsH = 64, kCsIn = kCsT + 15, kCsInH = kCsH + 15;
// six 5-bit fields (<= 16 per field) -> the e / o words of 10-bit fields
R2_DEV void widen5(uint32_t x, uint32_t& e, uint32_t& o) {
  e = x & 0x01f07c1fu;
  o = (x >> 5) & 0x01f07c1fu;
}
// shb: the shift-byte copy of the index map (k_mim_shift): a pixel counts as 1 << byte
__global__ void __launch_bounds__(128) k_cell_sums(const uint8_t* __restrict__ shb, uint2* __restrict__ out, int H, int W) {
  __shared__ uint8_t in[kCsInH][84];          // 21-word pitch: a column of rows hits distinct banks
  __shared__ uint32_t hs[kCsInH][kCsT + 1];   // horizontal 16-sums, 5-bit fields (odd pitch: conflict-free columns)
  const int b = blockIdx.z, ty0 = blockIdx.y * kCsH, tx0 = blockIdx.x * kCsT;
  const uint8_t* m = shb + (size_t)b * H * W;
  for (int i = threadIdx.x; i < kCsInH * 20; i += 128) {      // 79 rows x 80 bytes as words
    const int r = i / 20, q = i % 20;
    const int y = ty0 + r, x = tx0 + 4 * q;
    uint32_t v = 0;                           // beyond the map: only windows no descriptor reads
    if (y < H) {
      if (x + 3 < W && (W & 3) == 0) v = __ldg(reinterpret_cast<const uint32_t*>(m + (size_t)y * W + x));
      else for (int e = 0; e < 4; ++e) if (x + e < W) v |= (uint32_t)m[(size_t)y * W + x + e] << (8 * e);
    }
    *reinterpret_cast<uint32_t*>(&in[r][4 * q]) = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * kCsInH; i += 128) {       // (staged row, half of its 64 windows)
    const int r = i >> 1, x0 = (i & 1) * 32;
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 15; ++j) acc += one_hot(in[r][x0 + j]);
#pragma unroll 8
    for (int x = x0; x < x0 + 32; ++x) {
      acc += one_hot(in[r][x + 15]);
      hs[r][x] = acc;
      acc -= one_hot(in[r][x]);
    }
  }
  __syncthreads();
  {
    const int x = threadIdx.x & 63, r0 = (threadIdx.x >> 6) * 32;   // two threads per column: 32 output rows each
    uint32_t e = 0, o = 0, we, wo;
#pragma unroll
    for (int j = 0; j < 15; ++j) { widen5(hs[r0 + j][x], we, wo); e += we; o += wo; }
#pragma unroll 8
    for (int r = r0; r < r0 + 32; ++r) {
      widen5(hs[r + 15][x], we, wo);
      e += we; o += wo;
      if (ty0 + r < H && tx0 + x < W) out[((size_t)b * H + ty0 + r) * W + tx0 + x] = make_uint2(e, o);
      widen5(hs[r][x], we, wo);
      e -= we; o -= wo;
    }
  }
}

// The index map as shift bytes 5(v-1) in one pass over the planes, so the
// per-keypoint kernel stages them by TMA with no in-place transform of its
// ~21 KB neighbourhood (that pass was a fifth of its shared-memory traffic).
// Zero-filled bytes beyond the map then count as index 1, but no emitted
// descriptor ever samples them (the skip tests bound every sample).
__global__ void __launch_bounds__(256) k_mim_shift(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 w = __ldg(&in[i]);
    w.x = w.x * 5u - 0x05050505u;
    w.y = w.y * 5u - 0x05050505u;
    w.z = w.z * 5u - 0x05050505u;
    w.w = w.w * 5u - 0x05050505u;
    out[i] = w;
  }
}

struct DescWs {
  size_t off_chain, off_ticket, total;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

int per_kp(int mode, int O) { return (mode == 1 || mode == 3) ? O : (mode == 2 ? 2 : 1); }

DescWs plan_ws(int B, int S) {
  DescWs p{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = al(off + bytes); return o; };
  p.off_chain = take((size_t)B * S * sizeof(unsigned long long));   // look-back words per keypoint
  p.off_ticket = take((size_t)B * sizeof(unsigned));                  // start-order tickets per image
  p.total = off;
  return p;
}

constexpr int kMaxStride = 256;

}  // namespace

size_t describe_workspace_bytes(int B, int kp_stride, int grid, int O) {
  (void)grid;
  (void)O;
  return plan_ws(B, kp_stride > 0 ? kp_stride : 1).total;
}

size_t describe_workspace_bytes_hw(int B, int H, int W, int kp_stride, int grid, int O) {
  // + the shift-byte copy of the index maps and the dense 16 x 16 cell sums
  // (each used when the workspace holds it)
  return describe_workspace_bytes(B, kp_stride, grid, O) + al((size_t)B * H * W) + al((size_t)B * H * W * sizeof(uint2));
}

int describe_run(const uint8_t* mim, const DescribeArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int S = a.kp_stride > 0 ? a.kp_stride : 1;
  const DescWs p = plan_ws(a.B, S);
  if (ws_bytes < p.total) return 1;
  if (a.stride % 8 != 0) return 2;
  const int cs = a.patch / a.grid;
  if (a.O > kMaxOrientG || a.patch % a.grid != 0) return 2;
  GatherTables tab = gather_tables(a.patch, a.O);
  if (!tab.uv) return 3;
  // k_desc_main: 5-bit one-hot fields (O <= 6, cs <= 31 rows per thread), 4
  // columns per thread, integer keypoints; everything else: k_desc_generic
  const bool fast = !a.kp_xd && a.O <= 6 && cs == 16 && a.grid * a.grid * (cs / 4) <= kT && tab.soff &&
                    a.stride <= kMaxStride;
  if (!fast) {
    DescConstG g{};
    g.H = a.H; g.W = a.W; g.O = a.O; g.P = a.patch; g.g = a.grid; g.cs = cs;
    g.cells = a.grid * a.grid; g.dim = g.cells * a.O;
    g.ratio = a.ratio; g.rotate = a.rotate; g.mode = a.mode;
    for (int q = 0; q < a.O; ++q) g.bbf[q] = tab.hbbf[q];
    char* w = static_cast<char*>(ws);
    auto* chain = reinterpret_cast<unsigned long long*>(w + p.off_chain);
    auto* ticket = reinterpret_cast<unsigned*>(w + p.off_ticket);
    cudaMemsetAsync(a.count, 0, sizeof(int32_t) * a.B, st);
    cudaMemsetAsync(a.skipped, 0, sizeof(int32_t) * a.B, st);
    if (a.kp_stride == 0) return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
    cudaMemsetAsync(w, 0, p.total, st);
    const size_t smem = 3 * (size_t)g.cells * g.O * sizeof(uint32_t);
    auto kern = a.kp_xd ? k_desc_generic<true> : k_desc_generic<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<dim3(a.kp_stride, a.B), kTG, smem, st>>>(mim, a, g, tab.uv, chain, ticket);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
  }
  DescConst c{};
  c.H = a.H; c.W = a.W; c.O = a.O; c.P = a.patch; c.g = a.grid; c.cs = cs;
  c.cells = a.grid * a.grid; c.dim = c.cells * a.O; c.per = per_kp(a.mode, a.O);
  c.ratio = a.ratio; c.rotate = a.rotate; c.mode = a.mode;
  c.R = tab.radius;
  for (int q = 0; q < 8; ++q) c.bbox[q] = tab.hbbox[q];
  c.stride = tab.stride;
  c.rows = 2 * c.R + 1;
  char* w = static_cast<char*>(ws);
  auto* chain = reinterpret_cast<unsigned long long*>(w + p.off_chain);
  auto* ticket = reinterpret_cast<unsigned*>(w + p.off_ticket);
  cudaMemsetAsync(a.count, 0, sizeof(int32_t) * a.B, st);
  cudaMemsetAsync(a.skipped, 0, sizeof(int32_t) * a.B, st);
  if (a.kp_stride == 0) return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
  cudaMemsetAsync(w, 0, p.total, st);                 // look-back words and tickets
  const size_t smem = (size_t)c.rows * c.stride + 3 * (size_t)c.cells * c.O * sizeof(uint32_t) + 128;
  if (smem > 200 * 1024) return 2;
  dim3 grid(a.kp_stride, a.B);
  CUtensorMap tmap{};
  c.tma = 0;
  c.preshift = 0;
  auto enc = get_encode();
  if (enc && c.W % 16 == 0 && c.stride <= 256 && c.rows <= 256 && ((uintptr_t)mim & 15) == 0) {
    // the shift-byte copy when the workspace has room for it (the
    // height/width-aware size query), else the in-place transform
    const uint8_t* src = mim;
    const size_t n = (size_t)a.B * a.H * a.W;
    if (ws_bytes >= p.total + al(n)) {
      uint8_t* sh = static_cast<uint8_t*>(ws) + p.total;
      const size_t n16 = n / 16;
      k_mim_shift<<<(unsigned)std::min<size_t>((n16 + 255) / 256, 148 * 16), 256, 0, st>>>(
          reinterpret_cast<const uint4*>(mim), reinterpret_cast<uint4*>(sh), n16);
      src = sh;
      c.preshift = 1;
      // and the dense cell sums behind it (values 1..6 in 10-bit fields)
      if (kDescDense && a.O <= 6 && ws_bytes >= p.total + al(n) + al(n * sizeof(uint2)) && a.H >= 16 && a.W >= 16) {
        uint2* cs_out = reinterpret_cast<uint2*>(static_cast<uint8_t*>(ws) + p.total + al(n));
        k_cell_sums<<<dim3((a.W + kCsT - 1) / kCsT, (a.H + kCsH - 1) / kCsH, a.B), 128, 0, st>>>(sh, cs_out, a.H, a.W);
        c.dense = cs_out;
      }
    }
    // 2-D view (W, B*H): rows outside one image read its neighbour (or zeros
    // at the ends) -- never sampled by an emitted descriptor, see above
    cuuint64_t dims[2] = {(cuuint64_t)c.W, (cuuint64_t)c.H * a.B};
    cuuint64_t strides[1] = {(cuuint64_t)c.W};
    cuuint32_t box[2] = {(cuuint32_t)c.stride, (cuuint32_t)c.rows};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(src), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      c.tma = 1;
  }
  // the BASELINE grid (6 orientations, 6 x 6 cells) with constant indexing
  auto kern = (c.O == 6 && c.g == 6) ? k_desc_main<16, 6, 6> : k_desc_main<16, 0, 0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // shared-memory carveout (percent): what is not carved out stays L1 for the offset tables
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, R2_DESC_CARVE);
  kern<<<grid, kT, smem, st>>>(tmap, mim, a, c, tab, chain, ticket);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2
