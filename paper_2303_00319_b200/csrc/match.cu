// Brute-force nearest-neighbour matching on the 5th-gen tensor cores.
//
// Replaces ref: pkg/src/rift2/matcher.py:67-148 (_group, _min_over_row_groups,
// match_nn).  The reference ranks reference descriptors r for a target
// descriptor t by |r|^2 - 2 r.t on unit float64 vectors, i.e. by the cosine
// c_r.c_t / (|c_r| |c_t|) of the integer count vectors.  Here:
//
//   k_match_gemm  D = C_tgt . C_ref^T on fp16 counts (exact: counts <= 256,
//                 dots < 2^24) with tcgen05.mma (M=128 tgt rows, N=128 ref
//                 columns, K=224 in 14 steps) into NACC=4 TMEM accumulators;
//                 A (the CTA's target rows) resident in smem, B double
//                 buffered, both staged by TMA (128B swizzle).  Warp 0
//                 produces, warp 1 issues MMA, 16 epilogue warps (4 TMEM lane
//                 quarters x 4 32-column blocks) tcgen05.ld their chunk and
//                 keep an exact running argmax per target row: an fp32
//                 screen (FMUL2 + FMNMX3), a pending-chunk copy on a new
//                 maximum, and integer D^2 q comparisons only for near ties
//                 (1e-5 window) and once at the end; ties go to the smallest
//                 reference column (= keypoint id order).
//   k_match_index per pair: target variant groups, reference keypoint ranges
//   k_match_combine per target keypoint: best over its variants and over the
//                 column splits (exact 128-bit comparison), then the exact
//                 float64 distance of the winner (ref: matcher.py:137-141)
//   k_msort_*     per pair: order by (dist, ref, tgt) (ref: matcher.py:143-146),
//                 bucket sort on the distance bits, multi-CTA
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "match.h"
#include "sort.cuh"
#include "tma.cuh"

namespace r2 {

namespace {

constexpr int BM = 128;            // target rows per CTA (UMMA M)
constexpr int BN = 256;            // reference columns per tile (UMMA N)
constexpr int BK = 64;             // fp16 elements per 128-byte swizzle atom
constexpr int KBOX = 4;            // K boxes of 64 -> 256 >= 224
constexpr int A_BOX = BM * BK * 2;             // 16 KB per K box
constexpr int B_BOX = BN * BK * 2;             // 32 KB per K box (one ring stage)
constexpr int A_BYTES = KBOX * A_BOX;          // 64 KB, resident
constexpr int NSTAGE = 4;                      // B ring: K boxes in flight
constexpr int NACC = 2;                        // TMEM accumulator buffers
constexpr int TMEM_COLS = NACC * BN;           // 512: all of TMEM
// 8 epilogue warps (4 lane quarters x 2 column groups): 320 threads leave
// room for two chunks in flight per warp (~130 registers)
constexpr int NEPI = 8;
constexpr int CPW = BN / 32 / (NEPI / 4);      // 32-column chunks per epilogue warp per tile
constexpr int GEMM_THREADS = 64 + NEPI * 32;  // producer, MMA, epilogue warps
constexpr int BAR_OFF = A_BYTES + NSTAGE * B_BOX;
constexpr int SMEM_GEMM = BAR_OFF + 256 + NEPI * 64 * 4 + 4 * (NEPI / 4 - 1) * BM * 4 + 1024;
static_assert(SMEM_GEMM <= 227 * 1024, "GEMM shared memory");

#ifdef R2_GEMM_TRACE
// development trace: clock64 stamps of the pipeline roles of CTA (0, 0), and
// per CTA (SM id, globaltimer start / end, tiles)
__device__ unsigned long long g_trace[8][512];
__device__ unsigned long long g_cta[8192][4];
#define R2_TR(ev, i) do { if (blockIdx.x == 0 && blockIdx.y == 0 && (i) < 512) g_trace[ev][i] = clock64(); } while (0)
R2_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define R2_CTA(slot, val) do { const unsigned b_ = blockIdx.y * gridDim.x + blockIdx.x; \
  if (threadIdx.x == 0 && b_ < 8192) g_cta[b_][slot] = (val); } while (0)
#else
#define R2_TR(ev, i) do {} while (0)
#define R2_CTA(slot, val) do {} while (0)
#endif

struct Part {
  int D;      // integer dot product
  int q;      // reference squared norm
  int kp;     // reference keypoint id (-1: none)
  float s;    // screening score D / |c_r|
};

// ------------------------------------------------------------ PTX helpers
R2_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
R2_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte swizzled operand descriptor (8-row core groups 1024 B apart)
R2_DEV uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;                 // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: f16 x f16 -> f32, both K-major, M=128, N=BN
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

R2_DEV void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      :: "r"(tmem_d), "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate) : "memory");
}
R2_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

// TMEM load issue / completion, split so a chunk's load overlaps the
// previous chunk's processing: the wait names the destination registers as
// read-write, so nothing reads them before it
R2_DEV void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
R2_DEV void tmem_ld_wait(uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
        "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
        "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
        "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :: "memory");
}

R2_DEV void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// exact "a beats b" for candidates of the same target row: D_a/|c_a| > D_b/|c_b|
R2_DEV int cmp_exact(float Da, int qa, float Db, int qb) {
  const unsigned long long da = (unsigned long long)Da, db = (unsigned long long)Db;
  const unsigned long long l = da * da * (unsigned long long)qb;
  const unsigned long long r = db * db * (unsigned long long)qa;
  return l > r ? 1 : (l < r ? -1 : 0);
}

struct GemmParams {
  const int32_t* sqnorm;
  const int32_t* kp;
  const int32_t* count;
  const int32_t* ref_block;
  const int32_t* tgt_block;
  int cap, splits;
  Part* part;   // [n_pairs][cap][splits]
};

// screening factor 1/|c_r| (0 for an empty descriptor); same formula everywhere
R2_DEV float inv_norm(int q) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)q));
  return q > 0 ? r : 0.f;
}

// exact running-best update with one candidate column (ties keep the earlier column)
R2_DEV void take_exact(float D, int qq, float sj, int col, float& best, float& bestD, int& bestq, int& bestcol) {
  if (bestcol < 0 || sj > best * (1.f + 1e-5f)) {
    best = sj; bestD = D; bestcol = col; bestq = qq;
  } else if (sj >= best * (1.f - 1e-5f)) {
    if (cmp_exact(D, qq, bestD, bestq) > 0) { best = sj; bestD = D; bestcol = col; bestq = qq; }
  }
}

// fold a pending chunk (raw dot products rv of columns c0..c0+31, screening
// maximum rcm) into the exact best, columns in increasing order
R2_DEV void resolve_chunk(const float (&rv)[32], int c0, float rcm, int n_r, const int* __restrict__ sq,
                          float& best, float& bestD, int& bestq, int& bestcol) {
  const float lo = fmaxf(rcm, best) * (1.f - 1e-5f);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int col = c0 + j;
    if (col < n_r) {
      const int qq = __ldg(&sq[col]);
      const float sj = rv[j] * inv_norm(qq);
      if (sj >= lo) take_exact(rv[j], qq, sj, col, best, bestD, bestq, bestcol);
    }
  }
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
k_match_gemm(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB, GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for SWIZZLE_128B, as an offset so the pointer keeps its shared address space
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* full = bars;                 // [NSTAGE]
  uint64_t* empty = bars + NSTAGE;       // [NSTAGE]
  uint64_t* a_full = bars + 2 * NSTAGE;
  uint64_t* t_full = a_full + 1;         // [NACC]
  uint64_t* t_empty = t_full + NACC;     // [NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + NACC);
  float* s_inv = reinterpret_cast<float*>(smem + BAR_OFF + 256);   // [NEPI warps][2][32], 16-B aligned
  float* s_mrg_f = s_inv + NEPI * 64;                              // [2][NB-1][BM] best / D of blocks 1..
  int* s_mrg_i = reinterpret_cast<int*>(s_mrg_f + 2 * (NEPI / 4 - 1) * BM);   // [2][NB-1][BM] q / column

#ifdef R2_GEMM_TRACE
  {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    R2_CTA(0, smid);
    R2_CTA(1, gtimer());
    R2_CTA(3, 0ull);
  }
#endif
  const int pair = blockIdx.y;
  const int split = blockIdx.x % p.splits;
  const int mt = blockIdx.x / p.splits;
  const int rb = p.ref_block[pair], tb = p.tgt_block[pair];
  // counts past the buffer capacity are clamped (the rows do not exist)
  const int n_t = min(p.count[tb], p.cap), n_r = min(p.count[rb], p.cap);
  if (mt * BM >= n_t) return;
  const int n_tiles_all = (n_r + BN - 1) / BN;
  const int per = (n_tiles_all + p.splits - 1) / p.splits;
  const int nt0 = split * per;
  const int nt1 = min(n_tiles_all, nt0 + per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Part* out = p.part + ((size_t)pair * p.cap) * p.splits;
  if (nt0 >= nt1) {
    // empty split: publish "no candidate" for this tile's rows
    for (int r = threadIdx.x; r < BM; r += blockDim.x) {
      const int row = mt * BM + r;
      if (row < n_t) out[(size_t)row * p.splits + split] = Part{0, 1, -1, -1.f};
    }
    return;
  }
  const int ntiles = nt1 - nt0;
  R2_CTA(3, (unsigned long long)ntiles);
  const int rowA = tb * p.cap + mt * BM;
  const int rowB0 = rb * p.cap;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(a_full, 1);
    for (int s = 0; s < NACC; ++s) { mbar_init(&t_full[s], 1); mbar_init(&t_empty[s], NEPI); }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tmapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&tmapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_slot)), "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      mbar_expect_tx(a_full, A_BYTES);
      for (int kb = 0; kb < KBOX; ++kb) tma_load_2d(sA + kb * A_BOX, &tmapA, kb * BK, rowA, a_full);
      for (int i = 0; i < ntiles; ++i) {
        const int rowB = rowB0 + (nt0 + i) * BN;
        R2_TR(0, i);
        for (int kb = 0; kb < KBOX; ++kb) {
          const int u = i * KBOX + kb, s = u % NSTAGE;
          mbar_wait(&empty[s], ((u / NSTAGE) & 1) ^ 1);
          if (kb == 0) R2_TR(1, i);
          mbar_expect_tx(&full[s], B_BOX);
          tma_load_2d(sB + s * B_BOX, &tmapB, kb * BK, rowB, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer (single thread)
      mbar_wait(a_full, 0);
      const uint32_t a_base = smem_u32(sA);
      for (int i = 0; i < ntiles; ++i) {
        const int acc = i % NACC;
        R2_TR(2, i);
        mbar_wait(&t_empty[acc], ((i / NACC) & 1) ^ 1);
        R2_TR(4, i);
        const uint32_t d = tmem + acc * BN;
        // 14 K-steps of 16 over the 4 boxes (the last box holds K 192..223 + zero fill)
#pragma unroll
        for (int kb = 0; kb < KBOX; ++kb) {
          const int u = i * KBOX + kb, s = u % NSTAGE;
          mbar_wait(&full[s], (u / NSTAGE) & 1);
          if (kb == 0) R2_TR(3, i);
          tc_fence_after();
          const uint32_t b_base = smem_u32(sB + s * B_BOX);
#ifndef R2_EXP_NOMMA   // timing experiment (DESIGN 4): operand loads only
#pragma unroll
          for (int kk = 0; kk < (kb == KBOX - 1 ? 2 : 4); ++kk)
            mma_f16(d, smem_desc(a_base + kb * A_BOX + kk * 32), smem_desc(b_base + kk * 32),
                    (kb | kk) ? 1u : 0u);
#endif
          mma_commit(&empty[s]);
        }
        mma_commit(&t_full[acc]);
        R2_TR(5, i);
      }
    }
  } else {
    // ---- epilogue warps 2..17: TMEM lane quarter = warp % 4, 32-column block = (warp-2) / 4
    //
    // Per row (lane) the warp keeps an exactly-resolved best E = (bestD, bestq,
    // bestcol, best) and at most one *pending* chunk R: the 32 raw dot products
    // rv[] of the chunk whose screening maximum r_cm is the largest seen so far.
    // Screening scores s = D * rsqrt(q) carry < 2e-7 relative error, so with a
    // 1e-5 window a chunk is either (a) strictly below every candidate (skip),
    // (b) strictly above all of them (it replaces R and E: a copy, no exact
    // work), or (c) a near tie: only then is R resolved exactly into E before
    // the new chunk becomes R.  R is resolved once more after the last tile.
    // Record events are rare per row (~ln n) but frequent per warp, so (b)
    // is kept branch-light; exact work happens only for (c) and at the end.
    constexpr int NB = NEPI / 4;                    // column groups (warps per lane quarter)
    const int e = warp - 2;
    const int q = warp & 3, h = e >> 2;
    const int row_loc = q * 32 + lane;
    const int row = mt * BM + row_loc;
    const bool row_ok = row < n_t;
    float* inv_buf = s_inv + e * 64;                // two 32-float buffers (current / next chunk)
    const int* sq = p.sqnorm + (size_t)rb * p.cap;
    float best = -1.f, bestD = 0.f;
    int bestq = 1, bestcol = -1;
    float rv[32];
    float r_cm = -1.f;
    int r_c0 = -1;
#pragma unroll
    for (int j = 0; j < 32; ++j) rv[j] = 0.f;
    // chunk j = CPW * tile + k covers columns tile * BN + (h + NB * k) * 32 .. + 31:
    // increasing along j, so ties keep the first column
    auto chunk_c0 = [&](int j) { return (nt0 + j / CPW) * BN + (h + NB * (j % CPW)) * 32; };
    const int nch = ntiles * CPW;
    int q_nxt;
    {
      const int c = chunk_c0(0) + lane;
      q_nxt = c < n_r ? __ldg(&sq[c]) : 0;          // first chunk's squared norms
    }
    // Two chunks in flight: chunk j + 1's TMEM load is issued before chunk j
    // is processed and waited for after it; a tile's accumulator goes back to
    // the MMA warp as soon as its last chunk is in registers.
    auto issue = [&](uint32_t (&dst)[32], int j) {
      const int i = j / CPW, k = j % CPW, acc = i % NACC;
      if (k == 0) {
        mbar_wait(&t_full[acc], (i / NACC) & 1);
        tc_fence_after();
      }
      tmem_ld32_issue(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + (h + NB * k) * 32, dst);
    };
    auto landed = [&](uint32_t (&dst)[32], int j) {
      tmem_ld_wait(dst);
      if (j % CPW == CPW - 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[(j / CPW) % NACC]);
      }
    };
    // the screening and candidate bookkeeping of chunk j (raw dots in r)
    auto process = [&](const uint32_t (&r)[32], int j) {
#ifdef R2_EXP_NOEPI   // timing experiment (DESIGN 4): accumulators drained, not screened
      return;
#endif
      const int c0 = chunk_c0(j);
      float* ic = inv_buf + (j & 1) * 32;
      ic[lane] = inv_norm(q_nxt);
      {
        const int c = chunk_c0(j + 1) + lane;
        q_nxt = (j + 1 < nch && c < n_r) ? __ldg(&sq[c]) : 0;   // next chunk, in flight
      }
      __syncwarp();
      if (c0 >= n_r) return;                          // warp-uniform: past the reference rows
      // screening maximum; invalid tail columns carry inv = 0 (score 0)
      float cm = 0.f;
      const float4* iv = reinterpret_cast<const float4*>(ic);
#pragma unroll
      for (int q4 = 0; q4 < 8; ++q4) {
        const float4 f = iv[q4];
        const float2 a = __fmul2_rn(make_float2(__uint_as_float(r[4 * q4 + 0]), __uint_as_float(r[4 * q4 + 1])),
                                    make_float2(f.x, f.y));
        const float2 b = __fmul2_rn(make_float2(__uint_as_float(r[4 * q4 + 2]), __uint_as_float(r[4 * q4 + 3])),
                                    make_float2(f.z, f.w));
        cm = fmaxf(fmaxf(cm, a.x), a.y);
        cm = fmaxf(fmaxf(cm, b.x), b.y);
      }
      // rows past the target count (the last M-tile's padding) never take the
      // exact path: their zero / stale rows would tie on every chunk
      const float T = fmaxf(r_cm, best);
      const bool rec = row_ok && cm > T * (1.f + 1e-5f);     // for T < 0 (nothing yet) always true
      const bool near = row_ok && !rec && cm >= T * (1.f - 1e-5f);
      if (__any_sync(0xffffffffu, rec || near)) {
        if (near && r_c0 >= 0)
          resolve_chunk(rv, r_c0, r_cm, n_r, sq, best, bestD, bestq, bestcol);
        if (rec) { best = -1.f; bestD = 0.f; bestq = 1; bestcol = -1; }
        const bool take = rec || near;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) rv[jj] = take ? __uint_as_float(r[jj]) : rv[jj];
        r_cm = take ? cm : r_cm;
        r_c0 = take ? c0 : r_c0;
      }
    };
    uint32_t va[32], vb[32];
    if (nch > 0) {
      issue(va, 0);
      landed(va, 0);
    }
    for (int j = 0; j < nch; j += 2) {
      if (j + 1 < nch) issue(vb, j + 1);
      process(va, j);
      if (j + 1 >= nch) break;
      landed(vb, j + 1);
      if (j + 2 < nch) issue(va, j + 2);
      process(vb, j + 1);
      if (j + 2 < nch) landed(va, j + 2);
    }
    // the pending chunk, resolved once at the end
    if (row_ok && r_c0 >= 0) resolve_chunk(rv, r_c0, r_cm, n_r, sq, best, bestD, bestq, bestcol);
    // merge the NB column blocks of each row (exact; ties -> smaller column = smaller kp id)
    if (h > 0) {
      const int sidx = (h - 1) * BM + row_loc;
      s_mrg_f[sidx] = best;
      s_mrg_f[(NB - 1) * BM + sidx] = bestD;
      s_mrg_i[sidx] = bestq;
      s_mrg_i[(NB - 1) * BM + sidx] = bestcol;
    }
    named_sync(1, NEPI * 32);
    if (h == 0) {
      for (int o = 0; o < NB - 1; ++o) {
        const int sidx = o * BM + row_loc;
        const float ob = s_mrg_f[sidx], oD = s_mrg_f[(NB - 1) * BM + sidx];
        const int oq = s_mrg_i[sidx], oc = s_mrg_i[(NB - 1) * BM + sidx];
        if (oc < 0) continue;
        bool take;
        if (bestcol < 0) take = true;
        else {
          const int r = cmp_exact(oD, oq, bestD, bestq);
          take = r > 0 || (r == 0 && oc < bestcol);
        }
        if (take) { best = ob; bestD = oD; bestq = oq; bestcol = oc; }
      }
      if (row < n_t) {
        Part r;
        r.D = (int)bestD;
        r.q = bestq;
        r.kp = bestcol >= 0 ? __ldg(&p.kp[(size_t)rb * p.cap + bestcol]) : -1;
        r.s = best;
        out[(size_t)row * p.splits + split] = r;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(TMEM_COLS));
  }
#ifdef R2_GEMM_TRACE
  R2_CTA(2, gtimer());
#endif
}

// ------------------------------------------------------------ index / combine
struct IdxWs {
  int* gstart;   // [n_pairs][cap] target group start
  int* ng;       // [n_pairs]
  int* rstart;   // [n_pairs][cap] by reference kp id
  int* rend;     // [n_pairs][cap]
};

__global__ void __launch_bounds__(1024) k_match_index(MatchArgs a, IdxWs w) {
  __shared__ int s_warp[32];
  __shared__ int s_base, s_tot;
  const int pair = blockIdx.x;
  const int tb = a.tgt_block[pair], rb = a.ref_block[pair];
  const int n_t = min(a.count[tb], a.cap), n_r = min(a.count[rb], a.cap);
  const int* tk = a.kp + (size_t)tb * a.cap;
  const int* rk = a.kp + (size_t)rb * a.cap;
  int* gs = w.gstart + (size_t)pair * (a.cap + 1);
  int* rs = w.rstart + (size_t)pair * a.cap;
  int* re = w.rend + (size_t)pair * a.cap;
  for (int i = threadIdx.x; i < n_r; i += blockDim.x) {
    if ((unsigned)rk[i] >= (unsigned)a.cap) continue;   // ids outside [0, cap) break the ABI precondition
    if (i == 0 || rk[i] != rk[i - 1]) rs[rk[i]] = i;
    if (i == n_r - 1 || rk[i + 1] != rk[i]) re[rk[i]] = i + 1;
  }
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < n_t; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool st = i < n_t && (i == 0 || tk[i] != tk[i - 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, st);
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { const int t = s_warp[q]; s_warp[q] = run; run += t; }
      s_tot = run;
    }
    __syncthreads();
    if (st) gs[s_base + s_warp[wid] + __popc(bal & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) s_base += s_tot;
    __syncthreads();
  }
  // an empty reference set matches nothing (the dataclass API raises instead,
  // ref: matcher.py:105-106; a batch slot simply reports 0 matches)
  if (threadIdx.x == 0) { w.ng[pair] = n_r > 0 ? s_base : 0; gs[s_base] = n_t; }
}

// a beats b across target variants: Da^2 q_rb q_tb > Db^2 q_ra q_ta (128-bit)
R2_DEV int cmp_cross(const Part& a, int qta, const Part& b, int qtb) {
  const unsigned __int128 l = (unsigned __int128)((unsigned long long)a.D * (unsigned long long)a.D) *
                              ((unsigned long long)b.q * (unsigned long long)qtb);
  const unsigned __int128 r = (unsigned __int128)((unsigned long long)b.D * (unsigned long long)b.D) *
                              ((unsigned long long)a.q * (unsigned long long)qta);
  return l > r ? 1 : (l < r ? -1 : 0);
}

// Part of (pair, target row t, split s) at pair * pair_stride + t * row_stride + s * split_stride:
// the GEMM's own [pair][row][split] layout, or [part][pair][row] as gathered from G ranks
struct PartLayout {
  size_t pair_stride, row_stride, split_stride;
};

__global__ void __launch_bounds__(256) k_match_combine(MatchArgs a, IdxWs w, const Part* __restrict__ part,
                                                       int splits, PartLayout lay, K128* __restrict__ keys) {
  const int pair = blockIdx.y;
  const int warp_g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int ng = w.ng[pair];
  if (warp_g >= ng) return;
  const int tb = a.tgt_block[pair], rb = a.ref_block[pair];
  const int* gs = w.gstart + (size_t)pair * (a.cap + 1);
  const int t0 = gs[warp_g], t1 = gs[warp_g + 1];
  const Part* pp = part + (size_t)pair * lay.pair_stride;
  // best candidate over variants x splits (all lanes compute the same; cheap)
  Part best{0, 1, -1, -1.f};
  int best_qt = 1;
  for (int t = t0; t < t1; ++t) {
    const int qt = a.sqnorm[(size_t)tb * a.cap + t];
    for (int s = 0; s < splits; ++s) {
      const Part c = pp[(size_t)t * lay.row_stride + (size_t)s * lay.split_stride];
      if (c.kp < 0) continue;
      if (best.kp < 0) { best = c; best_qt = qt; continue; }
      const int r = cmp_cross(c, qt, best, best_qt);
      if (r > 0 || (r == 0 && c.kp < best.kp)) { best = c; best_qt = qt; }
    }
  }
  const int tkp = a.kp[(size_t)tb * a.cap + t0];
  double dmin = 0.0;
  if (best.kp >= 0) {
    // a winner outside this call's reference rows (row-sharded finish: the
    // rank owning it computes the distance) reports +inf
    const int r0 = w.rstart[(size_t)pair * a.cap + best.kp], r1 = w.rend[(size_t)pair * a.cap + best.kp];
    dmin = r1 > r0 ? 1e300 : INFINITY;
    for (int r = r0; r < r1; ++r) {
      const double ir = 1.0 / sqrt((double)a.sqnorm[(size_t)rb * a.cap + r]);
      const __half* cr = a.counts + ((size_t)rb * a.cap + r) * a.stride;
      for (int t = t0; t < t1; ++t) {
        const double it = 1.0 / sqrt((double)a.sqnorm[(size_t)tb * a.cap + t]);
        const __half* ct = a.counts + ((size_t)tb * a.cap + t) * a.stride;
        double acc = 0.0;
        for (int i = lane; i < a.dim; i += 32) {
          // reference vectors are c / ||c|| in float64 (ref: descriptor.py:161-164);
          // both products rounded on their own (no FMA contraction), so equal
          // descriptors are at distance exactly 0, as in the reference
          const double dv = __dsub_rn(__dmul_rn((double)__half2float(cr[i]), ir),
                                      __dmul_rn((double)__half2float(ct[i]), it));
          acc = fma(dv, dv, acc);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        dmin = fmin(dmin, acc);
      }
    }
    dmin = sqrt(dmin);
  }
  if (lane == 0) {
    K128 k;
    k.hi = (unsigned long long)__double_as_longlong(dmin);
    k.lo = ((unsigned long long)(unsigned)best.kp << 32) | (unsigned)tkp;
    keys[(size_t)pair * a.cap + warp_g] = k;
  }
}

// (dist, ref, tgt) order by bucket sort: a monotone linear bin of the
// float64 distance (in [0, 2]), a histogram, the
// bucket offsets, a scatter, and each key's rank among its own bucket's keys
// (keys are unique: tgt ids are).  All passes are multi-CTA per pair.
constexpr int kMsBins = 4096;
constexpr int kMsCtas = 16;

R2_DEV int ms_bin(const K128& k) {
  // distances of unit vectors lie in [0, 2]: linear bins, monotone in the key
  const double d = __longlong_as_double((long long)k.hi);
  if (!(d < 2.0)) return kMsBins - 1;             // includes the +inf of a non-local winner
  const int v = (int)(d * (kMsBins / 2));
  return v < 0 ? 0 : (v >= kMsBins ? kMsBins - 1 : v);
}

__global__ void __launch_bounds__(256) k_msort_hist(IdxWs w, const K128* __restrict__ keys, int cap,
                                                    unsigned* __restrict__ hist) {
  __shared__ unsigned h[kMsBins];
  const int pair = blockIdx.y;
  const int ng = w.ng[pair];
  for (int i = threadIdx.x; i < kMsBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const K128* k = keys + (size_t)pair * cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x) atomicAdd(&h[ms_bin(k[i])], 1u);
  __syncthreads();
  unsigned* g = hist + (size_t)pair * kMsBins;
  for (int i = threadIdx.x; i < kMsBins; i += blockDim.x)
    if (h[i]) atomicAdd(&g[i], h[i]);
}

__global__ void __launch_bounds__(1024) k_msort_scan(const unsigned* __restrict__ hist, unsigned* __restrict__ base) {
  __shared__ unsigned part[1024];
  const int pair = blockIdx.x;
  const unsigned* g = hist + (size_t)pair * kMsBins;
  unsigned* bb = base + (size_t)pair * kMsBins;
  constexpr int per = kMsBins / 1024;
  const int b0 = per * threadIdx.x;
  unsigned s = 0;
  for (int i = 0; i < per; ++i) s += g[b0 + i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const unsigned add = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += add;
    __syncthreads();
  }
  unsigned run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (int i = 0; i < per; ++i) { bb[b0 + i] = run; run += g[b0 + i]; }
}

__global__ void __launch_bounds__(256) k_msort_scatter(IdxWs w, const K128* __restrict__ keys, int cap,
                                                       const unsigned* __restrict__ base, unsigned* __restrict__ fill,
                                                       K128* __restrict__ out) {
  const int pair = blockIdx.y;
  const int ng = w.ng[pair];
  const K128* k = keys + (size_t)pair * cap;
  const unsigned* bb = base + (size_t)pair * kMsBins;
  unsigned* f = fill + (size_t)pair * kMsBins;
  K128* o = out + (size_t)pair * cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x) {
    const K128 key = k[i];
    const int bin = ms_bin(key);
    o[bb[bin] + atomicAdd(&f[bin], 1u)] = key;
  }
}

__global__ void __launch_bounds__(256) k_msort_rank(MatchArgs a, IdxWs w, const K128* __restrict__ bucketed,
                                                    const unsigned* __restrict__ hist,
                                                    const unsigned* __restrict__ base) {
  const int pair = blockIdx.y;
  const int ng = w.ng[pair];
  const K128* s = bucketed + (size_t)pair * a.cap;
  const unsigned* g = hist + (size_t)pair * kMsBins;
  const unsigned* bb = base + (size_t)pair * kMsBins;
  const int n = min(ng, a.tgt_kp_cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out_count[pair] = n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x) {
    const K128 mine = s[i];
    const int bin = ms_bin(mine);
    const unsigned lo = bb[bin], hi = lo + g[bin];
    unsigned pos = lo;
    for (unsigned j = lo; j < hi; ++j) pos += k_less(s[j], mine) ? 1u : 0u;
    if (pos < (unsigned)n) {
      const size_t o = (size_t)pair * a.tgt_kp_cap + pos;
      a.out_dist[o] = __longlong_as_double((long long)mine.hi);
      a.out_ref[o] = (int32_t)(mine.lo >> 32);
      a.out_tgt[o] = (int32_t)(mine.lo & 0xffffffffull);
    }
  }
}

// ------------------------------------------------ generic float64 vectors
// For descriptor sets that are not integer histograms (arbitrary unit
// vectors handed to match_nn): the reference's own key |r|^2 - 2 r.t in
// float64 (ref: matcher.py:125-135), min over both variant groups, first
// reference keypoint on ties.  One CTA per target keypoint group.
__global__ void __launch_bounds__(256) k_vec_best(const double* __restrict__ R, const double* __restrict__ T,
                                                  const int* __restrict__ rgs, int nrg, const int* __restrict__ tgs,
                                                  int ntg, const int* __restrict__ rkp, const int* __restrict__ tkp,
                                                  int dim, K128* __restrict__ keys) {
  __shared__ double s_v[256];
  __shared__ int s_j[256];
  const int g = blockIdx.x;
  if (g >= ntg) return;
  const int t0 = tgs[g], t1 = tgs[g + 1];
  double bv = 1e300;
  int bj = 0x7fffffff;
  for (int j = threadIdx.x; j < nrg; j += blockDim.x) {
    double v = 1e300;
    for (int r = rgs[j]; r < rgs[j + 1]; ++r) {
      const double* rr = R + (size_t)r * dim;
      double rsq = 0.0;
      for (int i = 0; i < dim; ++i) rsq += rr[i] * rr[i];
      for (int t = t0; t < t1; ++t) {
        const double* tt = T + (size_t)t * dim;
        double dot = 0.0;
        for (int i = 0; i < dim; ++i) dot += rr[i] * tt[i];
        v = fmin(v, rsq - 2.0 * dot);
      }
    }
    if (v < bv || (v == bv && j < bj)) { bv = v; bj = j; }
  }
  s_v[threadIdx.x] = bv;
  s_j[threadIdx.x] = bj;
  __syncthreads();
  for (int off = blockDim.x / 2; off; off >>= 1) {
    if ((int)threadIdx.x < off) {
      const double v2 = s_v[threadIdx.x + off];
      const int j2 = s_j[threadIdx.x + off];
      if (v2 < s_v[threadIdx.x] || (v2 == s_v[threadIdx.x] && j2 < s_j[threadIdx.x])) {
        s_v[threadIdx.x] = v2;
        s_j[threadIdx.x] = j2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int j = s_j[0];
    double dmin = 1e300;
    for (int r = rgs[j]; r < rgs[j + 1]; ++r)
      for (int t = t0; t < t1; ++t) {
        double acc = 0.0;
        for (int i = 0; i < dim; ++i) {
          const double d = R[(size_t)r * dim + i] - T[(size_t)t * dim + i];
          acc += d * d;
        }
        dmin = fmin(dmin, acc);
      }
    K128 k;
    k.hi = (unsigned long long)__double_as_longlong(sqrt(dmin));
    k.lo = ((unsigned long long)(unsigned)rkp[rgs[j]] << 32) | (unsigned)tkp[t0];
    keys[g] = k;
  }
}

__global__ void __launch_bounds__(1024) k_vec_groups(const int* __restrict__ kp, int n, int* __restrict__ gs,
                                                     int* __restrict__ ng) {
  __shared__ int s_warp[32];
  __shared__ int s_base, s_tot;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool st = i < n && (i == 0 || kp[i] != kp[i - 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, st);
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { const int t = s_warp[q]; s_warp[q] = run; run += t; }
      s_tot = run;
    }
    __syncthreads();
    if (st) gs[s_base + s_warp[wid] + __popc(bal & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (threadIdx.x == 0) s_base += s_tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) { *ng = s_base; gs[s_base] = n; }
}

__global__ void __launch_bounds__(1024) k_vec_sort(K128* __restrict__ keys, K128* __restrict__ tmp,
                                                   const int* __restrict__ ng, int* __restrict__ out_ref,
                                                   int* __restrict__ out_tgt, double* __restrict__ out_dist,
                                                   int* __restrict__ out_count) {
  extern __shared__ K128 s_keys[];
  const int n = *ng;
  sort_keys_block(keys, tmp, n, s_keys);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    out_dist[i] = __longlong_as_double((long long)keys[i].hi);
    out_ref[i] = (int)(keys[i].lo >> 32);
    out_tgt[i] = (int)(keys[i].lo & 0xffffffffull);
  }
  if (threadIdx.x == 0) *out_count = n;
}

// ------------------------------------------------------------ host
constexpr int kMaxSplits = 8;

struct MatchWs {
  size_t off_part, off_gstart, off_ng, off_rstart, off_rend, off_keys, off_tmp, off_mhist, off_mbase, off_mfill, total;
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

MatchWs plan_match(int n_pairs, int cap) {
  MatchWs p{};
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = al(off + bytes); return o; };
  p.off_part = take((size_t)n_pairs * cap * kMaxSplits * sizeof(Part));
  p.off_gstart = take((size_t)n_pairs * (cap + 1) * sizeof(int));
  p.off_ng = take((size_t)n_pairs * sizeof(int));
  p.off_rstart = take((size_t)n_pairs * cap * sizeof(int));
  p.off_rend = take((size_t)n_pairs * cap * sizeof(int));
  p.off_keys = take((size_t)n_pairs * cap * sizeof(K128));
  p.off_tmp = take((size_t)n_pairs * cap * sizeof(K128));
  p.off_mhist = take((size_t)n_pairs * kMsBins * sizeof(unsigned));
  p.off_mbase = take((size_t)n_pairs * kMsBins * sizeof(unsigned));
  p.off_mfill = take((size_t)n_pairs * kMsBins * sizeof(unsigned));
  p.total = off;
  return p;
}

}  // namespace

size_t match_workspace_bytes(int n_pairs, int cap, int tgt_kp_cap) {
  (void)tgt_kp_cap;
  return plan_match(n_pairs, cap > 0 ? cap : 1).total;
}

namespace {

// Launch k_match_gemm: per target row the exact best reference candidate of
// each column split, into part[pair][cap][splits].  splits <= 0: chosen to
// fill the SMs.  Returns the split count used (negative on error).
int gemm_launch(const MatchArgs& a, Part* part, int splits, cudaStream_t st) {
  if (a.stride != 224 && a.stride != 256) return -2;   // TMA boxes cover K <= 256
  auto encode = get_encode();
  if (!encode) return -3;
  // one descriptor-array tensor map per box shape: A = 128 target rows, B = 128 reference rows
  CUtensorMap tmapA, tmapB;
  cuuint64_t dims[2] = {(cuuint64_t)a.stride, (cuuint64_t)a.n_blocks * a.cap};
  cuuint64_t strides[1] = {(cuuint64_t)a.stride * 2};
  cuuint32_t boxA[2] = {BK, BM}, boxB[2] = {BK, BN};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&tmapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(a.counts), dims, strides,
                       boxA, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return -3;
  cr = encode(&tmapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(a.counts), dims, strides, boxB, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return -3;

  const int m_tiles = (a.cap + BM - 1) / BM;
  if (splits <= 0) {
    static const int forced = [] { const char* e = std::getenv("R2_GEMM_SPLITS"); return e ? std::atoi(e) : 0; }();
    if (forced > 0) splits = forced > kMaxSplits ? kMaxSplits : forced;   // experiment switch
  }
  if (splits <= 0) {
    // split the reference range only as far as needed to put one CTA on every SM:
    // a CTA that sees few column tiles keeps a weak running best and pays the
    // exact-candidate path far more often (~32/(i+1) columns per tile i)
    const int n_tiles_cap = (a.cap + BN - 1) / BN;
    const int ctas = m_tiles * a.n_pairs;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    splits = (n_sm + ctas - 1) / ctas;
    const int max_split = n_tiles_cap / 4 > 1 ? n_tiles_cap / 4 : 1;
    splits = splits > max_split ? max_split : splits;
    splits = splits < 1 ? 1 : (splits > kMaxSplits ? kMaxSplits : splits);
  }
  GemmParams gp{a.sqnorm, a.kp, a.count, a.ref_block, a.tgt_block, a.cap, splits, part};
  cudaFuncSetAttribute(k_match_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_GEMM);
  dim3 grid(m_tiles * splits, a.n_pairs);
  k_match_gemm<<<grid, GEMM_THREADS, SMEM_GEMM, st>>>(tmapA, tmapB, gp);
  return splits;
}

// variant groups, exact combine over the parts, winner distances, (dist, ref, tgt) order
void finish_launch(const MatchArgs& a, const Part* part, int n_parts, PartLayout lay, const MatchWs& p, char* w,
                   cudaStream_t st) {
  IdxWs iw{reinterpret_cast<int*>(w + p.off_gstart), reinterpret_cast<int*>(w + p.off_ng),
           reinterpret_cast<int*>(w + p.off_rstart), reinterpret_cast<int*>(w + p.off_rend)};
  K128* keys = reinterpret_cast<K128*>(w + p.off_keys);
  K128* tmp = reinterpret_cast<K128*>(w + p.off_tmp);
  k_match_index<<<a.n_pairs, 1024, 0, st>>>(a, iw);
  {
    dim3 g2((a.cap + 7) / 8, a.n_pairs);
    k_match_combine<<<g2, 256, 0, st>>>(a, iw, part, n_parts, lay, keys);
  }
  auto* mh = reinterpret_cast<unsigned*>(w + p.off_mhist);
  auto* mb = reinterpret_cast<unsigned*>(w + p.off_mbase);
  auto* mf = reinterpret_cast<unsigned*>(w + p.off_mfill);
  cudaMemsetAsync(mh, 0, (size_t)a.n_pairs * kMsBins * sizeof(unsigned), st);
  cudaMemsetAsync(mf, 0, (size_t)a.n_pairs * kMsBins * sizeof(unsigned), st);
  k_msort_hist<<<dim3(kMsCtas, a.n_pairs), 256, 0, st>>>(iw, keys, a.cap, mh);
  k_msort_scan<<<a.n_pairs, 1024, 0, st>>>(mh, mb);
  k_msort_scatter<<<dim3(kMsCtas, a.n_pairs), 256, 0, st>>>(iw, keys, a.cap, mb, mf, tmp);
  k_msort_rank<<<dim3(kMsCtas, a.n_pairs), 256, 0, st>>>(a, iw, tmp, mh, mb);
}

}  // namespace

int match_run(const MatchArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  const MatchWs p = plan_match(a.n_pairs, a.cap);
  if (ws_bytes < p.total) return 1;
  char* w = static_cast<char*>(ws);
  Part* part = reinterpret_cast<Part*>(w + p.off_part);
  const int splits = gemm_launch(a, part, 0, st);
  if (splits < 0) return -splits;
  finish_launch(a, part, splits, PartLayout{(size_t)a.cap * splits, (size_t)splits, 1}, p, w, st);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

int match_partial_run(const MatchArgs& a, void* parts, cudaStream_t st) {
  const int r = gemm_launch(a, static_cast<Part*>(parts), 1, st);
  if (r < 0) return -r;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

int match_finish_run(const MatchArgs& a, const void* parts, int n_parts, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  const MatchWs p = plan_match(a.n_pairs, a.cap);
  if (ws_bytes < p.total) return 1;
  // the reference rows may be a slice: keypoints without rows get empty ranges
  cudaMemsetAsync(static_cast<char*>(ws) + p.off_rstart, 0, (size_t)a.n_pairs * a.cap * sizeof(int), st);
  cudaMemsetAsync(static_cast<char*>(ws) + p.off_rend, 0, (size_t)a.n_pairs * a.cap * sizeof(int), st);
  finish_launch(a, static_cast<const Part*>(parts), n_parts,
                PartLayout{(size_t)a.cap, 1, (size_t)a.n_pairs * a.cap}, p, static_cast<char*>(ws), st);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2

namespace r2 {

size_t match_vectors_workspace_bytes(int nr, int nt) {
  auto al2 = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return al2((size_t)(nr + 1) * sizeof(int)) + al2((size_t)(nt + 1) * sizeof(int)) + 2 * al2(2 * sizeof(int)) +
         2 * al2((size_t)(nt + 1) * sizeof(K128));
}

int match_vectors_run(const double* R, const int* rkp, int nr, const double* T, const int* tkp, int nt, int dim,
                      int* out_ref, int* out_tgt, double* out_dist, int* out_count, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  if (ws_bytes < match_vectors_workspace_bytes(nr, nt)) return 1;
  auto al2 = [](size_t x) { return (x + 255) & ~(size_t)255; };
  char* w = static_cast<char*>(ws);
  int* rgs = reinterpret_cast<int*>(w);
  w += al2((size_t)(nr + 1) * sizeof(int));
  int* tgs = reinterpret_cast<int*>(w);
  w += al2((size_t)(nt + 1) * sizeof(int));
  int* nrg = reinterpret_cast<int*>(w);
  w += al2(2 * sizeof(int));
  int* ntg = reinterpret_cast<int*>(w);
  w += al2(2 * sizeof(int));
  K128* keys = reinterpret_cast<K128*>(w);
  w += al2((size_t)(nt + 1) * sizeof(K128));
  K128* tmp = reinterpret_cast<K128*>(w);
  k_vec_groups<<<1, 1024, 0, st>>>(rkp, nr, rgs, nrg);
  k_vec_groups<<<1, 1024, 0, st>>>(tkp, nt, tgs, ntg);
  int h_nrg = 0, h_ntg = 0;
  // group counts drive the launch size of this (non hot-path) entry point
  cudaMemcpyAsync(&h_nrg, nrg, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&h_ntg, ntg, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return 3;
  if (h_ntg > 0) k_vec_best<<<h_ntg, 256, 0, st>>>(R, T, rgs, h_nrg, tgs, h_ntg, rkp, tkp, dim, keys);
  const size_t sort_smem = kSortChunk * sizeof(K128);
  cudaFuncSetAttribute(k_vec_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem);
  k_vec_sort<<<1, 1024, sort_smem, st>>>(keys, tmp, ntg, out_ref, out_tgt, out_dist, out_count);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace r2

#ifdef R2_GEMM_TRACE
extern "C" int rift2_debug_gemm_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, r2::g_trace, sizeof(r2::g_trace)) == cudaSuccess ? 0 : 3;
}
extern "C" int rift2_debug_gemm_ctas(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, r2::g_cta, sizeof(r2::g_cta)) == cudaSuccess ? 0 : 3;
}
#endif
