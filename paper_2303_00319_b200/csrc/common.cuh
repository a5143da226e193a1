// Shared helpers for the RIFT2 B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define R2_DEV __device__ __forceinline__

namespace r2 {

// ---- complex float2 arithmetic -------------------------------------------
// sm_100 packed fp32x2 instructions (FADD2 / FMUL2 / FFMA2, with operand
// swap and broadcast modifiers) do a complex add in one instruction and a
// complex multiply in two, halving the FP issue slots of the FFT kernels,
// which are issue/latency bound rather than FP-pipe bound.
#ifndef R2_PACKED
#define R2_PACKED 1
#endif
#if R2_PACKED
R2_DEV float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
R2_DEV float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
R2_DEV float2 cmul(float2 a, float2 b) {
  // (a.x b.x - a.y b.y, a.y b.x + a.x b.y)
  return __ffma2_rn(make_float2(a.y, a.x), make_float2(-b.y, b.y), __fmul2_rn(a, make_float2(b.x, b.x)));
}
// a * (c - i s) for constants c, s: (c a.x + s a.y, c a.y - s a.x)
R2_DEV float2 cmul_cs(float2 a, float c, float s) {
  return __ffma2_rn(make_float2(a.y, a.x), make_float2(s, -s), __fmul2_rn(a, make_float2(c, c)));
}
#else
R2_DEV float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
R2_DEV float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
R2_DEV float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
R2_DEV float2 cmul_cs(float2 a, float c, float s) {
  return make_float2(fmaf(c, a.x, s * a.y), fmaf(c, a.y, -s * a.x));
}
#endif
R2_DEV float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
#if R2_PACKED
R2_DEV float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
#else
R2_DEV float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
#endif
// multiply by -i (forward-transform quarter turn)
R2_DEV float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }

// Padded shared-memory index: one float2 of padding per 32 keeps the
// strided accesses of the FFT passes bank-conflict free.
R2_DEV int pad32(int i) { return i + (i >> 5); }
__host__ __device__ constexpr int padded_len(int n) { return n + (n >> 5) + 1; }

// ---- warp helpers ----------------------------------------------------------
R2_DEV unsigned lane_id() { unsigned r; asm volatile("mov.u32 %0, %%laneid;" : "=r"(r)); return r; }

// named barrier for a group of `nthreads` threads (id 1..15; 0 is __syncthreads)
R2_DEV void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(nthreads) : "memory");
}

// warp-aggregated atomic increment returning this lane's slot
R2_DEV unsigned agg_inc(unsigned* ctr, bool pred) {
  unsigned mask = __ballot_sync(0xffffffffu, pred);
  unsigned slot = 0;
  if (mask) {
    int leader = __ffs(mask) - 1;
    unsigned base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(ctr, (unsigned)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    slot = base + __popc(mask & ((1u << lane_id()) - 1u));
  }
  return slot;
}

}  // namespace r2
