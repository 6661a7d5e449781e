// tcgen05 (5th-generation tensor core) helpers: TMEM allocation, UMMA
// shared-memory / instruction descriptors, MMA issue, commit and TMEM loads.
#pragma once

#include <stdint.h>

#include "akv_tma.cuh"

namespace akv {

// UMMA shared-memory descriptor of a K-major operand stored as 128-byte
// swizzled rows (the TMA SWIZZLE_128B layout): start address, LBO = 1
// (ignored for swizzled K-major), SBO = 1024 B between 8-row groups,
// version 1 (Blackwell), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  return (uint64_t)((smem_addr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 accumulator, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// arrive on `bar` when every previously issued tcgen05.mma has completed
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// one full warp: allocate `cols` TMEM columns, base address written to smem
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 64 consecutive fp32 columns of this thread's TMEM lane: two x32 loads in
// flight behind one wait
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
  uint32_t r[64];
#define AKV_LD32(OFF, R)                                                                        \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"        \
      : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]),   \
        "=r"(R[7]), "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]),             \
        "=r"(R[13]), "=r"(R[14]), "=r"(R[15]), "=r"(R[16]), "=r"(R[17]), "=r"(R[18]),          \
        "=r"(R[19]), "=r"(R[20]), "=r"(R[21]), "=r"(R[22]), "=r"(R[23]), "=r"(R[24]),          \
        "=r"(R[25]), "=r"(R[26]), "=r"(R[27]), "=r"(R[28]), "=r"(R[29]), "=r"(R[30]),          \
        "=r"(R[31])                                                                             \
      : "r"(taddr + (OFF)))
  AKV_LD32(0, r);
  AKV_LD32(32, (r + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// 128 consecutive fp32 columns (a full 128-wide accumulator row): four x32
// loads in flight behind one wait
__device__ __forceinline__ void tmem_ld128(uint32_t taddr, float* v) {
  uint32_t r[128];
  AKV_LD32(0, r);
  AKV_LD32(32, (r + 32));
  AKV_LD32(64, (r + 64));
  AKV_LD32(96, (r + 96));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 128; ++i) v[i] = __uint_as_float(r[i]);
}
#undef AKV_LD32

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2: two lanes of work per issued
// instruction) for the softmax epilogues.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// exp2 of both lanes (MUFU)
__device__ __forceinline__ uint64_t f2_exp2(uint64_t x) {
  float a, b;
  f2_unpack(x, a, b);
  float ya, yb;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ya) : "f"(a));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(yb) : "f"(b));
  return f2_pack(ya, yb);
}

// 2^x for x <= 0 on the FMA pipe (MUFU stays free for the other lanes of the
// work): x = j + f with j = round(x) taken from the mantissa of x + 1.5*2^23,
// 2^f on [-0.5, 0.5] by a degree-5 minimax polynomial (max relative error
// 1.9e-7 in fp32, like ex2.approx), 2^j added to the exponent field.  Inputs
// below -125 clamp (the result is < 2^-125, negligible next to any sum of
// probabilities); the caller guarantees x <= 0 (x - running max).
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = 1.3264727e-3f;
  p = fmaf(p, f, 9.6715129e-3f);
  p = fmaf(p, f, 5.5507337e-2f);
  p = fmaf(p, f, 2.4022242e-1f);
  p = fmaf(p, f, 6.9314698e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// exp2_fma on both lanes of a packed pair: FADD2 / FFMA2 for the rounding
// split and the polynomial, scalar clamp and exponent insertion
__device__ __forceinline__ uint64_t f2_exp2_fma(uint64_t x2) {
  float a, b;
  f2_unpack(x2, a, b);
  x2 = f2_pack(fmaxf(a, -125.f), fmaxf(b, -125.f));
  const uint64_t M = f2_pack(12582912.f, 12582912.f), nM = f2_pack(-12582912.f, -12582912.f);
  const uint64_t t = f2_add(x2, M);
  uint64_t f;
  {
    float r0, r1, x0, x1;
    f2_unpack(f2_add(t, nM), r0, r1);
    f2_unpack(x2, x0, x1);
    f = f2_add(x2, f2_pack(-r0, -r1));
  }
  uint64_t p = f2_pack(1.3264727e-3f, 1.3264727e-3f);
  p = f2_fma(p, f, f2_pack(9.6715129e-3f, 9.6715129e-3f));
  p = f2_fma(p, f, f2_pack(5.5507337e-2f, 5.5507337e-2f));
  p = f2_fma(p, f, f2_pack(2.4022242e-1f, 2.4022242e-1f));
  p = f2_fma(p, f, f2_pack(6.9314698e-1f, 6.9314698e-1f));
  p = f2_fma(p, f, f2_pack(1.0f, 1.0f));
  float p0, p1, t0, t1;
  f2_unpack(p, p0, p1);
  f2_unpack(t, t0, t1);
  return f2_pack(__int_as_float(__float_as_int(p0) + ((__float_as_int(t0) - 0x4B400000) << 23)),
                 __int_as_float(__float_as_int(p1) + ((__float_as_int(t1) - 0x4B400000) << 23)));
}

// share of the exponentials of the unmasked row-pass tiles evaluated on the
// FMA pipe: every kPolyEvery-th pair, 0 = none.  Measured at config 4 (B200):
// row pass 5.67 -> 5.40 ms with a quarter on the FMA pipe; neither the MUFU
// (XU ~60 %) nor the issue slots (~64 %) saturate - the epilogue is latency
// bound at 16 epilogue warps per SM.  An eighth (kPolyEvery 8): K1 at config 1
// 0.2013 -> 0.1981 ms, config 4 unchanged (2 of 8 on the FMA pipe: slower).
#ifndef AKV_POLY_EVERY
#define AKV_POLY_EVERY 8
#endif
constexpr int kPolyEvery = AKV_POLY_EVERY;

__device__ __forceinline__ float exp2_mixed(float x, int c) {
  return (kPolyEvery > 0 && c % (kPolyEvery > 0 ? kPolyEvery : 1) == kPolyEvery - 1)
             ? exp2_fma(x) : fast_exp2(x);
}

}  // namespace akv
