// fastron_device.cuh — device building blocks shared by the sm_100a kernels of the
// Fastron FK hot path: packed-f32x2 arithmetic, the per-control-point RBF term,
// the support-tile layout, mbarrier + cp.async.bulk (TMA bulk copy) helpers.
//
// The FK-kernel term (Eq. 4) is evaluated on PAIRS of control
// points (m, m+1) with the packed FP32 pipe (FADD2/FMUL2/FFMA2) and one MUFU op per
// control point: ex2.approx (Gaussian, north star) or rcp.approx (RQ, Eq. 3,
// PAPER.md:115-117). Positions are pre-scaled so that
//   Gaussian: exp(-gamma d^2) = 2^-(c d)^2,   c = sqrt(gamma log2 e)
//   RQ:       (1 + gamma/2 d^2)^-2 = 1 / (1 + (c d)^2)^2,   c = sqrt(gamma / 2).
// Every kernel that evaluates K_FK (score, Gram, edge) calls term_pair() below with
// identically scaled fp32 inputs, so the same (q, s) pair yields the same bits
// everywhere ("one term function").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fastron {

constexpr int kGaussian = 0;
constexpr int kRQ = 1;         // RQ, fast term (7 packed ops per pair): Gram, lazy columns, edges, scoring pass 1
constexpr int kRQPrecise = 2;  // RQ, Newton-corrected term + offset lanes: the scores near the boundary

// Support tile: TS supports per tile. Each support is MP/2 pair records of 8 floats
// (x_m, x_m+1, y_m, y_m+1, z_m, z_m+1, 0, 0), pre-scaled, followed after the TS
// records by TS alpha values stored as double (the fp64 accumulation operand).
// Padded control points (m >= M) hold kPadCoord so their term is exactly 0; padded
// supports (index >= ns) hold zeros and alpha = 0. The pad keeps d2 finite (3e36 < FLT_MAX):
// an infinite d2 would make the RQ Newton step's rcp(-inf) * inf a NaN; at 3e36 every term
// shape gives exactly 0 (2^-3e36, and (3e36)^-2 underflows).
constexpr int kTileSupports = 64;
constexpr float kPadCoord = 1.0e18f;

__host__ __device__ constexpr int64_t tile_record_floats(int mp) { return (int64_t)kTileSupports * (mp / 2) * 8; }
__host__ __device__ constexpr int64_t tile_floats(int mp) { return tile_record_floats(mp) + 2 * kTileSupports; }
__host__ __device__ constexpr int64_t tile_bytes(int mp) { return tile_floats(mp) * 4; }

// ---------------------------------------------------------------------------------
// packed f32x2 helpers (PTX .f32x2, sm_100a): one instruction, two IEEE rn results
// ---------------------------------------------------------------------------------
typedef unsigned long long f2;

__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo(f2 v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float hi(f2 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float ex2_neg(float x) {  // 2^-x on the MUFU (source negation is free)
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// The RBF terms of control points (m, m+1) for one (query, support) pair.
// Gaussian: d2 = dx*dx; d2 = fma(dy,dy,d2); d2 = fma(dz,dz,d2); t = 2^-d2
// RQ:       w = fma(dx,dx,1); w = fma(dy,dy,w); w = fma(dz,dz,w); t = rcp(w*w)
// (the kernels accumulate through accum_term below, which evaluates RQ as rcp(w)^2)
template <int KIND>
__device__ __forceinline__ f2 term_from_diffs(f2 dx, f2 dy, f2 dz) {
  if (KIND == kGaussian) {
    f2 s = mul2(dx, dx);
    s = fma2(dy, dy, s);
    s = fma2(dz, dz, s);
    return pk(ex2_neg(lo(s)), ex2_neg(hi(s)));
  } else {
    const f2 one = pk(1.0f, 1.0f);
    f2 w = fma2(dx, dx, one);
    w = fma2(dy, dy, w);
    w = fma2(dz, dz, w);
    w = mul2(w, w);
    return pk(rcp_approx(lo(w)), rcp_approx(hi(w)));
  }
}

template <int KIND>
__device__ __forceinline__ f2 term_pair(f2 ux, f2 uy, f2 uz, f2 vx, f2 vy, f2 vz) {
  return term_from_diffs<KIND>(sub2(ux, vx), sub2(uy, vy), sub2(uz, vz));
}

// RQ term evaluation. kRQ (fast): w = 1 + d2 as one FFMA chain seeded with 1, r = rcp(w),
// t = r^2 (7 packed ops per pair; w rounded three times at ulp(w): ~3e-6 rms at the
// headline size — ample for the Gram (relative 1e-4) and for scores away from 0).
// kRQPrecise: s = d2 first (rounded at ulp(d2)), w = 1 + s, r0 = rcp(w), then one Newton
// step against the UNROUNDED 1 + s: e = (1 - r0) - r0 s, r = r0 (1 + e); the residual
// removes both the rounding of w and the rcp.approx error (11 packed ops per pair,
// ~1.4e-6 rms with the offset lanes). The scoring kernels use it for the
// queries whose fast score lies within kRefineTau of 0 (score.cu, pass 2) and for small
// batches. FASTRON_RQ_NEWTON=0 makes kRQPrecise the fast term (A/B).
#ifndef FASTRON_RQ_NEWTON
#define FASTRON_RQ_NEWTON 1
#endif

// acc (+)= the terms of control points (m, m+1): the per-lane running sum over the pairs
// p = 0, 1, ... (first: p == 0, the lane starts from `init`). Every kernel accumulates
// through this one function, so the Gram, the scores and the lazy columns stay
// bit-identical for the same KIND.
// Gaussian: t = 2^-d2 as above, then acc + t. RQ: the square of r = (1 + d2)^-1 rides in
// the accumulating FFMA2. kRQPrecise: the MUFU takes the source negation for free, so the
// Newton step runs on nr0 = rcp(-w) = -r0 without separate negations:
//   u = 1 + nr0 (= 1 - r0, exact for r0 >= 1/2), e = fma(nr0, s, u), nr = fma(nr0, e, nr0)
//   (= -r), acc = fma(nr, nr, acc).
template <int KIND>
__device__ __forceinline__ void accum_term(f2& acc, f2 dx, f2 dy, f2 dz, bool first, f2 init = 0ull) {
  if (KIND == kGaussian) {
    const f2 t = term_from_diffs<KIND>(dx, dy, dz);
    acc = first ? (init ? add2(init, t) : t) : add2(acc, t);
  } else if (KIND == kRQPrecise && FASTRON_RQ_NEWTON) {
    const f2 one = pk(1.0f, 1.0f);
    f2 s = mul2(dx, dx);
    s = fma2(dy, dy, s);
    s = fma2(dz, dz, s);
    const f2 w = add2(s, one);
    const f2 nr0 = pk(rcp_approx(-lo(w)), rcp_approx(-hi(w)));
    const f2 u = add2(one, nr0);
    const f2 e = fma2(nr0, s, u);
    const f2 nr = fma2(nr0, e, nr0);
    acc = fma2(nr, nr, first ? init : acc);
  } else {
    const f2 one = pk(1.0f, 1.0f);
    f2 w = fma2(dx, dx, one);
    w = fma2(dy, dy, w);
    w = fma2(dz, dz, w);
    const f2 r = pk(rcp_approx(lo(w)), rcp_approx(hi(w)));
    acc = first ? (init ? fma2(r, r, init) : mul2(r, r)) : fma2(r, r, acc);
  }
}

// Lane offset of the scoring kernels' precise RQ sums (A/B knob FASTRON_RQ_OFFSET,
// 1 = default). Under RQ every support contributes (k >= 0.14 on these arms), and each fp32
// lane sums NP terms of mean ~0.35 (headline): the rounding of the running sum at
// ulp(~1.4) was ~1.6e-6 rms of the headline score error. Starting each lane from -NP/4
// keeps the running sums near 0; the scoring kernels add 2 * (NP/4) * sum(alpha) back in
// fp64 (exact), so the value is unchanged and only the rounding shrinks.
#ifndef FASTRON_RQ_OFFSET
#define FASTRON_RQ_OFFSET 1
#endif
template <int KIND, int NP>
__host__ __device__ constexpr float rq_lane_offset() {
  return (KIND == kRQPrecise && FASTRON_RQ_OFFSET) ? 0.25f * (float)NP : 0.0f;
}

// Sum over the M control points of one (query, support) pair, in the fixed order
// (t0 + t2 + t4 + ...) + (t1 + t3 + ...): the canonical K_FK numerator shared by all kernels.
__device__ __forceinline__ float pair_sum(f2 acc) { return lo(acc) + hi(acc); }

// fp32 -> fp64 for x >= 0 on the integer (ALU) pipe: exact for normal x; x == 0 maps to
// 2^-127 (< 6e-39, far below any tolerance). cvt.f64.f32 (F2F) would issue on the MUFU
// pipe that bounds this kernel (measured: tools/precision_probe.cu), this does not.
__device__ __forceinline__ double nonneg_f32_to_f64(float x) {
  const uint32_t b = __float_as_uint(x);
  return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}

// The same for either sign (the offset RQ lane sums): magnitude as above, sign bit copied
// (5 ALU instructions).
__device__ __forceinline__ double f32_to_f64_alu(float x) {
  const uint32_t b = __float_as_uint(x);
  return __hiloint2double((int)((((b & 0x7fffffffu) >> 3) + 0x38000000u) | (b & 0x80000000u)), (int)(b << 29));
}

// Promotion of the RQ lane sums: the Newton step leaves the RQ kernel FMA-pipe and issue
// bound with the MUFU only ~60 % busy, so there the conversion instruction (F2F, on the
// MUFU pipe: 2 per support and query) is cheaper than the 2 x 5 ALU instructions of
// f32_to_f64_alu. A/B knob FASTRON_RQ_F2F (1 = default).
#ifndef FASTRON_RQ_F2F
#define FASTRON_RQ_F2F 1
#endif
__device__ __forceinline__ double rq_lane_to_f64(float x) {
#if FASTRON_RQ_F2F
  return (double)x;
#else
  return f32_to_f64_alu(x);
#endif
}

// ---------------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk global -> shared), CTA scope
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}

}  // namespace fastron
