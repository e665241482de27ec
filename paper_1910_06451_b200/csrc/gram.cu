// gram.cu — K3, the FK-kernel Gram matrix K_ij = K_FK(X_i, X_j) (
// Algorithm 1's "computeKernelMatrixColumn").
//
// Two forms, both evaluating every entry with term_pair()'s arithmetic and the control-point
// summation order of fastron_score, so K_ij is bit-identical to fastron_score(alpha = e_i)
// for M a power of two and the two forms give the same matrix bit for bit (tested); K is
// exactly symmetric and K_ii = 1 exactly (d^2 = 0 gives 2^0 = rcp(1) = 1).
//
// Column-slot form (gram2_kernel, MP <= 8 — cfg3 and every M = 8 Gram): the scoring
// kernel's structure with stores in place of the alpha-weighted sum — a CTA owns 384 columns
// (3 per thread, in registers, read coalesced from the positions) and one 64-row tile
// (TMA); see the comment above gram2_kernel. Mirror entries go out in whole 32-byte sectors.
//
// Tile form (gram_kernel, MP > 8 and layouts with ldk % 4 != 0): upper-triangular 128x128
// tiles (bi <= bj). One CTA of 4 warps owns a column block bj and T consecutive row tiles bi
// of it (T = 1 for shallow triangles, up to 4 for deep ones, so the column prologue is paid
// once per T tiles):
//  * COLUMN points live in registers: each lane holds CPL consecutive columns (2 at
//    M <= 16, 1 above) as pre-scaled f32x2 control-point pairs (the packed records of
//    the scoring kernel); a warp covers 32*CPL columns;
//  * each tile's 128 ROW points arrive as two packed support tiles by TMA bulk copies
//    into a 2-stage ring (tile t+1 loads while tile t computes); each warp walks a
//    contiguous row range; a row record is a warp-broadcast LDS.128 + LDS.64 shared by
//    the lane's CPL columns;
//  * the (bi, bj) block is stored straight from registers: for a fixed row each lane
//    writes its CPL consecutive floats as one vector store (the warp covers 32*CPL
//    consecutive floats). The lane keeps its last 4 rows x CPL values in registers and
//    writes the mirrored (bj, bi) block from them: one 16-byte segment per column per 4
//    rows — no shared-memory transpose, about one store per row per lane;
//  * the 4 rows of a chunk are processed pair-major (each control-point pair for all 4
//    rows x CPL columns): 4*CPL independent chains instead of one row's dependency tail;
//  * __launch_bounds__ asks for 4 resident CTAs at M <= 8 and 3 above.
// JOINT = true builds the joint-space RBF Gram of the "Fastron RBF" baseline (PAPER.md:37,
// :114-117) from zero-padded pseudo points: one RBF term of the whole squared distance.
#include <cstdio>

#include "fastron_device.cuh"
#include "internal.h"

namespace fastron {

#ifndef FASTRON_GRAM_WARPS
#define FASTRON_GRAM_WARPS 4
#endif
#ifndef FASTRON_GRAM_CPL8
#define FASTRON_GRAM_CPL8 2
#endif
constexpr int kGT = 32 * FASTRON_GRAM_WARPS;  // threads per Gram CTA
constexpr int kGW = kGT / 32;
constexpr int kGB = 128;             // tile edge (2 support tiles)
#ifndef FASTRON_GRAM_CHUNK
#define FASTRON_GRAM_CHUNK 4
#endif
constexpr int kChunkRows = FASTRON_GRAM_CHUNK;  // rows per mirror chunk (held in registers): 4 or 8

// Work units, column-block-major: column block b holds row tiles 0..b (the upper triangle),
// cut into ceil((b+1)/T) units of T consecutive row tiles. units_before(b) = sum over
// k = 1..b of ceil(k/T) = T*q*(q+1)/2 + r*(q+1) with b = q*T + r.
__host__ __device__ inline int64_t units_before(int64_t b, int T) {
  const int q = (int)b / T, r = (int)b - q * T;  // b < 2^31 (the launch checks units < 2^31)
  return (int64_t)T * q * (q + 1) / 2 + (int64_t)r * (q + 1);
}

__device__ __forceinline__ void unit_coords(int64_t u, int64_t nb, int T, int64_t& bj, int64_t& bi_first) {
  // largest b with units_before(b) <= u: units_before(b) ~ (b^2 + T*b) / (2T), so start
  // from the root of b^2 + T*b - 2*T*u and step to the exact value (no 64-bit divisions)
  const double t = (double)T;
  int64_t b = (int64_t)((sqrt(t * t + 8.0 * t * (double)u) - t) * 0.5);
  b = b < 0 ? 0 : b > nb - 1 ? nb - 1 : b;
  while (b > 0 && units_before(b, T) > u) --b;
  while (b + 1 < nb && units_before(b + 1, T) <= u) ++b;
  bj = b;
  bi_first = (u - units_before(b, T)) * T;
}

#ifndef FASTRON_GRAM_RI4
#define FASTRON_GRAM_RI4 1  // rows interleaved per pair loop at CPL = 4
#endif
#ifndef FASTRON_GRAM_RI2
#define FASTRON_GRAM_RI2 kChunkRows  // ... at CPL <= 2
#endif

__host__ __device__ constexpr int gram_cpl(int mp) {  // columns per lane
  return mp <= 8 ? FASTRON_GRAM_CPL8 : mp <= 16 ? (FASTRON_GRAM_CPL8 < 2 ? FASTRON_GRAM_CPL8 : 2) : 1;
}

// resident CTAs per SM the register allocation must allow: 4 at M <= 8, 3 above
__host__ __device__ constexpr int gram_min_blocks(int mp) { return (mp <= 8 ? 16 : 12) / kGW; }

template <int MP, int KIND, bool JOINT>
__global__ void __launch_bounds__(kGT, gram_min_blocks(MP))
    gram_kernel(const float* __restrict__ packed, int64_t n, int M, int m_pow2, float inv_m, float* __restrict__ K,
                int64_t ldk, int T) {
  constexpr int NP = MP / 2;
  constexpr int CPL = gram_cpl(MP);           // columns per lane
  constexpr int RI = CPL >= 4 ? FASTRON_GRAM_RI4 : FASTRON_GRAM_RI2;  // rows interleaved per pair loop
  constexpr int WC = 32 * CPL;                // columns per warp
  constexpr int G = kGB / WC;                 // column groups (warps sharing a row range)
  constexpr int R = kGW / G;                  // row groups
  constexpr int RW = kGB / R;                 // rows per warp (contiguous)
  constexpr int64_t TF = tile_floats(MP);
  constexpr uint32_t TB = (uint32_t)tile_bytes(MP);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);  // one mbarrier per row stage
  float* const stage0 = reinterpret_cast<float*>(smem_raw + 128);  // stage s: 2 packed tiles at stage0 + 2*TF*s

  // the CTA's unit: column block bj and its row tiles bi_first..bi_last (<= bj), T per unit
  const int64_t nb = (n + kGB - 1) / kGB;
  int64_t bj, bi_first;
  unit_coords(blockIdx.x, nb, T, bj, bi_first);
  const int64_t bi_last = min(bj, bi_first + T - 1);
  const int64_t j0 = bj * kGB;
  const int64_t n_tiles = (n + kTileSupports - 1) / kTileSupports;
  auto issue_rows = [&](int64_t bi, int s) {  // TMA the row tile pair of block bi into stage s
    const int rt = (n_tiles - 2 * bi) >= 2 ? 2 : 1;
    mbar_expect_tx(bar + s, TB * rt);
    for (int c = 0; c < rt; ++c) tma_bulk_g2s(stage0 + (2 * s + c) * TF, packed + (2 * bi + c) * TF, TB, bar + s);
  };

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cg = warp % G, rg = warp / G;
  const int cbase = cg * WC;   // first column of this warp (tile-relative)
  const int rbase = rg * RW;   // first row of this warp (tile-relative)
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) issue_rows(bi_first, 0);

  // the lane's CPL consecutive columns cbase + CPL*lane + h, read from the packed (scaled) records
  f2 ux[CPL][NP], uy[CPL][NP], uz[CPL][NP];
#pragma unroll
  for (int h = 0; h < CPL; ++h) {
    const int64_t j = j0 + cbase + CPL * lane + h;
    const int64_t jj = j < n ? j : 0;
    const float* rec = packed + (jj / kTileSupports) * TF + (jj % kTileSupports) * NP * 8;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float4 xy = __ldg(reinterpret_cast<const float4*>(rec + p * 8));
      const float2 zz = __ldg(reinterpret_cast<const float2*>(rec + p * 8 + 4));
      ux[h][p] = pk(xy.x, xy.y);
      uy[h][p] = pk(xy.z, xy.w);
      uz[h][p] = pk(zz.x, zz.y);
    }
    // odd M: the packed records pad control point MP-1 with a far value; on the column
    // side it becomes 0 (as a scoring query's), so padded - pad is far and the term is
    // exactly 0 — not 1, which pad - pad would give
    if (!JOINT && M < MP) {
      ux[h][NP - 1] = pk(lo(ux[h][NP - 1]), 0.0f);
      uy[h][NP - 1] = pk(lo(uy[h][NP - 1]), 0.0f);
      uz[h][NP - 1] = pk(lo(uz[h][NP - 1]), 0.0f);
    }
  }
  const int64_t c0 = j0 + cbase + CPL * lane;  // the lane's first column
  const bool cols_full = c0 + CPL <= n;
  // vector stores need CPL-float (direct) and 32-byte (mirror) alignment of the rows
  const bool vec_ok = (ldk % 8) == 0 && (reinterpret_cast<uintptr_t>(K) & 31) == 0;

  // the unit's row tiles stream through a 2-stage TMA ring; the columns stay in registers
  for (int64_t bi = bi_first; bi <= bi_last; ++bi) {
  const int t = (int)(bi - bi_first), s = t & 1;
  if (tid == 0 && bi < bi_last) issue_rows(bi + 1, s ^ 1);  // stage s^1 was released below
  mbar_wait(bar + s, (t >> 1) & 1);
  const float* rows = stage0 + 2 * s * TF;
  const int64_t i0 = bi * kGB;
  const bool mirror = bi != bj;
  const int rows_here = (int)min((int64_t)kGB, n - i0);
  // fixed trip counts (no early exits) so loads of the next row overlap this row's math;
  // rows past the matrix edge are computed on stale shared memory but never stored
  const int q_end = min(RW, ((rows_here - rbase + kChunkRows - 1) / kChunkRows) * kChunkRows);
  for (int q0 = 0; q0 < q_end; q0 += kChunkRows) {
    float v[kChunkRows][CPL];  // the chunk's rows x CPL columns, kept for the mirror block
    // pair-major over RI rows at a time: RI x CPL independent accumulation chains per
    // control-point pair (same per-entry summation order as fastron_score)
    f2 acc[kChunkRows][CPL];
#pragma unroll
    for (int q1 = 0; q1 < kChunkRows; q1 += RI) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
#pragma unroll
      for (int qq = q1; qq < q1 + RI; ++qq) {
        const int r = rbase + q0 + qq;
        const float* rec = rows + (r / kTileSupports) * TF + (r % kTileSupports) * NP * 8;
        const float4 xy = *reinterpret_cast<const float4*>(rec + p * 8);
        const float2 zz = *reinterpret_cast<const float2*>(rec + p * 8 + 4);
        const f2 vx = pk(xy.x, xy.y), vy = pk(xy.z, xy.w), vz = pk(zz.x, zz.y);
        f2 dx[CPL], dy[CPL], dz[CPL];
#pragma unroll
        for (int h = 0; h < CPL; ++h) dx[h] = sub2(ux[h][p], vx);
#pragma unroll
        for (int h = 0; h < CPL; ++h) dy[h] = sub2(uy[h][p], vy);
#pragma unroll
        for (int h = 0; h < CPL; ++h) dz[h] = sub2(uz[h][p], vz);
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          if (JOINT) {  // squared joint-space distance, summed over all pseudo points
            acc[qq][h] = p == 0 ? mul2(dx[h], dx[h]) : fma2(dx[h], dx[h], acc[qq][h]);
            acc[qq][h] = fma2(dy[h], dy[h], acc[qq][h]);
            acc[qq][h] = fma2(dz[h], dz[h], acc[qq][h]);
          } else {
            accum_term<KIND>(acc[qq][h], dx[h], dy[h], dz[h], p == 0);
          }
        }
      }
    }
#pragma unroll
    for (int qq = q1; qq < q1 + RI; ++qq) {
      float* Kd = K + (i0 + rbase + q0 + qq) * ldk + c0;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        float x;
        if (JOINT) {
          const float d2 = pair_sum(acc[qq][h]);
          if (KIND == kGaussian) {
            x = ex2_neg(d2);
          } else {
            const float w = 1.0f + d2;
            x = rcp_approx(w * w);
          }
        } else {
          const float ks = pair_sum(acc[qq][h]);
          x = m_pow2 ? ks * inv_m : __fdiv_rn(ks, (float)M);
        }
        v[qq][h] = x;
      }
      // direct block: row i0 + r, the lane's CPL consecutive columns (the warp writes
      // 32*CPL consecutive floats)
      if (rbase + q0 + qq < rows_here) {
        if (CPL == 4 && vec_ok && cols_full) {
          *reinterpret_cast<float4*>(Kd) = make_float4(v[qq][0], v[qq][CPL > 1 ? 1 : 0], v[qq][CPL > 2 ? 2 : 0],
                                                       v[qq][CPL > 3 ? 3 : 0]);
        } else if (CPL == 2 && vec_ok && cols_full) {
          *reinterpret_cast<float2*>(Kd) = make_float2(v[qq][0], v[qq][CPL > 1 ? 1 : 0]);
        } else {
#pragma unroll
          for (int h = 0; h < CPL; ++h)
            if (c0 + h < n) Kd[h] = v[qq][h];
        }
      }
    }
    }
    if (mirror) {
      // mirror block: row c0 + h, columns i0 + rbase + q0 .. +7 (one 32-byte segment)
      const int nrow = min(kChunkRows, rows_here - (rbase + q0));
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        if (c0 + h >= n) continue;
        float* Kr = K + (c0 + h) * ldk + i0 + rbase + q0;
        if (nrow == kChunkRows && vec_ok) {
#pragma unroll
          for (int k4 = 0; k4 < kChunkRows / 4; ++k4)
            reinterpret_cast<float4*>(Kr)[k4] =
                make_float4(v[4 * k4][h], v[4 * k4 + 1][h], v[4 * k4 + 2][h], v[4 * k4 + 3][h]);
        } else {
#pragma unroll
          for (int qq = 0; qq < kChunkRows; ++qq)
            if (qq < nrow) Kr[qq] = v[qq][h];
        }
      }
    }
  }
  __syncthreads();  // every warp is done with stage s before it is refilled
  }
}

// ---------------------------------------------------------------------------------
// K3, column-slot form: the scoring kernel's structure with a store in place of the
// alpha-weighted accumulation.
// ---------------------------------------------------------------------------------
// A CTA of 128 threads owns a column block of W = 128 * QT columns (thread t holds columns
// j0 + j * 128 + t, j < QT, as pre-scaled f32x2 pairs in registers, like a scoring thread's
// QT queries) and ONE 64-row tile of the rows that block needs. Every row record is a
// warp-broadcast LDS.128 + LDS.64 shared by the QT columns; per row a thread computes QT
// entries with term_pair's arithmetic (accum_term, then pair_sum * 1/M: the same bits as
// fastron_score(alpha = e_i) for M a power of two) and stores them: for a fixed row the
// CTA's 128 threads write 128 consecutive floats (one 128-byte line per warp). The mirror
// entries of 4 consecutive rows are kept in registers and written as one 16-byte segment
// per column.
// Which rows a block needs: with NBf = floor(n / W) full blocks and R = n - W NBf remainder
// columns (E = ceil(R / 64) remainder row tiles), full block b takes the row tiles of
// [0, W (b + 1)) — the tiles above its W x W diagonal block (entries stored twice, K[r][c]
// and mirrored K[c][r]) and the diagonal block itself (computed in full, stored directly,
// which covers it) — plus the E remainder tiles (stored twice). The remainder columns then
// need only their own R x R diagonal block: E more units. (A remainder block treated like a
// full one would cost a full block's column of tiles for R live columns: 84 of 630 units
// at cfg3, R = 8.) Units: full block b has TPB (b + 1) + E of them (TPB = W / 64), so
// units_before(b) = QT b (b + 1) + E b, inverted by a square root plus an exact step.
// Predicated global stores with no compiler memory clobber: the kernel never reads K, so
// letting the compiler move shared-memory loads across these stores is safe.
__device__ __forceinline__ void st_global_if(float* p, float v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f32 [%0], %1;\n}" ::"l"(p), "f"(v),
               "r"((int)pred));
}
// one 32-byte store (st.global.v8.f32, sm_100): a whole sector per lane in one instruction
__device__ __forceinline__ void st_global_v8_if(float* p, const float (&v)[8], bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %9, 0;\n @q st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n}" ::"l"(p),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "r"((int)pred));
}
__device__ __forceinline__ void st_global_v4_if(float* p, float a, float b, float c, float d, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q st.global.v4.f32 [%0], {%1, %2, %3, %4};\n}" ::"l"(p),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"((int)pred));
}

constexpr int kG2NT = 128;
#ifndef FASTRON_G2_QT16
#define FASTRON_G2_QT16 2
#endif
__host__ __device__ constexpr int g2_qt(int mp) { return mp <= 8 ? 3 : mp <= 16 ? FASTRON_G2_QT16 : 1; }

// units before column block b (b <= NBf): QT b (b + 1) + E b
// hb: half the unit rows per block width (W / UH / 2: QT for 64-row units, 2 QT for 32-row ones)
__host__ __device__ inline int64_t g2_units_before(int64_t b, int hb, int64_t E) { return (int64_t)hb * b * (b + 1) + E * b; }

struct G2Unit {
  int64_t b;     // column block (NBf: the remainder block)
  int64_t tile;  // row tile
};

__host__ __device__ inline G2Unit g2_unit(int64_t u, int64_t nbf, int hb, int64_t E) {
  // largest b <= nbf with units_before(b) <= u: hb b^2 + (hb + E) b = u
  const double A = (double)hb, B = (double)(hb + E);
  int64_t b = (int64_t)((-B + sqrt(B * B + 4.0 * A * (double)u)) / (2.0 * A));
  b = b < 0 ? 0 : b > nbf ? nbf : b;
  while (b > 0 && g2_units_before(b, hb, E) > u) --b;
  while (b < nbf && g2_units_before(b + 1, hb, E) <= u) ++b;
  const int64_t k = u - g2_units_before(b, hb, E);
  const int64_t tpb = 2 * hb, tf = nbf * tpb;  // unit tiles per block width; first remainder tile
  G2Unit r;
  r.b = b;
  r.tile = b == nbf ? tf + k : (k < tpb * (b + 1) ? k : tf + (k - tpb * (b + 1)));
  return r;
}

// POW2: M is a power of two, so 1/M is an exact multiply (a compile-time choice: a runtime
// branch per row would end the row's basic block and stop the compiler from overlapping
// consecutive rows)
// resident CTAs per SM the register allocation must allow (4 x 4 warps at M <= 8: the
// scoring kernel's occupancy; 2 above)
__host__ __device__ constexpr int g2_min_blocks(int mp) { return mp <= 8 ? 4 : g2_qt(mp) <= 2 ? 3 : 2; }

// RP (rows packed): the row tile comes from the pack kernel's tiles by one TMA bulk copy (the
// A/B winner above M = 8: cfg5 0.892 against 0.929 ms with rows from the positions); else
// the CTA reads its rows from the positions itself and no pack kernel runs (cfg3 52.1 ->
// 45.8 us per fastron_gram call: the pack launch and its round trip were ~6 us of it).
__host__ __device__ constexpr bool g2_rows_packed(int mp) { return mp > 8; }

// V8: the 8-row mirror sector as one 256-bit store per column (needs 32-byte aligned rows:
// ldk % 8 == 0); a compile-time choice — as a runtime branch it cost cfg3 2 us (spills)
// UH: rows per unit (64, or 32 for shallow triangles: twice the units, so the block
// scheduler can even out the SMs' loads); the packed row tiles (RP) need 64
template <int MP, int KIND, bool JOINT, bool POW2, bool V8, int UH>
__global__ void __launch_bounds__(kG2NT, g2_min_blocks(MP)) gram2_kernel(const float* __restrict__ packed,
                                                                         const float4* __restrict__ pos, int64_t ldp,
                                                                         float scale, int64_t n, int M, float inv_m,
                                                                         float* __restrict__ K, int64_t ldk, int smask) {
  constexpr int QT = g2_qt(MP);
  constexpr int NP = MP / 2;
  constexpr int W = kG2NT * QT;
  constexpr int TS = UH;
  constexpr bool RP = g2_rows_packed(MP);
  static_assert(!RP || UH == kTileSupports, "packed row tiles are 64 rows");
  constexpr int64_t TF = tile_floats(MP);
  // planes (!RP): the tile's 64 row points s_xy[p][s] = (x_2p, x_2p+1, y_2p, y_2p+1) and
  // s_z[p][s] = (z_2p, z_2p+1) of row s, pre-scaled (the packed record's contents)
  __shared__ float4 s_xy[RP ? 1 : NP][TS];
  __shared__ float2 s_z[RP ? 1 : NP][TS];
  __shared__ __align__(128) float s_tile[RP ? TF : 4];  // RP: the packed tile (records, then alpha)
  __shared__ uint64_t s_bar;

  constexpr int HB = W / UH / 2;
  const int64_t nbf = n / W, E = (n - nbf * W + UH - 1) / UH;
  const G2Unit U = g2_unit(blockIdx.x, nbf, HB, E);
  const int64_t j0 = U.b * W;
  const int64_t r0 = U.tile * UH;
  const int rows_here = (int)min((int64_t)UH, n - r0);
  const bool mirror = r0 < j0 || r0 >= j0 + W;  // outside the block's diagonal square: store both
  const int tid = threadIdx.x;
#ifdef FASTRON_GRAM_PROF
  unsigned long long t_start, t_pro = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  if (RP && tid == 0) {
    mbar_init(&s_bar, 1);
    fence_barrier_init();
    mbar_expect_tx(&s_bar, (uint32_t)(TF * 4));
    tma_bulk_g2s(s_tile, packed + U.tile * TF, (uint32_t)(TF * 4), &s_bar);
  }
  // !RP: the row points, straight from the positions: thread (s, p) loads control points 2p
  // and 2p+1 of row r0 + s (consecutive threads, consecutive 16-byte elements) and scales
  // them as the pack kernel scales a support (__fmul_rn by the same constant, the padded
  // point m = M of an odd M at kPadCoord, rows past n zero) — the same bits as the packed
  // tile, with no pack kernel and no copy in between
  constexpr int RIT = (NP * TS + kG2NT - 1) / kG2NT;  // row items per thread (compile time: loads batched)
  float4 ra[RIT], rb[RIT];
#pragma unroll
  for (int it = 0; it < RIT; ++it) {
    const int idx = it * kG2NT + tid, sr = idx % TS, p = idx / TS;
    const int64_t r = r0 + sr;
    ra[it] = rb[it] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!RP && idx < NP * TS && r < n) {
      ra[it] = __ldg(pos + (int64_t)(2 * p) * ldp + r);
      if (2 * p + 1 < M) rb[it] = __ldg(pos + (int64_t)(2 * p + 1) * ldp + r);
    }
  }
#pragma unroll
  for (int it = 0; it < RIT; ++it) {
    const int idx = it * kG2NT + tid, sr = idx % TS, p = idx / TS;
    if (RP || idx >= NP * TS) continue;
    const float4 a = ra[it], b = rb[it];
    float bx = __fmul_rn(b.x, scale), by = __fmul_rn(b.y, scale), bz = __fmul_rn(b.z, scale);
    if (2 * p + 1 >= M) bx = by = bz = JOINT ? 0.0f : kPadCoord;
    s_xy[p][sr] = make_float4(__fmul_rn(a.x, scale), bx, __fmul_rn(a.y, scale), by);
    s_z[p][sr] = make_float2(__fmul_rn(a.z, scale), bz);
  }

  // the thread's QT columns straight from the control-point positions (SoA float4 [M][ldp]:
  // consecutive threads read consecutive 16-byte elements, all QT * M loads in flight at
  // once), scaled exactly as the pack kernel scales the row records (__fmul_rn by the same
  // constant: the same bits); padded control points m >= M are 0 on the column side, so
  // against a row's padded point the term is exactly 0. Reading the packed records instead
  // (one 128-byte record per lane) put 32 lines behind every load instruction and left the
  // columns arriving ~4 us after the CTA started (-DFASTRON_GRAM_PROF).
  f2 ux[QT][NP], uy[QT][NP], uz[QT][NP];
  bool col_ok[QT];
#pragma unroll
  for (int j = 0; j < QT; ++j) {
    const int64_t c = j0 + j * kG2NT + tid;
    col_ok[j] = c < n;
    float px[MP], py[MP], pz[MP];
#pragma unroll
    for (int m = 0; m < MP; ++m) {
      px[m] = py[m] = pz[m] = 0.0f;
      if (m < M && col_ok[j]) {
        const float4 v = __ldg(pos + (int64_t)m * ldp + c);
        px[m] = __fmul_rn(v.x, scale);
        py[m] = __fmul_rn(v.y, scale);
        pz[m] = __fmul_rn(v.z, scale);
      }
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      ux[j][p] = pk(px[2 * p], px[2 * p + 1]);
      uy[j][p] = pk(py[2 * p], py[2 * p + 1]);
      uz[j][p] = pk(pz[2 * p], pz[2 * p + 1]);
    }
  }
  float* Kd = K + r0 * ldk + j0 + tid;  // row r0, the thread's first column
  float* const Kc = K + (j0 + tid) * ldk + r0;  // row c = j0 + tid, column r0: the mirror entries
  const int64_t kc_step = (int64_t)kG2NT * ldk;  // to the thread's next column slot
#ifdef FASTRON_GRAM_PROF
  unsigned long long t_cols;
  {
    float sink = lo(ux[0][0]) + lo(uy[QT - 1][NP - 1]) + lo(uz[QT - 1][0]);
    if (sink == -12345.f) K[0] = sink;  // the column loads have landed
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_cols));
  }
#endif
  __syncthreads();  // the row planes are complete (RP: the barrier's initialisation is visible)
  if (RP) mbar_wait(&s_bar, 0u);
#ifdef FASTRON_GRAM_PROF
  {
    float sink = lo(ux[0][0]) + lo(uy[QT - 1][NP - 1]);
    if (sink == -12345.f) K[0] = sink;  // the column loads have landed
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_pro));
  }
#endif

  // 4 rows: their QT x 4 entries first (12 independent chains at QT = 3), then the direct
  // stores (128 consecutive floats per row and column slot)
  auto rows4 = [&](int c4, float (&v)[4][QT]) {
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      f2 acc[QT];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        float4 xy;
        float2 zz;
        if (RP) {
          const float* rec = s_tile + (c4 + rr) * NP * 8 + p * 8;
          xy = *reinterpret_cast<const float4*>(rec);
          zz = *reinterpret_cast<const float2*>(rec + 4);
        } else {
          xy = s_xy[p][c4 + rr];
          zz = s_z[p][c4 + rr];
        }
        const f2 vx = pk(xy.x, xy.y), vy = pk(xy.z, xy.w), vz = pk(zz.x, zz.y);
        f2 dx[QT], dy[QT], dz[QT];
#pragma unroll
        for (int j = 0; j < QT; ++j) dx[j] = sub2(ux[j][p], vx);
#pragma unroll
        for (int j = 0; j < QT; ++j) dy[j] = sub2(uy[j][p], vy);
#pragma unroll
        for (int j = 0; j < QT; ++j) dz[j] = sub2(uz[j][p], vz);
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          if (JOINT) {  // squared joint-space distance, summed over all pseudo points
            acc[j] = p == 0 ? mul2(dx[j], dx[j]) : fma2(dx[j], dx[j], acc[j]);
            acc[j] = fma2(dy[j], dy[j], acc[j]);
            acc[j] = fma2(dz[j], dz[j], acc[j]);
          } else {
            accum_term<KIND>(acc[j], dx[j], dy[j], dz[j], p == 0);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < QT; ++j) {
        if (JOINT) {
          const float d2 = pair_sum(acc[j]);
          if (KIND == kGaussian) {
            v[rr][j] = ex2_neg(d2);
          } else {
            const float w = 1.0f + d2;
            v[rr][j] = rcp_approx(w * w);
          }
        } else {
          const float ks = pair_sum(acc[j]);
          v[rr][j] = POW2 ? ks * inv_m : __fdiv_rn(ks, (float)M);
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
      for (int j = 0; j < QT; ++j)
        st_global_if(Kd + j * kG2NT, v[rr][j], col_ok[j] && c4 + rr < rows_here && (smask & 1));
      Kd += ldk;
    }
  };
  // mirror entries K[c][r0 + c8 .. + 7] in whole 32-byte sectors (two 16-byte stores per
  // column and 8 rows): 16-byte half-sector writes ran at ~1.2 TB/s against ~4 TB/s for
  // full sectors (tools/store_probe.cu), which bounded the Gram at large N
  auto mirror_rows = [&](int c, int nrows, const float (&v)[4][QT]) {  // rows c .. c + nrows - 1 (<= 4)
#pragma unroll
    for (int j = 0; j < QT; ++j) {
      float* Kr = Kc + j * kc_step + c;
      if (nrows == 4) {
        st_global_v4_if(Kr, v[0][j], v[1][j], v[2][j], v[3][j], col_ok[j]);
      } else {
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) st_global_if(Kr + rr, v[rr][j], col_ok[j] && rr < nrows);
      }
    }
  };
  const bool do_mirror = mirror && (smask & 2);
#pragma unroll 1
  for (int c8 = 0; c8 < rows_here; c8 += 8) {
    // both halves always (rows past n read the tile's zero padding and are never stored):
    // one basic block, so the compiler may overlap the two halves
    float va[4][QT], vb[4][QT];
    rows4(c8, va);
    rows4(c8 + 4, vb);
    const bool second = c8 + 4 < rows_here;
    if (do_mirror) {
      if (c8 + 8 <= rows_here) {  // the usual case: one full sector per column
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          float* Kr = Kc + j * kc_step + c8;
          if (V8) {  // one 256-bit store per column (A/B: cfg3 45.8 -> 43.9 us, cfg5 0.90 -> 0.87 ms)
            const float w8[8] = {va[0][j], va[1][j], va[2][j], va[3][j], vb[0][j], vb[1][j], vb[2][j], vb[3][j]};
            st_global_v8_if(Kr, w8, col_ok[j]);
          } else {
            st_global_v4_if(Kr, va[0][j], va[1][j], va[2][j], va[3][j], col_ok[j]);
            st_global_v4_if(Kr + 4, vb[0][j], vb[1][j], vb[2][j], vb[3][j], col_ok[j]);
          }
        }
      } else {  // the matrix's last rows
        mirror_rows(c8, min(4, rows_here - c8), va);
        if (second) mirror_rows(c8 + 4, rows_here - c8 - 4, vb);
      }
    }
  }
#ifdef FASTRON_GRAM_PROF
  if (tid == 0) {
    unsigned long long t_end;
    unsigned int smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("gram prof unit %d sm %u start %llu first-tile %llu end %llu rows %d cols %llu\n", blockIdx.x, smid, t_start,
           t_pro - t_start, t_end, rows_here, t_cols - t_start);
  }
#endif
}

template <int MP, int KIND, bool JOINT, bool POW2, bool V8, int UH>
static cudaError_t run_gram2_u(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M, float* K,
                               int64_t ldk, cudaStream_t st) {
  constexpr int W = kG2NT * g2_qt(MP);
  const int64_t nbf = n / W, R = n - nbf * W, E = (R + UH - 1) / UH;
  const int64_t units = g2_units_before(nbf, W / UH / 2, E) + (R > 0 ? E : 0);
  if (units > 0x7fffffff) return cudaErrorInvalidValue;
  static const int smask = [] {  // probing only: 1 direct stores, 2 mirror stores
    const char* e = getenv("FASTRON_GRAM_STORES");
    return e ? atoi(e) : 3;
  }();
  gram2_kernel<MP, KIND, JOINT, POW2, V8, UH><<<(unsigned)units, kG2NT, 0, st>>>(packed, pos, ldp, scale, n, M,
                                                                              1.0f / (float)M, K, ldk, smask);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

// 32-row units while the 64-row triangle fills at most half the resident slots (N = 2,560:
// 27.6 -> 22.6 us); at cfg3 (560 units for 592 slots) they measured equal (44.6 vs 44.4 us:
// the better balance over SMs is paid back in twice the CTA prologues); FASTRON_GRAM_UH overrides
template <int MP, int KIND, bool JOINT, bool POW2>
static cudaError_t run_gram2_m(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M, float* K,
                               int64_t ldk, cudaStream_t st) {
  if (g2_rows_packed(MP)) {
    const cudaError_t pe = launch_pack(pos, ldp, nullptr, n, M, scale, packed, st, JOINT);
    if (pe != cudaSuccess) return pe;
  }
  const bool v8 = (ldk % 8) == 0 && (reinterpret_cast<uintptr_t>(K) & 31) == 0;
  bool half = false;
  if constexpr (!g2_rows_packed(MP)) {
    constexpr int W = kG2NT * g2_qt(MP);
    const int64_t nbf = n / W, E = (n - nbf * W + 63) / 64;
    const int64_t units64 = g2_units_before(nbf, W / 64 / 2, E) + E;
    static const int env = [] {
      const char* e = getenv("FASTRON_GRAM_UH");
      return e ? atoi(e) : 0;
    }();
    half = env ? env == 32 : 2 * units64 <= (int64_t)device_info().sms * g2_min_blocks(MP);
    if (half)
      return v8 ? run_gram2_u<MP, KIND, JOINT, POW2, true, 32>(packed, pos, ldp, scale, n, M, K, ldk, st)
                : run_gram2_u<MP, KIND, JOINT, POW2, false, 32>(packed, pos, ldp, scale, n, M, K, ldk, st);
  }
  return v8 ? run_gram2_u<MP, KIND, JOINT, POW2, true, 64>(packed, pos, ldp, scale, n, M, K, ldk, st)
            : run_gram2_u<MP, KIND, JOINT, POW2, false, 64>(packed, pos, ldp, scale, n, M, K, ldk, st);
}

template <int MP, int KIND, bool JOINT>
static cudaError_t run_gram(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M, float* K,
                            int64_t ldk, cudaStream_t st);

template <int MP, int KIND, bool JOINT>
static cudaError_t run_gram2(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M,
                             float* K, int64_t ldk, cudaStream_t st) {
  // the mirror's 16-byte stores need ldk % 4 == 0 and a 16-byte aligned K; other layouts
  // take the tile form
  if ((ldk % 4) != 0 || (reinterpret_cast<uintptr_t>(K) & 15) != 0)
    return run_gram<MP, KIND, JOINT>(packed, pos, ldp, scale, n, M, K, ldk, st);
  // JOINT takes no 1/M; the exact-multiply instance exists where M can be a power of two
  constexpr bool kCanPow2 = !JOINT && (MP & (MP - 1)) == 0;
  if constexpr (JOINT) {
    return run_gram2_m<MP, KIND, JOINT, true>(packed, pos, ldp, scale, n, M, K, ldk, st);
  } else if constexpr (kCanPow2) {
    if ((M & (M - 1)) == 0) return run_gram2_m<MP, KIND, JOINT, true>(packed, pos, ldp, scale, n, M, K, ldk, st);
  }
  if constexpr (!JOINT) return run_gram2_m<MP, KIND, JOINT, false>(packed, pos, ldp, scale, n, M, K, ldk, st);
  return cudaErrorInvalidValue;
}

// row tiles per CTA: 1 while the triangle is only a few waves deep (occupancy first);
// for deep triangles up to 4, keeping >= ~4 waves of units so the tail stays short
// (measured at N = 20,000, M = 16: T = 1, 2, 4, 6, 8 -> 1.11, 1.03, 1.01, 1.03, 1.05 ms).
// Two row stages then cost 4 tiles of shared memory, which fits the resident CTAs for
// MP <= 16 only. FASTRON_GRAM_T overrides (probing).
static int gram_rows_per_unit(int64_t tiles, int mp) {
  static const int env = [] {
    const char* e = getenv("FASTRON_GRAM_T");
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env;
  if (mp > 16) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t slots = (int64_t)sms * gram_min_blocks(mp);
  int64_t T = tiles / (4 * slots);
  return (int)(T < 1 ? 1 : T > 4 ? 4 : T);
}

template <int MP, int KIND, bool JOINT>
static cudaError_t run_gram(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M, float* K,
                            int64_t ldk, cudaStream_t st) {
  // the tile form streams packed support tiles: pack the points first
  cudaError_t pe = launch_pack(pos, ldp, nullptr, n, M, scale, packed, st, JOINT);
  if (pe != cudaSuccess) return pe;
  const int64_t nb = (n + kGB - 1) / kGB;
  const int64_t tiles = nb * (nb + 1) / 2;
  const int T = gram_rows_per_unit(tiles, MP);
  const size_t smem = 128 + (T > 1 ? 4 : 2) * tile_bytes(MP);  // one or two row stages
  static std::atomic<int> attr[kMaxDevices];
  const int dev = device_slot();
  if (!attr[dev].load()) {
    cudaFuncSetAttribute(gram_kernel<MP, KIND, JOINT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(128 + 4 * tile_bytes(MP)));
    attr[dev].store(1);
  }
  const int64_t units = units_before(nb, T);
  if (units > 0x7fffffff) return cudaErrorInvalidValue;
  const int m_pow2 = (M & (M - 1)) == 0;
  gram_kernel<MP, KIND, JOINT><<<(unsigned)units, kGT, smem, st>>>(packed, n, M, m_pow2, 1.0f / (float)M, K, ldk, T);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

// Which form runs: the column-slot form up to MP = FASTRON_G2_MAXMP, the tile form above and
// for ldk % 4 != 0. A/B on one box (bit-identical matrices): cfg3 52.0 vs 58.4 us; N = 20,000
// at M = 8 0.55 vs 1.02 ms; cfg5 (M = 16) with 2 columns per thread (168 registers, 3 CTAs
// per SM) 0.896 vs 1.008 ms — with 3 (255 registers, 2 CTAs per SM) it was 1.05 ms.
#ifndef FASTRON_G2_MAXMP
#define FASTRON_G2_MAXMP 16
#endif
template <int MP, int KIND, bool JOINT>
static cudaError_t run_gram_any(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M,
                                float* K, int64_t ldk, cudaStream_t st) {
  if constexpr (MP <= FASTRON_G2_MAXMP) return run_gram2<MP, KIND, JOINT>(packed, pos, ldp, scale, n, M, K, ldk, st);
  else return run_gram<MP, KIND, JOINT>(packed, pos, ldp, scale, n, M, K, ldk, st);
}
#define FASTRON_RUN_GRAM run_gram_any

cudaError_t launch_gram_joint(float* packed, const float4* pts, float scale, int64_t n, int D, int kind, float* K,
                              int64_t ldk, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int Mj = joint_points(D);
  switch (padded_m(Mj)) {
    case 2:
      return kind == kGaussian ? FASTRON_RUN_GRAM<2, kGaussian, true>(packed, pts, n, scale, n, Mj, K, ldk, st)
                               : FASTRON_RUN_GRAM<2, kRQ, true>(packed, pts, n, scale, n, Mj, K, ldk, st);
    case 4:
      return kind == kGaussian ? FASTRON_RUN_GRAM<4, kGaussian, true>(packed, pts, n, scale, n, Mj, K, ldk, st)
                               : FASTRON_RUN_GRAM<4, kRQ, true>(packed, pts, n, scale, n, Mj, K, ldk, st);
    case 6:
      return kind == kGaussian ? FASTRON_RUN_GRAM<6, kGaussian, true>(packed, pts, n, scale, n, Mj, K, ldk, st)
                               : FASTRON_RUN_GRAM<6, kRQ, true>(packed, pts, n, scale, n, Mj, K, ldk, st);
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M, int kind,
                        float* K, int64_t ldk, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int MP = padded_m(M);
#define FASTRON_GCASE(mp)                                                                          \
  case mp:                                                                                         \
    return kind == kGaussian ? FASTRON_RUN_GRAM<mp, kGaussian, false>(packed, pos, ldp, scale, n, M, K, ldk, st) \
                             : FASTRON_RUN_GRAM<mp, kRQ, false>(packed, pos, ldp, scale, n, M, K, ldk, st);
  switch (MP) {
    FASTRON_GCASE(2)
    FASTRON_GCASE(4)
    FASTRON_GCASE(6)
    FASTRON_GCASE(8)
    FASTRON_GCASE(10)
    FASTRON_GCASE(12)
    FASTRON_GCASE(14)
    FASTRON_GCASE(16)
    FASTRON_GCASE(18)
    FASTRON_GCASE(20)
    FASTRON_GCASE(22)
    FASTRON_GCASE(24)
    FASTRON_GCASE(26)
    FASTRON_GCASE(28)
    FASTRON_GCASE(30)
    FASTRON_GCASE(32)
    default:
      return cudaErrorInvalidValue;
  }
#undef FASTRON_GCASE
}

}  // namespace fastron
