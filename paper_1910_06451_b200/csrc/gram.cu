// gram.cu — K3, the FK-kernel Gram matrix K_ij = K_FK(X_i, X_j) (
// Algorithm 1's "computeKernelMatrixColumn").
//
// Upper-triangular 128x128 tiles (bi <= bj). One CTA of 4 warps owns a column block bj
// and T consecutive row tiles bi of it (T = 1 for shallow triangles, up to 4 for deep
// ones, so the column prologue is paid once per T tiles):
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
// The same term_pair() and control-point summation order as fastron_score make K_ij
// bit-identical to fastron_score(alpha = e_i) for M a power of two; K is exactly
// symmetric (each unordered pair is computed once, or as the exact mirror image on
// diagonal tiles), and K_ii = 1 exactly (d^2 = 0 gives 2^0 = rcp(1) = 1).
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

template <int MP, int KIND, bool JOINT = false>
static cudaError_t run_gram(const float* packed, int64_t n, int M, float* K, int64_t ldk, cudaStream_t st) {
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

cudaError_t launch_gram_joint(const float* packed, int64_t n, int D, int kind, float* K, int64_t ldk, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int Mj = joint_points(D);
  switch (padded_m(Mj)) {
    case 2:
      return kind == kGaussian ? run_gram<2, kGaussian, true>(packed, n, Mj, K, ldk, st)
                               : run_gram<2, kRQ, true>(packed, n, Mj, K, ldk, st);
    case 4:
      return kind == kGaussian ? run_gram<4, kGaussian, true>(packed, n, Mj, K, ldk, st)
                               : run_gram<4, kRQ, true>(packed, n, Mj, K, ldk, st);
    case 6:
      return kind == kGaussian ? run_gram<6, kGaussian, true>(packed, n, Mj, K, ldk, st)
                               : run_gram<6, kRQ, true>(packed, n, Mj, K, ldk, st);
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram(const float* packed, int64_t n, int M, int kind, float* K, int64_t ldk, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int MP = padded_m(M);
#define FASTRON_GCASE(mp)                                                                          \
  case mp:                                                                                         \
    return kind == kGaussian ? run_gram<mp, kGaussian>(packed, n, M, K, ldk, st)                   \
                             : run_gram<mp, kRQ>(packed, n, M, K, ldk, st);
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
