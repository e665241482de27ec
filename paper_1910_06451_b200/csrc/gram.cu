// gram.cu — K3, the FK-kernel Gram matrix K_ij = K_FK(X_i, X_j) (
// Algorithm 1 line "computeKernelMatrixColumn").
//
// Upper-triangular 128x128 tiles, one CTA per tile (bi <= bj). The 128 column points
// arrive as two packed support tiles by TMA bulk copy; each of the 256 threads holds
// 2 row points in registers and evaluates 2 x 32 entries with the same term_pair()
// as the scoring kernel, so K_ij is bit-identical to fastron_score with alpha = e_i
// (the sum over m in the same order, then the exact 1/M for M a power of two).
// The tile is staged in shared memory (row stride 129 floats: conflict-free
// transposed reads) and written twice with coalesced stores: as (bi, bj) and, off the
// diagonal, transposed as (bj, bi). K is therefore exactly symmetric and its diagonal
// is exactly 1 (d^2 = 0 gives 2^0 = rcp(1) = 1).
#include "fastron_device.cuh"
#include "internal.h"

namespace fastron {

constexpr int kGT = 256;   // threads per Gram CTA
constexpr int kGB = 128;   // tile edge (2 support tiles)
constexpr int kGS = kGB + 1;

__device__ __forceinline__ void tile_coords(int64_t t, int64_t nb, int64_t& bi, int64_t& bj) {
  // row-major enumeration of the upper triangle: row bi holds tiles bi..nb-1
  double d = (double)(2 * nb + 1);
  int64_t r = (int64_t)((d - sqrt(d * d - 8.0 * (double)t)) * 0.5);
  auto start = [&](int64_t row) { return row * nb - row * (row - 1) / 2; };
  while (r > 0 && start(r) > t) --r;
  while (start(r + 1) <= t) ++r;
  bi = r;
  bj = r + (t - start(r));
}

template <int MP, int KIND>
__global__ void __launch_bounds__(kGT) gram_kernel(const float* __restrict__ packed, int64_t n, int M, int m_pow2,
                                                   float inv_m, float* __restrict__ K, int64_t ldk) {
  constexpr int NP = MP / 2;
  constexpr int64_t TF = tile_floats(MP);
  constexpr uint32_t TB = (uint32_t)tile_bytes(MP);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  float* cols = reinterpret_cast<float*>(smem_raw + 128);      // 2 packed tiles
  float* Ks = cols + 2 * TF;                                    // [128][129]

  const int64_t nb = (n + kGB - 1) / kGB;
  int64_t bi, bj;
  tile_coords(blockIdx.x, nb, bi, bj);
  const int64_t i0 = bi * kGB, j0 = bj * kGB;
  const int64_t n_tiles = (n + kTileSupports - 1) / kTileSupports;
  const int ct = (n_tiles - 2 * bj) >= 2 ? 2 : 1;  // column tiles present

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(bar, TB * ct);
    for (int c = 0; c < ct; ++c) tma_bulk_g2s(cols + c * TF, packed + (2 * bj + c) * TF, TB, bar);
  }

  // rows r and r + 64 of the row block, read from the same packed (scaled) records
  const int r = tid & 63;
  const int cg = tid >> 6;  // column group of 32
  f2 ux[2][NP], uy[2][NP], uz[2][NP];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + r + 64 * h;
    const int64_t ii = i < n ? i : 0;
    const float* rec = packed + (ii / kTileSupports) * TF + (ii % kTileSupports) * NP * 8;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float4 xy = __ldg(reinterpret_cast<const float4*>(rec + p * 8));
      const float2 zz = __ldg(reinterpret_cast<const float2*>(rec + p * 8 + 4));
      ux[h][p] = pk(xy.x, xy.y);
      uy[h][p] = pk(xy.z, xy.w);
      uz[h][p] = pk(zz.x, zz.y);
    }
  }
  mbar_wait(bar, 0);

#pragma unroll 2
  for (int cc = 0; cc < 32; ++cc) {
    const int c = cg * 32 + cc;
    const float* rec = cols + (c / kTileSupports) * TF + (c % kTileSupports) * NP * 8;
    f2 acc[2];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float4 xy = *reinterpret_cast<const float4*>(rec + p * 8);
      const float2 zz = *reinterpret_cast<const float2*>(rec + p * 8 + 4);
      const f2 vx = pk(xy.x, xy.y), vy = pk(xy.z, xy.w), vz = pk(zz.x, zz.y);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const f2 t = term_pair<KIND>(ux[h][p], uy[h][p], uz[h][p], vx, vy, vz);
        acc[h] = p == 0 ? t : add2(acc[h], t);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float ks = pair_sum(acc[h]);
      Ks[(r + 64 * h) * kGS + c] = m_pow2 ? ks * inv_m : __fdiv_rn(ks, (float)M);
    }
  }
  __syncthreads();

  // coalesced stores: tile (bi, bj) row by row, then its transpose as (bj, bi)
  const int lane = tid & 31, warp = tid >> 5;
  for (int rr = warp; rr < kGB; rr += kGT / 32) {
    const int64_t i = i0 + rr;
    if (i >= n) break;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = lane + 32 * q;
      if (j0 + c < n) K[i * ldk + j0 + c] = Ks[rr * kGS + c];
    }
  }
  if (bi != bj) {
    for (int c = warp; c < kGB; c += kGT / 32) {
      const int64_t j = j0 + c;
      if (j >= n) break;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = lane + 32 * q;
        if (i0 + rr < n) K[j * ldk + i0 + rr] = Ks[rr * kGS + c];
      }
    }
  }
}

template <int MP, int KIND>
static cudaError_t run_gram(const float* packed, int64_t n, int M, float* K, int64_t ldk, cudaStream_t st) {
  const size_t smem = 128 + 2 * tile_bytes(MP) + (size_t)kGB * kGS * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gram_kernel<MP, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t nb = (n + kGB - 1) / kGB;
  const int64_t tiles = nb * (nb + 1) / 2;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  const int m_pow2 = (M & (M - 1)) == 0;
  gram_kernel<MP, KIND><<<(unsigned)tiles, kGT, smem, st>>>(packed, n, M, m_pow2, 1.0f / (float)M, K, ldk);
  g_launches.fetch_add(1);
  return cudaGetLastError();
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
