// update.cu — the pieces of the Fastron model-update cycle around Algorithm 1
// ("two-stage active learning", and :219 loadPreviousModel):
//
//  * active_samples_kernel: stage 1 draws configurations near each support point, stage 2
//    uniformly in the joint limits. The random numbers are inputs (standard
//    normal and U[0,1) arrays), so the draw is reproducible and testable.
//  * label_capsules_kernel: the geometric collision check that labels the new samples and
//    re-labels the support points (the paper uses FCL — a comparison system —
//    here the workload's capsule-vs-box scene, R12). One thread per
//    configuration; capsules are the segments between consecutive chain points; the
//    segment-box distance is minimised exactly in fp64 (piecewise quadratic split at the
//    slab crossings). Tangency counts as collision.
//  * matvec_kernel: F = K alpha for a warm start whose alpha changed support set
//    (F must match the loaded alpha), fixed summation order.
//  * matvec_lazy_kernel: the same F = K alpha without the Gram, for the lazy Algorithm 1:
//    each K entry is computed from the packed records with the Gram's term function,
//    summation order and 1/M (so it equals K3's entry bit for bit), then accumulated in
//    matvec_kernel's fp64 order.
#include "fastron_device.cuh"
#include "internal.h"

namespace fastron {

__global__ void active_samples_kernel(const float* __restrict__ S, int64_t ns, int64_t lds, int D, int n_near,
                                      const float* __restrict__ z, const float* __restrict__ sigma,
                                      const float* __restrict__ u, int64_t n_uniform, const float* __restrict__ lo,
                                      const float* __restrict__ hi, float* __restrict__ out, int64_t ldo) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_stage1 = ns * n_near;
  if (r >= n_stage1 + n_uniform) return;
  float* o = out + r * ldo;
  if (r < n_stage1) {  // stage 1: s_i + sigma * z, clamped to the joint limits
    const float* s = S + (r / n_near) * lds;
    const float* zr = z + r * D;
    for (int d = 0; d < D; ++d) {
      const float v = __fadd_rn(s[d], __fmul_rn(sigma[d], zr[d]));
      o[d] = fminf(fmaxf(v, lo[d]), hi[d]);
    }
  } else {  // stage 2: lo + u (hi - lo)
    const float* ur = u + (r - n_stage1) * D;
    for (int d = 0; d < D; ++d) o[d] = __fadd_rn(lo[d], __fmul_rn(ur[d], __fsub_rn(hi[d], lo[d])));
  }
}

struct CapsuleScene {
  int32_t n_cubes;
  int32_t n_chain;
  int32_t chain[33];  // control-point indices of the chain; -1 = the base origin (0, 0, 0)
  float radius;
  double box[kMaxCubes][6];  // lo xyz, hi xyz
};

__device__ double seg_box_dist2(const double p0[3], const double p1[3], const double* box) {
  double dv[3], t[8];
  int nt = 0;
  t[nt++] = 0.0;
  t[nt++] = 1.0;
  for (int a = 0; a < 3; ++a) {
    dv[a] = p1[a] - p0[a];
    if (dv[a] != 0.0) {
      const double ta = (box[a] - p0[a]) / dv[a], tb = (box[3 + a] - p0[a]) / dv[a];
      if (ta > 0.0 && ta < 1.0) t[nt++] = ta;
      if (tb > 0.0 && tb < 1.0) t[nt++] = tb;
    }
  }
  for (int i = 1; i < nt; ++i) {  // insertion sort of <= 8 breakpoints
    const double v = t[i];
    int j = i - 1;
    while (j >= 0 && t[j] > v) {
      t[j + 1] = t[j];
      --j;
    }
    t[j + 1] = v;
  }
  double best = INFINITY;
  for (int k = 0; k + 1 < nt; ++k) {
    const double ta = t[k], tb = t[k + 1], tm = 0.5 * (ta + tb);
    double A = 0.0, B = 0.0, C = 0.0;
    for (int a = 0; a < 3; ++a) {
      const double pm = p0[a] + tm * dv[a];
      double bound;
      if (pm < box[a]) bound = box[a];
      else if (pm > box[3 + a]) bound = box[3 + a];
      else continue;  // inside the slab on this axis over the whole piece
      const double e = p0[a] - bound;
      A += dv[a] * dv[a];
      B += 2.0 * dv[a] * e;
      C += e * e;
    }
    double ts = A > 0.0 ? -B / (2.0 * A) : ta;
    ts = fmin(fmax(ts, ta), tb);
    const double v = fmax(A * ts * ts + B * ts + C, 0.0);
    best = fmin(best, v);
  }
  return best;
}

__global__ void label_capsules_kernel(const __grid_constant__ CapsuleScene sc, const float4* __restrict__ pos,
                                      int64_t ldp, int64_t n, int8_t* __restrict__ label) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double r2 = (double)sc.radius * (double)sc.radius;
  bool hit = false;
  double prev[3];
  for (int c = 0; c < sc.n_chain && !hit; ++c) {
    double cur[3] = {0.0, 0.0, 0.0};
    const int m = sc.chain[c];
    if (m >= 0) {
      const float4 p = pos[(int64_t)m * ldp + k];
      cur[0] = p.x; cur[1] = p.y; cur[2] = p.z;
    }
    if (c > 0) {
      for (int b = 0; b < sc.n_cubes && !hit; ++b) hit = seg_box_dist2(prev, cur, sc.box[b]) <= r2;
    }
    prev[0] = cur[0]; prev[1] = cur[1]; prev[2] = cur[2];
  }
  label[k] = hit ? 1 : -1;
}

// F_j = sum_i alpha_i K[i][j] over the nonzero alpha_i, in index order (deterministic:
// separately rounded multiply and add, the oracle's order). A warm start's alpha is sparse
// (the previous support set), and a plain loop over i is one dependent DRAM round trip per
// nonzero row (8,446 points, 2,482 nonzero: 0.95 ms). Here the CTA first compacts the next
// nonzero indices, in order, into shared memory (ballot + prefix per 128-index chunk), then
// every thread walks that list with kMvUnroll row loads in flight and adds them in list
// order — the same operations in the same order, so the same bits.
constexpr int kMvNT = 128;
constexpr int kMvSeg = 2048;    // nonzero entries per shared-memory segment
constexpr int kMvUnroll = 16;   // K loads in flight per thread
__global__ void __launch_bounds__(kMvNT) matvec_kernel(const float* __restrict__ K, int64_t n, int64_t ldk,
                                                       const double* __restrict__ alpha, double* __restrict__ F) {
  __shared__ int32_t s_idx[kMvSeg];
  __shared__ double s_a[kMvSeg];
  __shared__ int s_wcnt[kMvNT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j = (int64_t)blockIdx.x * kMvNT + tid;
  const bool live = j < n;
  const float* Kj = K + (live ? j : 0);
  double f = 0.0;
  int64_t base = 0;  // next index of alpha to scan (uniform)
  while (base < n) {
    int cnt = 0;  // entries in the segment (uniform)
    while (base < n && cnt + kMvNT <= kMvSeg) {
      const int64_t i = base + tid;
      const double a = i < n ? alpha[i] : 0.0;
      const bool nz = a != 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, nz);
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      int ofs = cnt, total = 0;
#pragma unroll
      for (int w = 0; w < kMvNT / 32; ++w) {
        if (w < warp) ofs += s_wcnt[w];
        total += s_wcnt[w];
      }
      if (nz) {
        const int at = ofs + __popc(bal & ((1u << lane) - 1u));
        s_idx[at] = (int32_t)i;
        s_a[at] = a;
      }
      cnt += total;
      base += kMvNT;
      __syncthreads();
    }
    if (live) {
      for (int t = 0; t < cnt; t += kMvUnroll) {
        float kv[kMvUnroll];
#pragma unroll
        for (int k = 0; k < kMvUnroll; ++k) kv[k] = t + k < cnt ? __ldg(Kj + (int64_t)s_idx[t + k] * ldk) : 0.0f;
#pragma unroll
        for (int k = 0; k < kMvUnroll; ++k)
          if (t + k < cnt) f = __dadd_rn(f, __dmul_rn(s_a[t + k], (double)kv[k]));
      }
    }
    __syncthreads();  // the segment is consumed before it is refilled
  }
  if (live) F[j] = f;
}

template <int MP, int KIND>
__global__ void __launch_bounds__(128) matvec_lazy_kernel(const float* __restrict__ packed, int64_t n, int M,
                                                          int m_pow2, float inv_m, const double* __restrict__ alpha,
                                                          double* __restrict__ F) {
  constexpr int NP = MP / 2;
  constexpr int64_t TF = tile_floats(MP);
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  // column j in registers, its padded point (odd M) at 0 as on K3's column side
  f2 ux[NP], uy[NP], uz[NP];
  const float* rj = packed + (j / kTileSupports) * TF + (j % kTileSupports) * NP * 8;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float4 xy = __ldg(reinterpret_cast<const float4*>(rj + p * 8));
    const float2 zz = __ldg(reinterpret_cast<const float2*>(rj + p * 8 + 4));
    ux[p] = pk(xy.x, xy.y);
    uy[p] = pk(xy.z, xy.w);
    uz[p] = pk(zz.x, zz.y);
  }
  if (M < MP) {
    ux[NP - 1] = pk(lo(ux[NP - 1]), 0.0f);
    uy[NP - 1] = pk(lo(uy[NP - 1]), 0.0f);
    uz[NP - 1] = pk(lo(uz[NP - 1]), 0.0f);
  }
  double f = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double a = __ldg(alpha + i);  // uniform across the CTA
    if (a == 0.0) continue;
    const float* ri = packed + (i / kTileSupports) * TF + (i % kTileSupports) * NP * 8;
    f2 acc;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float4 xy = __ldg(reinterpret_cast<const float4*>(ri + p * 8));
      const float2 zz = __ldg(reinterpret_cast<const float2*>(ri + p * 8 + 4));
      accum_term<KIND>(acc, sub2(ux[p], pk(xy.x, xy.y)), sub2(uy[p], pk(xy.z, xy.w)), sub2(uz[p], pk(zz.x, zz.y)),
                       p == 0);
    }
    const float ks = pair_sum(acc);
    const float v = m_pow2 ? ks * inv_m : __fdiv_rn(ks, (float)M);
    f = __dadd_rn(f, __dmul_rn(a, (double)v));
  }
  F[j] = f;
}

cudaError_t launch_matvec_lazy(const float* packed, int64_t n, int M, int kind, const double* alpha, double* F,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int m_pow2 = (M & (M - 1)) == 0;
  const float inv_m = 1.0f / (float)M;
  const unsigned grid = (unsigned)((n + 127) / 128);
  switch (padded_m(M)) {
#define FASTRON_MVCASE(mp)                                                                                      \
  case mp:                                                                                                      \
    if (kind == kGaussian)                                                                                      \
      matvec_lazy_kernel<mp, kGaussian><<<grid, 128, 0, st>>>(packed, n, M, m_pow2, inv_m, alpha, F);           \
    else                                                                                                        \
      matvec_lazy_kernel<mp, kRQ><<<grid, 128, 0, st>>>(packed, n, M, m_pow2, inv_m, alpha, F);                 \
    break;
    FASTRON_MVCASE(2)
    FASTRON_MVCASE(4)
    FASTRON_MVCASE(6)
    FASTRON_MVCASE(8)
    FASTRON_MVCASE(10)
    FASTRON_MVCASE(12)
    FASTRON_MVCASE(14)
    FASTRON_MVCASE(16)
    FASTRON_MVCASE(18)
    FASTRON_MVCASE(20)
    FASTRON_MVCASE(22)
    FASTRON_MVCASE(24)
    FASTRON_MVCASE(26)
    FASTRON_MVCASE(28)
    FASTRON_MVCASE(30)
    FASTRON_MVCASE(32)
#undef FASTRON_MVCASE
    default:
      return cudaErrorInvalidValue;
  }
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_active_samples(const float* S, int64_t ns, int64_t lds, int D, int n_near, const float* z,
                                  const float* sigma, const float* u, int64_t n_uniform, const float* lo,
                                  const float* hi, float* out, int64_t ldo, cudaStream_t st) {
  const int64_t total = ns * n_near + n_uniform;
  if (total <= 0) return cudaSuccess;
  active_samples_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(S, ns, lds, D, n_near, z, sigma, u, n_uniform,
                                                                          lo, hi, out, ldo);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_label_capsules(const float4* pos, int64_t ldp, int64_t n, const int32_t* chain, int n_chain,
                                  const double* boxes, int n_cubes, float radius, int8_t* label, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n_chain > 33 || n_cubes > kMaxCubes) return cudaErrorInvalidValue;
  CapsuleScene sc = {};
  sc.n_cubes = n_cubes;
  sc.n_chain = n_chain;
  for (int c = 0; c < n_chain; ++c) sc.chain[c] = chain[c];
  sc.radius = radius;
  for (int b = 0; b < n_cubes; ++b)
    for (int c = 0; c < 6; ++c) sc.box[b][c] = boxes[6 * b + c];
  label_capsules_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(sc, pos, ldp, n, label);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_matvec(const float* K, int64_t n, int64_t ldk, const double* alpha, double* F, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  matvec_kernel<<<(unsigned)((n + kMvNT - 1) / kMvNT), kMvNT, 0, st>>>(K, n, ldk, alpha, F);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace fastron
