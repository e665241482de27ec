// train.cu — K5, Algorithm 1 "Fastron Model Update Algorithm" (PAPER.md:206-252,
// Eq. 6-9) as ONE persistent kernel: no host round trip per iteration.
//
// A thread-block cluster of C CTAs (C = 1..16, 512 threads each) owns the training
// state on chip. Thread t of CTA r owns the EPT slots j = k*512 + t (k < EPT) of the
// CTA's slice [r*chunk, r*chunk + len). The margins are kept signed by the label,
// G = y F, in registers; Y = y alpha (>= 0 by the constraint
// y_i alpha_i >= 0) lives in shared memory and is only touched by its
// owner thread. With y = +-1 every operation is exactly the oracle's on F and alpha
// with the sign moved (IEEE rounding is sign-symmetric): y fl(F + fl(d K)) =
// fl(G + y fl(d K)), y fl(F - alpha) = fl(G - Y), y fl(b y - F) = fl(b - G).
//
// One iteration (the common "add" path):
//   1. issue all EPT loads of the needed row of K (= column i, K symmetric) at once
//      (one L2 round trip; the evict-last hint keeps K resident in L2);
//   2. apply the pending rank-one update G_j += y_j fl(delta K_ij) (Eq. 8) and track the
//      thread's min of G (two interleaved chains; lowest index on ties, R9);
//   3. warp REDUX on order-preserving integer keys -> the owning lane writes the warp
//      candidate with Y and y of the winner -> __syncthreads -> warp 0 reduces the warp
//      candidates (with C > 1: CTA candidates exchanged through DSMEM behind one
//      cluster barrier) and takes the decision of Alg. 1 -> __syncthreads.
// The redundant-support scan argmax_{alpha != 0} y (F - alpha) is only
// needed when the add branch does not `continue` (min margin > 0, or the S_max gate
// blocks the add); it runs as a second pass in exactly those iterations.
// count(alpha != 0) for the S_max gate is maintained from the decisions.
// All alpha/F arithmetic is separately rounded fp64 multiply and add, matching the oracle
// compiled with -ffp-contract=off, so traces are bit-identical on the same K
// (R13). removeNonsupportPoints is an ordered compaction.
#include <cooperative_groups.h>

#include <cstdlib>

#include "fastron_device.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace fastron {

constexpr int kTrainNT = 512;
constexpr int kTrainWarps = kTrainNT / 32;
constexpr int kMaxCluster = 16;
constexpr int kMaxEPT = 12;                                 // slots per thread in registers
constexpr int64_t kChunkMax = (int64_t)kTrainNT * kMaxEPT;  // 6144 slots per CTA
constexpr int kNone = 0x7fffffff;

enum { ACT_STOP = 0, ACT_ADD = 1, ACT_REMOVE = 2, ACT_CHECK_REMOVAL = 3 };

struct TrainResultDev {
  int64_t iterations, n_add, n_remove;
  int32_t converged, n_support;
};

struct Cand {    // a (key, index) winner with its payload
  uint64_t key;  // order-preserving bits of the value (-0 == +0)
  double G;      // y F at the winner (min pass)
  double Y;      // y alpha at the winner
  int32_t idx;   // kNone if empty
  int32_t y;     // label at the winner
};

struct Decision {
  int32_t action;
  int32_t idx;    // row of the rank-one update = slot whose Y changes
  double delta;   // Eq. 6 (or -alpha_i for a removal)
  double newY;    // y_i alpha_i after the step
  int64_t nnz;    // count(alpha != 0) after the step
  int32_t converged;
  int32_t pad;
};

struct TrainArgs {
  const float* K;
  int64_t n, ldk;
  const int8_t* y;
  double beta;
  int64_t iter_max, s_max;
  double* alpha;
  double* F;
  int32_t* support_idx;
  int32_t* trace;
  TrainResultDev* result;
  int64_t chunk;
};

__device__ __forceinline__ Cand cand_none(bool for_max) { return Cand{for_max ? 0ull : ~0ull, 0.0, 0.0, kNone, 1}; }

// Monotone map double -> uint64 (a < b  <=>  key(a) < key(b) for non-NaN; -0 == +0).
__device__ __forceinline__ uint64_t order_key(double x) {
  const uint64_t u = (uint64_t)__double_as_longlong(x + 0.0);  // -0 + 0 = +0
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

// Warp-wide lexicographic best over (key, idx): minimum key (MAX_KEY: maximum key), then
// minimum idx, with integer REDUX. Returns the lane holding the winner (-1: all empty).
template <bool MAX_KEY>
__device__ __forceinline__ int warp_argbest(uint64_t key, int idx, uint64_t& bkey, int& bidx) {
  const unsigned full = 0xffffffffu;
  const bool live = idx != kNone;
  const uint32_t h = (uint32_t)(key >> 32), l = (uint32_t)key;
  uint32_t bh, bl;
  if (MAX_KEY) {
    bh = __reduce_max_sync(full, live ? h : 0u);
    bl = __reduce_max_sync(full, (live && h == bh) ? l : 0u);
  } else {
    bh = __reduce_min_sync(full, live ? h : 0xffffffffu);
    bl = __reduce_min_sync(full, (live && h == bh) ? l : 0xffffffffu);
  }
  const bool eq = live && h == bh && l == bl;
  bidx = (int)__reduce_min_sync(full, eq ? (unsigned)idx : (unsigned)kNone);
  bkey = ((uint64_t)bh << 32) | bl;
  const unsigned own = __ballot_sync(full, eq && idx == bidx);
  return own ? __ffs(own) - 1 : -1;
}

// Reduce a warp's worth of candidates (one per lane) to the lexicographic best, with its payload.
template <bool MAX_KEY>
__device__ __forceinline__ Cand warp_best(const Cand& c) {
  Cand b;
  const int bl = warp_argbest<MAX_KEY>(c.key, c.idx, b.key, b.idx);
  const int src = bl < 0 ? 0 : bl;
  b.G = __shfl_sync(0xffffffffu, c.G, src);
  b.Y = __shfl_sync(0xffffffffu, c.Y, src);
  b.y = __shfl_sync(0xffffffffu, c.y, src);
  return b;
}

__device__ __forceinline__ float ld_evict_last(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// Alg. 1's branch on the min candidate.
__device__ __forceinline__ Decision decide_min(const Cand& b, int64_t iters, int64_t nnz, const TrainArgs& A) {
  Decision d = {};
  const bool has = b.idx != kNone;
  const double m = has ? key_value(b.key) : INFINITY;
  d.nnz = nnz;
  if (iters >= A.iter_max || !has) {
    d.action = ACT_STOP;
    d.converged = has && m > 0.0;
  } else if (m <= 0.0 && (nnz < A.s_max || b.Y != 0.0)) {
    d.action = ACT_ADD;
    const double beta_i = b.y > 0 ? A.beta : 1.0;   // b_i = beta^(0.5 (y_i + 1))
    const double sdelta = __dsub_rn(beta_i, b.G);   // y_i delta, delta = b_i y_i - F_i (Eq. 6)
    d.idx = b.idx;
    d.delta = b.y > 0 ? sdelta : -sdelta;
    d.newY = __dadd_rn(b.Y, sdelta);                 // y_i (alpha_i + delta) (Eq. 7)
    d.nnz = nnz + (b.Y == 0.0 && d.newY != 0.0) - (b.Y != 0.0 && d.newY == 0.0);
  } else {
    d.action = ACT_CHECK_REMOVAL;
    d.converged = m > 0.0;
  }
  return d;
}

// Alg. 1's redundant-support branch.
__device__ __forceinline__ Decision decide_removal(Decision d, const Cand& b) {
  if (b.idx != kNone && key_value(b.key) > 0.0) {
    d.action = ACT_REMOVE;
    d.idx = b.idx;
    d.delta = b.y > 0 ? -b.Y : b.Y;  // -alpha_i = -y_i (y_i alpha_i)
    d.newY = 0.0;
    d.nnz = d.nnz - 1;
  } else {
    d.action = ACT_STOP;
  }
  return d;
}

template <int EPT>
__global__ void __launch_bounds__(kTrainNT, 1) train_kernel(const __grid_constant__ TrainArgs A) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_Y = reinterpret_cast<double*>(smem_raw);  // [chunk], owner-thread access only
  __shared__ Cand s_warp[2][kTrainWarps];
  __shared__ Cand s_cta[2];
  __shared__ int32_t s_cta_cnt[2];
  __shared__ Decision s_dec[2];
  __shared__ int32_t s_cnt[kTrainWarps];

  const int lo = rank * (int)A.chunk;
  const int hi = (int)min(A.n, (int64_t)lo + A.chunk);
  const int len = max(hi - lo, 0);
  const int jlast = max(len - 1, 0);

  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));

  // ---- load state; dead slots hold G = +inf (never the argmin) ----
  double G[EPT];
  uint32_t yneg = 0;  // bit k: y of slot k is -1 (C_free)
  int cnt0 = 0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int j = k * kTrainNT + tid;
    const bool live = j < len;
    const bool neg = live && A.y[lo + j] < 0;
    const double f = live ? A.F[lo + j] : INFINITY;
    const double a = live ? A.alpha[lo + j] : 0.0;
    G[k] = neg ? -f : f;
    if (live) s_Y[j] = neg ? -a : a;
    if (neg) yneg |= 1u << k;
    cnt0 += (live && a != 0.0);
  }
  // initial count(alpha != 0) over the cluster
  {
    const int wsum = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt0);
    if (lane == 0) s_cnt[warp] = wsum;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < kTrainWarps; ++w) t += s_cnt[w];
      s_cta_cnt[0] = t;
    }
    cluster.sync();
  }
  int64_t nnz = 0;
  for (int r = 0; r < C; ++r) nnz += *cluster.map_shared_rank(&s_cta_cnt[0], r);

  // loop invariants: clamped K-row offsets of the slots and the label sign bit of each
  // slot as an fp64 high-word mask (y_j fl(d K) is fl(d K) with its sign flipped)
  int koff[EPT];
  uint32_t sgn[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    koff[k] = min(k * kTrainNT + tid, jlast);
    sgn[k] = ((yneg >> k) & 1u) << 31;
  }

  int64_t iters = 0, n_add = 0, n_remove = 0;
  int upd_i = -1;  // row of the pending rank-one update of F
  double upd_delta = 0.0;
  int parity = 0;
  int converged = 0;

  for (;;) {
    // ---- 1. all loads of the pending K row, then the fused update + min scan ----
    float kr[EPT];
    const bool have_upd = upd_i >= 0;
    if (have_upd) {
      const float* Krow = A.K + (int64_t)upd_i * A.ldk + lo;
#pragma unroll
      for (int k = 0; k < EPT; ++k) kr[k] = ld_evict_last(Krow + koff[k], pol);
    }
    double m0 = INFINITY, m1 = INFINITY;  // two interleaved chains (even / odd k)
    int k0 = -1, k1 = -1;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      if (have_upd) {
        const double p = __dmul_rn(upd_delta, (double)kr[k]);
        const double sp = __hiloint2double(__double2hiint(p) ^ (int)sgn[k], __double2loint(p));  // y_j p
        G[k] = __dadd_rn(G[k], sp);  // Eq. 8, signed
      }
      if (k & 1) {
        if (G[k] < m1) { m1 = G[k]; k1 = k; }
      } else {
        if (G[k] < m0) { m0 = G[k]; k0 = k; }
      }
    }
    // merge (slot order == index order inside a thread; the lower slot wins ties)
    double mk = m0;
    int mkk = k0;
    if (m1 < m0 || (m1 == m0 && k1 >= 0 && k1 < k0)) { mk = m1; mkk = k1; }
    const int my_idx = (mkk >= 0 && mk != INFINITY) ? lo + mkk * kTrainNT + tid : kNone;
    {
      uint64_t wkey;
      int widx;
      const int wl = warp_argbest<false>(order_key(mk), my_idx, wkey, widx);
      if (lane == wl) {  // the owner lane attaches the payload of the warp winner
        s_warp[parity][warp] = Cand{wkey, mk, s_Y[mkk * kTrainNT + tid], widx, ((yneg >> mkk) & 1u) ? -1 : 1};
      } else if (wl < 0 && lane == 0) {
        s_warp[parity][warp] = cand_none(false);
      }
    }
    __syncthreads();

    // ---- 2. warp 0: CTA (and cluster) reduction + the decision of Algorithm 1 ----
    if (warp == 0) {
      const Cand best = warp_best<false>(lane < kTrainWarps ? s_warp[parity][lane] : cand_none(false));
      if (C == 1) {
        if (lane == 0) s_dec[parity] = decide_min(best, iters, nnz, A);
      } else if (lane == 0) {
        s_cta[parity] = best;
      }
    }
    if (C > 1) {
      cluster.sync();
      if (warp == 0) {
        const Cand best = warp_best<false>(lane < C ? *cluster.map_shared_rank(&s_cta[parity], lane) : cand_none(false));
        if (lane == 0) s_dec[parity] = decide_min(best, iters, nnz, A);
      }
    }
    __syncthreads();
    Decision d = s_dec[parity];

    // ---- 3. only when the add branch does not `continue`: the removal scan ----
    if (d.action == ACT_CHECK_REMOVAL) {
      const int q = parity ^ 1;
      double rk = -INFINITY;
      int rkk = -1;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int j = k * kTrainNT + tid;
        if (j < len) {
          const double Yk = s_Y[j];
          const double r = __dsub_rn(G[k], Yk);  // y (F - alpha)
          if (Yk != 0.0 && r > rk) { rk = r; rkk = k; }
        }
      }
      const int ridx = rkk >= 0 ? lo + rkk * kTrainNT + tid : kNone;
      {
        uint64_t wkey;
        int widx;
        const int wl = warp_argbest<true>(order_key(rk), ridx, wkey, widx);
        if (lane == wl) {
          s_warp[q][warp] = Cand{wkey, 0.0, s_Y[rkk * kTrainNT + tid], widx, ((yneg >> rkk) & 1u) ? -1 : 1};
        } else if (wl < 0 && lane == 0) {
          s_warp[q][warp] = cand_none(true);
        }
      }
      __syncthreads();
      if (warp == 0) {
        const Cand best = warp_best<true>(lane < kTrainWarps ? s_warp[q][lane] : cand_none(true));
        if (C == 1) {
          if (lane == 0) s_dec[q] = decide_removal(d, best);
        } else if (lane == 0) {
          s_cta[q] = best;
        }
      }
      if (C > 1) {
        cluster.sync();
        if (warp == 0) {
          const Cand best = warp_best<true>(lane < C ? *cluster.map_shared_rank(&s_cta[q], lane) : cand_none(true));
          if (lane == 0) s_dec[q] = decide_removal(d, best);
        }
      }
      __syncthreads();
      d = s_dec[q];
      parity = q;  // buffers of parity q were used last; the loop flips back below
    }

    if (d.action == ACT_STOP) {
      converged = d.converged;
      break;
    }
    // apply the step: the owner thread updates Y_i, everyone records the pending
    // rank-one update of G for the next pass
    if (d.idx >= lo && d.idx < hi && ((d.idx - lo) % kTrainNT) == tid) s_Y[d.idx - lo] = d.newY;
    if (tid == 0 && rank == 0 && A.trace) A.trace[iters] = d.action == ACT_ADD ? d.idx : -(d.idx + 1);
    if (d.action == ACT_ADD) ++n_add;
    else ++n_remove;
    upd_i = d.idx;
    upd_delta = d.delta;
    nnz = d.nnz;
    ++iters;
    parity ^= 1;
  }

  // ---- write back (F = y G, alpha = y Y) + removeNonsupportPoints ----
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int j = k * kTrainNT + tid;
    if (j < len) {
      const bool neg = (yneg >> k) & 1u;
      const double Yk = s_Y[j];
      A.alpha[lo + j] = neg ? -Yk : Yk;
      A.F[lo + j] = neg ? -G[k] : G[k];
      cnt += Yk != 0.0;
    }
  }
  {  // per-CTA support counts -> prefix over the cluster ranks
    const int wsum = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
    __syncthreads();
    if (lane == 0) s_cnt[warp] = wsum;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < kTrainWarps; ++w) t += s_cnt[w];
      s_cta_cnt[1] = t;
    }
    cluster.sync();
  }
  int64_t offset = 0, total = 0;
  for (int r = 0; r < C; ++r) {
    const int c = *cluster.map_shared_rank(&s_cta_cnt[1], r);
    if (r < rank) offset += c;
    total += c;
  }
  if (A.support_idx) {
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int j = k * kTrainNT + tid;
      const bool flag = j < len && s_Y[j] != 0.0;
      const unsigned ballot = __ballot_sync(0xffffffffu, flag);
      __syncthreads();
      if (lane == 0) s_cnt[warp] = __popc(ballot);
      __syncthreads();
      int before = 0, slice_total = 0;
      for (int w2 = 0; w2 < kTrainWarps; ++w2) {
        if (w2 < warp) before += s_cnt[w2];
        slice_total += s_cnt[w2];
      }
      if (flag) A.support_idx[offset + before + __popc(ballot & ((1u << lane) - 1u))] = lo + j;
      offset += slice_total;
    }
  }
  if (rank == 0 && tid == 0) {
    A.result->iterations = iters;
    A.result->n_add = n_add;
    A.result->n_remove = n_remove;
    A.result->converged = converged;
    A.result->n_support = (int32_t)total;
  }
  cluster.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

int64_t train_max_n() { return kChunkMax * kMaxCluster; }

template <int EPT>
static cudaError_t launch_ept(const TrainArgs& A, int C, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(train_kernel<EPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(train_kernel<EPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kChunkMax * 8));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(kTrainNT, 1, 1);
  cfg.dynamicSmemBytes = (size_t)A.chunk * 8;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, train_kernel<EPT>, A);
}

cudaError_t launch_train(const float* K, int64_t n, int64_t ldk, const int8_t* y, double beta, int64_t iter_max,
                         int64_t s_max, double* alpha, double* F, int32_t* support_idx, int32_t* trace, void* result,
                         cudaStream_t st) {
  int C = (int)((n + kChunkMax - 1) / kChunkMax);
  if (C < 1) C = 1;
  if (const char* env = getenv("FASTRON_TRAIN_CLUSTER")) {  // tuning override (>= the minimum)
    const int c = atoi(env);
    if (c > C) C = c;
  }
  if (C > kMaxCluster) return cudaErrorInvalidValue;
  TrainArgs A;
  A.K = K;
  A.n = n;
  A.ldk = ldk;
  A.y = y;
  A.beta = beta;
  A.iter_max = iter_max;
  A.s_max = s_max;
  A.alpha = alpha;
  A.F = F;
  A.support_idx = support_idx;
  A.trace = trace;
  A.result = reinterpret_cast<TrainResultDev*>(result);
  A.chunk = (n + C - 1) / C;
  if (A.chunk < 1) A.chunk = 1;
  const int64_t ept = (A.chunk + kTrainNT - 1) / kTrainNT;
  cudaError_t e;
  if (ept <= 2) e = launch_ept<2>(A, C, st);
  else if (ept <= 4) e = launch_ept<4>(A, C, st);
  else if (ept <= 8) e = launch_ept<8>(A, C, st);
  else e = launch_ept<12>(A, C, st);
  g_launches.fetch_add(1);
  return e;
}

}  // namespace fastron
