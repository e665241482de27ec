// train.cu — K5, Algorithm 1 "Fastron Model Update Algorithm" (PAPER.md:206-252,
// Eq. 6-9) as ONE persistent kernel: no host round trip per iteration.
//
// A thread-block cluster of C CTAs (C = 1..16) owns the training state on chip: CTA r
// holds the slice [r*chunk, (r+1)*chunk) of alpha (fp64), F (fp64) and y (int8) in
// shared memory. One iteration is one fused pass over each slice:
//   1. apply the previous step's rank-one update F_j += delta * K[i][j] (Eq. 8; a
//      removal is delta = -alpha_i) reading row i of K (= column i, K
//      symmetric) from L2/HBM, and in the same pass
//   2. scan for argmin_j y_j F_j (Eq. 9, misclassification test PAPER.md:223) and for
//      argmax_{alpha_j != 0} y_j (F_j - alpha_j) (redundant-support test PAPER.md:235),
//      lowest index on ties (R9), and count(alpha != 0) for the S_max gate (:227);
//   3. reduce per CTA (warp shuffles), exchange one candidate record per CTA through
//      distributed shared memory behind a single cluster barrier (double-buffered by
//      iteration parity), and let every CTA take the same decision.
// alpha/F arithmetic uses separately rounded fp64 multiply and add (__dmul_rn /
// __dadd_rn), matching the oracle compiled with -ffp-contract=off, so traces are
// bit-identical on the same K (R13). removeNonsupportPoints
// is an ordered compaction of the alpha != 0 indices.
#include <cooperative_groups.h>

#include "fastron_device.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace fastron {

constexpr int kTrainNT = 1024;
constexpr int kTrainWarps = kTrainNT / 32;
constexpr int kMaxCluster = 16;
constexpr int64_t kChunkMax = 12288;  // elements per CTA: 12288 * 17 B = 204 KB of shared memory

struct TrainResultDev {
  int64_t iterations, n_add, n_remove;
  int32_t converged, n_support;
};

struct Cand {
  double mkey;    // min y F over the slice
  double mF;      // F at the argmin
  double malpha;  // alpha at the argmin
  double rkey;    // max y (F - alpha) over alpha != 0
  double ralpha;  // alpha at the argmax
  int32_t midx;
  int32_t ridx;   // -1 if no alpha != 0 in the slice
  int32_t nnz;
  int32_t my;     // y at the argmin
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

__device__ __forceinline__ bool min_better(double k, int i, double bk, int bi) {
  return k < bk || (k == bk && i < bi);
}
__device__ __forceinline__ bool max_better(double k, int i, double bk, int bi) {
  return k > bk || (k == bk && i < bi);
}

__global__ void __launch_bounds__(kTrainNT, 1) train_kernel(const __grid_constant__ TrainArgs A) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_alpha = reinterpret_cast<double*>(smem_raw);
  double* s_F = s_alpha + A.chunk;
  int8_t* s_y = reinterpret_cast<int8_t*>(s_F + A.chunk);
  __shared__ Cand s_cand[2];
  __shared__ Cand s_warp[kTrainWarps];
  __shared__ Cand s_dec;
  __shared__ int32_t s_flags[2];  // [0] = action (0 stop, 1 add, 2 remove), [1] = converged
  __shared__ int32_t s_scan[kTrainWarps];

  const int64_t lo = (int64_t)rank * A.chunk;
  const int64_t hi = min(A.n, lo + A.chunk);
  const int64_t len = max(hi - lo, (int64_t)0);

  for (int64_t j = tid; j < len; j += kTrainNT) {
    s_alpha[j] = A.alpha[lo + j];
    s_F[j] = A.F[lo + j];
    s_y[j] = A.y[lo + j];
  }
  __syncthreads();

  int64_t iters = 0, n_add = 0, n_remove = 0;
  int64_t upd_i = -1;
  double upd_delta = 0.0;
  int parity = 0;
  int converged = 0;

  for (;;) {
    // ---- fused rank-one update + scan of the slice ----
    double mk = INFINITY, mF = 0.0, ma = 0.0, rk = -INFINITY, ra = 0.0;
    int mi = 0x7fffffff, ri = 0x7fffffff, nnz = 0, my = 1;
    const float* Krow = upd_i >= 0 ? A.K + upd_i * A.ldk + lo : nullptr;
    for (int64_t j = tid; j < len; j += kTrainNT) {
      double F = s_F[j];
      if (Krow) {
        F = __dadd_rn(F, __dmul_rn(upd_delta, (double)__ldg(Krow + j)));
        s_F[j] = F;
      }
      const double yj = (double)s_y[j];
      const double a = s_alpha[j];
      const double m = __dmul_rn(yj, F);
      const int idx = (int)(lo + j);
      if (min_better(m, idx, mk, mi)) { mk = m; mi = idx; mF = F; ma = a; my = (int)s_y[j]; }
      if (a != 0.0) {
        ++nnz;
        const double r = __dmul_rn(yj, __dsub_rn(F, a));
        if (max_better(r, idx, rk, ri)) { rk = r; ri = idx; ra = a; }
      }
    }
    // warp reduction
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double omk = __shfl_down_sync(0xffffffffu, mk, off), omF = __shfl_down_sync(0xffffffffu, mF, off);
      const double oma = __shfl_down_sync(0xffffffffu, ma, off);
      const int omi = __shfl_down_sync(0xffffffffu, mi, off), omy = __shfl_down_sync(0xffffffffu, my, off);
      const double ork = __shfl_down_sync(0xffffffffu, rk, off), ora = __shfl_down_sync(0xffffffffu, ra, off);
      const int ori = __shfl_down_sync(0xffffffffu, ri, off);
      nnz += __shfl_down_sync(0xffffffffu, nnz, off);
      if (min_better(omk, omi, mk, mi)) { mk = omk; mi = omi; mF = omF; ma = oma; my = omy; }
      if (max_better(ork, ori, rk, ri)) { rk = ork; ri = ori; ra = ora; }
    }
    if (lane == 0) s_warp[warp] = Cand{mk, mF, ma, rk, ra, mi, ri, nnz, my};
    __syncthreads();
    if (warp == 0) {
      Cand c = s_warp[lane];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        Cand o;
        o.mkey = __shfl_down_sync(0xffffffffu, c.mkey, off);
        o.mF = __shfl_down_sync(0xffffffffu, c.mF, off);
        o.malpha = __shfl_down_sync(0xffffffffu, c.malpha, off);
        o.midx = __shfl_down_sync(0xffffffffu, c.midx, off);
        o.my = __shfl_down_sync(0xffffffffu, c.my, off);
        o.rkey = __shfl_down_sync(0xffffffffu, c.rkey, off);
        o.ralpha = __shfl_down_sync(0xffffffffu, c.ralpha, off);
        o.ridx = __shfl_down_sync(0xffffffffu, c.ridx, off);
        o.nnz = __shfl_down_sync(0xffffffffu, c.nnz, off);
        c.nnz += o.nnz;
        if (min_better(o.mkey, o.midx, c.mkey, c.midx)) { c.mkey = o.mkey; c.midx = o.midx; c.mF = o.mF; c.malpha = o.malpha; c.my = o.my; }
        if (max_better(o.rkey, o.ridx, c.rkey, c.ridx)) { c.rkey = o.rkey; c.ridx = o.ridx; c.ralpha = o.ralpha; }
      }
      if (lane == 0) s_cand[parity] = c;
    }
    // ---- exchange across the cluster (one barrier per iteration) ----
    cluster.sync();
    if (warp == 0) {
      Cand c;
      c.mkey = INFINITY; c.rkey = -INFINITY; c.midx = 0x7fffffff; c.ridx = 0x7fffffff; c.nnz = 0;
      c.mF = c.malpha = c.ralpha = 0.0; c.my = 1;
      if (lane < C) c = *cluster.map_shared_rank(&s_cand[parity], lane);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        Cand o;
        o.mkey = __shfl_down_sync(0xffffffffu, c.mkey, off);
        o.mF = __shfl_down_sync(0xffffffffu, c.mF, off);
        o.malpha = __shfl_down_sync(0xffffffffu, c.malpha, off);
        o.midx = __shfl_down_sync(0xffffffffu, c.midx, off);
        o.my = __shfl_down_sync(0xffffffffu, c.my, off);
        o.rkey = __shfl_down_sync(0xffffffffu, c.rkey, off);
        o.ralpha = __shfl_down_sync(0xffffffffu, c.ralpha, off);
        o.ridx = __shfl_down_sync(0xffffffffu, c.ridx, off);
        o.nnz = __shfl_down_sync(0xffffffffu, c.nnz, off);
        c.nnz += o.nnz;
        if (min_better(o.mkey, o.midx, c.mkey, c.midx)) { c.mkey = o.mkey; c.midx = o.midx; c.mF = o.mF; c.malpha = o.malpha; c.my = o.my; }
        if (max_better(o.rkey, o.ridx, c.rkey, c.ridx)) { c.rkey = o.rkey; c.ridx = o.ridx; c.ralpha = o.ralpha; }
      }
      if (lane == 0) {
        int action = 0;
        int conv = 0;
        if (iters >= A.iter_max) {
          conv = (A.n > 0 && c.mkey > 0.0);
        } else if (c.mkey <= 0.0 && ((int64_t)c.nnz < A.s_max || c.malpha != 0.0)) {
          action = 1;  // add / adjust (Eq. 6-8)
        } else if (c.ridx != 0x7fffffff && c.rkey > 0.0) {
          action = 2;  // remove a redundant support point
        } else {
          conv = (A.n > 0 && c.mkey > 0.0);
        }
        s_dec = c;
        s_flags[0] = action;
        s_flags[1] = conv;
      }
    }
    __syncthreads();
    const int action = s_flags[0];
    if (action == 0) {
      converged = s_flags[1];
      break;
    }
    const Cand d = s_dec;
    if (action == 1) {
      const double b = d.my > 0 ? A.beta : 1.0;  // b_i = beta^(0.5 (y_i + 1))
      const double delta = __dsub_rn(__dmul_rn(b, (double)d.my), d.mF);
      upd_i = d.midx;
      upd_delta = delta;
      if (tid == 0 && d.midx >= lo && d.midx < hi) s_alpha[d.midx - lo] = __dadd_rn(d.malpha, delta);
      if (tid == 0 && rank == 0 && A.trace) A.trace[iters] = d.midx;
      ++n_add;
    } else {
      upd_i = d.ridx;
      upd_delta = -d.ralpha;
      if (tid == 0 && d.ridx >= lo && d.ridx < hi) s_alpha[d.ridx - lo] = 0.0;
      if (tid == 0 && rank == 0 && A.trace) A.trace[iters] = -(d.ridx + 1);
      ++n_remove;
    }
    ++iters;
    parity ^= 1;
    // s_alpha write by tid 0 is read in the next scan by its owner thread
    __syncthreads();
  }

  // ---- write back + removeNonsupportPoints (ordered compaction) ----
  for (int64_t j = tid; j < len; j += kTrainNT) {
    A.alpha[lo + j] = s_alpha[j];
    A.F[lo + j] = s_F[j];
  }
  // slice nnz of every rank lives in s_cand[parity] of that rank (published this iteration)
  int64_t offset = 0;
  int64_t total = 0;
  for (int r = 0; r < C; ++r) {
    const int cnt = cluster.map_shared_rank(&s_cand[parity], r)->nnz;
    if (r < rank) offset += cnt;
    total += cnt;
  }
  if (A.support_idx) {
    for (int64_t base = 0; base < len; base += kTrainNT) {
      const int64_t j = base + tid;
      const bool flag = j < len && s_alpha[j] != 0.0;
      const unsigned ballot = __ballot_sync(0xffffffffu, flag);
      if (lane == 0) s_scan[warp] = __popc(ballot);
      __syncthreads();
      int before = 0, chunk_total = 0;
      for (int w = 0; w < kTrainWarps; ++w) {
        if (w < warp) before += s_scan[w];
        chunk_total += s_scan[w];
      }
      if (flag) A.support_idx[offset + before + __popc(ballot & ((1u << lane) - 1u))] = (int32_t)(lo + j);
      offset += chunk_total;
      __syncthreads();
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

cudaError_t launch_train(const float* K, int64_t n, int64_t ldk, const int8_t* y, double beta, int64_t iter_max,
                         int64_t s_max, double* alpha, double* F, int32_t* support_idx, int32_t* trace, void* result,
                         cudaStream_t st) {
  int C = (int)((n + kChunkMax - 1) / kChunkMax);
  if (C < 1) C = 1;
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
  const size_t smem = (size_t)A.chunk * 17 + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kChunkMax * 17 + 16));
    cudaFuncSetAttribute(train_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(kTrainNT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, train_kernel, A);
  g_launches.fetch_add(1);
  return e;
}

}  // namespace fastron
