// train.cu — K5, Algorithm 1 "Fastron Model Update Algorithm" (PAPER.md:206-252,
// Eq. 6-9) as ONE persistent kernel: no host round trip per iteration.
//
// A thread-block cluster of C CTAs (C = 1..16, 256 threads each) owns the training
// state on chip. Thread t of CTA r owns the EPT slots j = k*256 + t (k < EPT) of the
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
//      candidate with Y and y of the winner -> __syncthreads -> every warp reduces the
//      warp candidates and takes the (identical) decision of Alg. 1 itself, so no second
//      barrier is needed. With C > 1, warp 0 first sends the CTA winner into every CTA's
//      inbox (st.async into DSMEM, completing bytes on the receiver's mbarrier) and all
//      warps wait on their own inbox barrier before reducing the C CTA winners.
// The redundant-support scan argmax_{alpha != 0} y (F - alpha) is only
// needed when the add branch does not `continue` (min margin > 0, or the S_max gate
// blocks the add); it runs as a second pass in exactly those iterations.
// count(alpha != 0) for the S_max gate is maintained from the decisions.
// All alpha/F arithmetic is separately rounded fp64 multiply and add, matching the oracle
// compiled with -ffp-contract=off, so traces are bit-identical on the same K
// (R13). removeNonsupportPoints is an ordered compaction.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "fastron_device.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace fastron {

#ifndef FASTRON_TRAIN_NT
#define FASTRON_TRAIN_NT 256
#endif
constexpr int kTrainNT = FASTRON_TRAIN_NT;
constexpr int kTrainWarps = kTrainNT / 32;
constexpr int kMaxCluster = 16;
constexpr int kMaxEPT = 6144 / kTrainNT;                    // slots per thread in registers
constexpr int64_t kChunkMax = (int64_t)kTrainNT * kMaxEPT;  // 6144 slots per CTA
constexpr int kNone = 0x7fffffff;

enum { ACT_STOP = 0, ACT_ADD = 1, ACT_REMOVE = 2, ACT_CHECK_REMOVAL = 3 };

struct TrainResultDev {
  int64_t iterations, n_add, n_remove;
  int32_t converged, n_support;
};

struct WCand {    // a warp winner: the key, its index and label (16 bytes, one STS.128)
  uint64_t key;   // order-preserving bits of the value (-0 == +0); y F = key_value(key)
  int32_t idx;    // kNone if empty
  int32_t y;      // label at the winner
};

struct __align__(16) Cand {  // a CTA winner with its payload (32 bytes: an inbox entry, two 16-byte DSMEM stores)
  uint64_t key;
  double Y;       // y alpha at the winner
  int32_t idx;    // kNone if empty
  int32_t y;
  int32_t slot;   // lazy mode: column-cache slot of the winner's K column (-1: not cached)
  int32_t pad;
};

struct Decision {
  int32_t action;
  int32_t idx;    // row of the rank-one update = slot whose Y changes
  int32_t slot;      // lazy mode: cache slot holding column idx (-1: compute it)
  int32_t new_slot;  // lazy mode: cache slot to store the computed column in (-1: none)
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
  // lazy-column mode: K columns computed on demand and cached
  const float* packed;   // pre-scaled training points in the scoring tile layout
  float* cache;          // [cache_cols][n]
  f2* gpts;              // GPTS instances: the point planes in global memory (L2), per rank
  int64_t cache_cols;
  int32_t M, m_pow2;
  float inv_m;
  int32_t smem_planes;   // GPTS instances: the first planes of a slice stay in shared memory
};

__device__ __forceinline__ Cand cand_none(bool for_max) { return Cand{for_max ? 0ull : ~0ull, 0.0, kNone, 1, -1, 0}; }
__device__ __forceinline__ WCand wcand_none(bool for_max) { return WCand{for_max ? 0ull : ~0ull, kNone, 1}; }

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
  const uint32_t bh = MAX_KEY ? __reduce_max_sync(full, live ? h : 0u) : __reduce_min_sync(full, live ? h : 0xffffffffu);
  const unsigned hmask = __ballot_sync(full, live && h == bh);
  if (__popc(hmask) == 1) {  // common case: the high word alone decides (one REDUX + one vote)
    const int wl = __ffs(hmask) - 1;
    bidx = __shfl_sync(full, idx, wl);
    bkey = ((uint64_t)bh << 32) | __shfl_sync(full, l, wl);
    return wl;
  }
  if (hmask == 0u) {  // every lane empty
    bidx = kNone;
    bkey = MAX_KEY ? 0ull : ~0ull;
    return -1;
  }
  const uint32_t bl = MAX_KEY ? __reduce_max_sync(full, (live && h == bh) ? l : 0u)
                              : __reduce_min_sync(full, (live && h == bh) ? l : 0xffffffffu);
  const bool eq = live && h == bh && l == bl;
  bidx = (int)__reduce_min_sync(full, eq ? (unsigned)idx : (unsigned)kNone);
  bkey = ((uint64_t)bh << 32) | bl;
  const unsigned own = __ballot_sync(full, eq && idx == bidx);
  return own ? __ffs(own) - 1 : -1;
}

// The lane holding the warp's lexicographic best (key, idx) — warp_argbest without
// distributing the winner (its owner already has it). -1: every lane empty.
template <bool MAX_KEY>
__device__ __forceinline__ int warp_arglane(uint64_t key, int idx) {
  const unsigned full = 0xffffffffu;
  const bool live = idx != kNone;
  const uint32_t h = (uint32_t)(key >> 32), l = (uint32_t)key;
  const uint32_t bh = MAX_KEY ? __reduce_max_sync(full, live ? h : 0u) : __reduce_min_sync(full, live ? h : 0xffffffffu);
  const unsigned hmask = __ballot_sync(full, live && h == bh);
  if (hmask == 0u) return -1;
  if (__popc(hmask) == 1) return __ffs(hmask) - 1;
  const uint32_t bl = MAX_KEY ? __reduce_max_sync(full, (live && h == bh) ? l : 0u)
                              : __reduce_min_sync(full, (live && h == bh) ? l : 0xffffffffu);
  const bool eq = live && h == bh && l == bl;
  const int bidx = (int)__reduce_min_sync(full, eq ? (unsigned)idx : (unsigned)kNone);
  const unsigned own = __ballot_sync(full, eq && idx == bidx);
  return own ? __ffs(own) - 1 : -1;
}

// (key, idx) of a beats that of b: smaller key (MAX_KEY: larger), then smaller idx. Empty
// entries carry the neutral key and idx = kNone (the largest index), so they lose to any
// live entry — the order warp_argbest implements, as a plain comparison.
template <bool MAX_KEY>
__device__ __forceinline__ bool cand_beats(uint64_t ka, int ia, uint64_t kb, int ib) {
  // bitwise, not short-circuit: the compiler otherwise branches at every comparison
  return (bool)((int)(MAX_KEY ? ka > kb : ka < kb) | ((int)(ka == kb) & (int)((unsigned)ia < (unsigned)ib)));
}

// The best of up to 8 candidates every lane has read itself (broadcast loads): a 3-level
// selection tree in registers. Against warp_argbest (REDUX -> vote -> shuffles, each a
// dependent MIO round trip, ~130 cycles + payload) this is 8 independent loads and 3
// dependent compare-select levels, but ~100 instructions: it pays where one warp runs it
// (the CTA stage of a cluster: N = 8,446, C = 9 1.139 -> 1.128 us per iteration), not
// where all warps run it redundantly.
template <bool MAX_KEY>
__device__ __forceinline__ Cand best_of8(Cand (&e)[8]) {
#pragma unroll
  for (int st = 4; st >= 1; st >>= 1)
#pragma unroll
    for (int i = 0; i < st; ++i)
    {  // field-wise selects (no branches)
      const bool t = cand_beats<MAX_KEY>(e[i + st].key, e[i + st].idx, e[i].key, e[i].idx);
      e[i].key = t ? e[i + st].key : e[i].key;
      e[i].Y = t ? e[i + st].Y : e[i].Y;
      e[i].idx = t ? e[i + st].idx : e[i].idx;
      e[i].y = t ? e[i + st].y : e[i].y;
      e[i].slot = t ? e[i + st].slot : e[i].slot;
    }
  return e[0];
}

// ---- cluster exchange of the CTA winners (C > 1) ----
// CTA r's winner goes into slot [b][r] of every CTA's inbox by st.async (DSMEM stores that
// complete transaction bytes on the receiver's mbarrier); each CTA then waits on its own
// inbox barrier — a point-to-point hand-off instead of a cluster-wide barrier.
constexpr uint32_t kCandMsgBytes = 32;  // key, Y | idx, y, slot, pad

__device__ __forceinline__ uint32_t cluster_addr(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v2b64(uint32_t dst, uint64_t a, uint64_t b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               ::"r"(dst), "l"(a), "l"(b), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_v2b32(uint32_t dst, uint32_t a, uint32_t b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];"
               ::"r"(dst), "r"(a), "r"(b), "r"(bar) : "memory");
}
// wait with cluster-scope acquire: the peers' st.async data is visible afterwards
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// K rows are read-only for the kernel's lifetime: the non-coherent path. The lazy column
// cache is written by this kernel, so its reads take the coherent path.
template <bool COHERENT>
__device__ __forceinline__ float ld_evict_last(const float* p, uint64_t pol) {
  float v;
  if (COHERENT)
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// Lazy mode: column idx is read from its cache slot, or computed and stored in the next
// free slot while the cache has room (computeKernelMatrixColumn).
__device__ __forceinline__ void assign_column(Decision& d, int slot, int nfree, const TrainArgs& A) {
  d.slot = slot;
  d.new_slot = (slot < 0 && nfree < A.cache_cols) ? nfree : -1;
}

// Alg. 1's branch on the min candidate.
__device__ __forceinline__ Decision decide_min(const Cand& b, int64_t iters, int64_t nnz, int nfree,
                                               const TrainArgs& A) {
  Decision d = {};
  d.slot = d.new_slot = -1;
  const bool has = b.idx != kNone;
  const double m = has ? key_value(b.key) : INFINITY;
  d.nnz = nnz;
  if (iters >= A.iter_max || !has) {
    d.action = ACT_STOP;
    d.converged = has && m > 0.0;
  } else if (m <= 0.0 && (nnz < A.s_max || b.Y != 0.0)) {
    d.action = ACT_ADD;
    const double beta_i = b.y > 0 ? A.beta : 1.0;   // b_i = beta^(0.5 (y_i + 1))
    const double sdelta = __dsub_rn(beta_i, m);     // y_i delta, delta = b_i y_i - F_i (Eq. 6); m = y_i F_i
    d.idx = b.idx;
    d.delta = b.y > 0 ? sdelta : -sdelta;
    d.newY = __dadd_rn(b.Y, sdelta);                 // y_i (alpha_i + delta) (Eq. 7)
    d.nnz = nnz + (b.Y == 0.0 && d.newY != 0.0) - (b.Y != 0.0 && d.newY == 0.0);
    assign_column(d, b.slot, nfree, A);
  } else {
    d.action = ACT_CHECK_REMOVAL;
    d.converged = m > 0.0;
  }
  return d;
}

// Alg. 1's redundant-support branch.
__device__ __forceinline__ Decision decide_removal(Decision d, const Cand& b, int nfree, const TrainArgs& A) {
  if (b.idx != kNone && key_value(b.key) > 0.0) {
    d.action = ACT_REMOVE;
    d.idx = b.idx;
    d.delta = b.y > 0 ? -b.Y : b.Y;  // -alpha_i = -y_i (y_i alpha_i)
    d.newY = 0.0;
    d.nnz = d.nnz - 1;
    assign_column(d, b.slot, nfree, A);
  } else {
    d.action = ACT_STOP;
  }
  return d;
}

// LMP = 0: K is given (fastron_train). LMP > 0: lazy columns of the FK kernel with LMP
// padded control points and term LKIND (fastron_train_lazy).
// GPTS: the lazy mode's point planes live in global memory (L2-resident scratch from the
// workspace) instead of shared memory — slices too large for the 200 KB budget (N = 20,000
// at M = 16: 1,250 points x 192 B per CTA). A computed column then reads its planes from L2.
// ONE: single-CTA instance (launched with C = 1 only) that keeps the winners' payload beside
// the warp winners (the dependent shared-memory load after the REDUX costs it more than
// the wider records: N = 1,000 0.80 against 0.81 us per iteration).
// NSPL (GPTS only): planes [0, NSPL) of a slice stay in shared memory, the rest in L2 — a
// compile-time split, so every plane access is a plain LDS or LDG (a runtime split through
// generic pointers cost more than it saved: 2.70 -> 3.23 us per iteration at cfg5 scale).
template <int EPT, int LMP, int LKIND, bool GPTS = false, bool ONE = false, int NSPL = 0>
__global__ void __launch_bounds__(kTrainNT, 1) train_kernel(const __grid_constant__ TrainArgs A) {
  constexpr bool LAZY = LMP > 0;
  constexpr int LNP = LAZY ? LMP / 2 : 1;
  constexpr int64_t LTF = tile_floats(LAZY ? LMP : 2);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s_Y = reinterpret_cast<double*>(smem_raw);  // [chunk], owner-thread access only
  // lazy mode: the slice's pre-scaled points as structure-of-arrays f32x2 planes
  // s_pts[(p * 3 + coord) * chunk + j] (control points 2p, 2p+1 of point j): a thread reads
  // its own points, so consecutive lanes read consecutive 8-byte words — conflict-free
  // (a per-point record layout put every lane on the same banks: 32-way conflicts, ~11k
  // cycles per computed column). Then the cache slot of each local index's K column.
  // GPTS: planes [0, smem_planes) of the slice in shared memory, the rest in the workspace
  // (L2): at cfg5 scale 20 of the 24 planes fit, so a computed column reads 40 KB instead
  // of 240 KB through L2.
  f2* s_pts = reinterpret_cast<f2*>(smem_raw + ((A.chunk * 8 + 15) & ~15ll));
  f2* g_pts = GPTS ? A.gpts + (int64_t)rank * LNP * 3 * A.chunk : nullptr;
  constexpr int n_spl = GPTS ? NSPL : LNP * 3;
  int32_t* s_slot = reinterpret_cast<int32_t*>(s_pts + (LAZY ? A.chunk * n_spl : 0));
  // (plane pl = p * 3 + coord; pl is a constant after unrolling, so pl < n_spl folds)
  __shared__ __align__(16) WCand s_warp[2][kTrainWarps];
  __shared__ double s_wY[2][ONE ? kTrainWarps : 1];      // ONE: Y and cache slot of the warp winners
  __shared__ int32_t s_wslot[2][ONE ? kTrainWarps : 1];
  __shared__ Cand s_inbox[2][kMaxCluster];                  // C > 1: the CTA winners of an exchange
  __shared__ __align__(8) uint64_t s_inbar[2];              // their arrival barriers
  __shared__ int32_t s_cta_cnt[2];
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
    if (LAZY && live) {
      s_slot[j] = -1;
      const int64_t g = lo + j;
      const float* src = A.packed + (g / kTileSupports) * LTF + (g % kTileSupports) * LNP * 8;
#pragma unroll
      for (int p = 0; p < LNP; ++p) {
        const float4 xy = *reinterpret_cast<const float4*>(src + p * 8);
        const float2 zz = *reinterpret_cast<const float2*>(src + p * 8 + 4);
        if (p * 3 + 0 < n_spl) s_pts[(int64_t)(p * 3 + 0) * A.chunk + j] = pk(xy.x, xy.y);
        else g_pts[(int64_t)(p * 3 + 0) * A.chunk + j] = pk(xy.x, xy.y);
        if (p * 3 + 1 < n_spl) s_pts[(int64_t)(p * 3 + 1) * A.chunk + j] = pk(xy.z, xy.w);
        else g_pts[(int64_t)(p * 3 + 1) * A.chunk + j] = pk(xy.z, xy.w);
        if (p * 3 + 2 < n_spl) s_pts[(int64_t)(p * 3 + 2) * A.chunk + j] = pk(zz.x, zz.y);
        else g_pts[(int64_t)(p * 3 + 2) * A.chunk + j] = pk(zz.x, zz.y);
      }
    }
  }
  if (tid == 0) {  // inbox barriers: one local arrival (with the expected bytes) per exchange
    mbar_init(&s_inbar[0], 1);
    mbar_init(&s_inbar[1], 1);
    fence_barrier_init();
  }
  // initial count(alpha != 0) over the cluster (its cluster barrier also publishes the
  // initialised inbox barriers to the peers)
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

  // C > 1: exchange number ex uses inbox slot ex & 1 at barrier phase (ex >> 1) & 1. A peer
  // cannot send into a slot again before this CTA has consumed it: its next message there
  // needs this CTA's message of the exchange in between, sent only after this CTA's
  // barrier that follows its reads.
  uint32_t ex = 0;
#ifdef FASTRON_TRAIN_PROF
  unsigned long long prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long prof_miss = 0, n_miss = 0;  // lazy mode: cycles in computed columns
  unsigned long long tp = clock64();
#define PROF_MARK(i)                         \
  do {                                       \
    const unsigned long long tn = clock64(); \
    prof[i] += tn - tp;                      \
    tp = tn;                                 \
  } while (0)
#else
#define PROF_MARK(i) \
  do {               \
  } while (0)
#endif
  // The CTA's winner from the warp winners of buffer q (every lane of the calling warp gets
  // it): a selection tree over the 8 records, then the payload of the one winner: in a cluster
  // (C > 1, warp 0 only) Y (and the lazy mode's cache slot) by a broadcast load from this
  // CTA's shared memory, so the warp stage moves 16 bytes per warp and never touches Y
  // (cfg3, C = 5: 1.155 -> 1.128 us per iteration).
  auto cta_best = [&](int q, bool for_max) -> Cand {
    if (ONE) {
      // one CTA, every warp redundantly: REDUX argbest, the payload the owner lanes stored
      // beside their warp winners by shuffles
      const WCand w = lane < kTrainWarps ? s_warp[q][lane] : wcand_none(for_max);
      const double Yl = lane < kTrainWarps ? s_wY[q][lane] : 0.0;
      const int sl = (LAZY && lane < kTrainWarps) ? s_wslot[q][lane] : -1;
      Cand b = cand_none(for_max);
      const int wl = for_max ? warp_argbest<true>(w.key, w.idx, b.key, b.idx) : warp_argbest<false>(w.key, w.idx, b.key, b.idx);
      const int src = wl < 0 ? 0 : wl;
      b.y = __shfl_sync(0xffffffffu, w.y, src);
      b.Y = __shfl_sync(0xffffffffu, Yl, src);
      if (LAZY) b.slot = __shfl_sync(0xffffffffu, sl, src);
      return b;
    }
    if (C == 1) {
      // one CTA without the ONE instance (lazy mode, forced C): REDUX argbest, the winner's
      // payload by a broadcast load
      const WCand w = lane < kTrainWarps ? s_warp[q][lane] : wcand_none(for_max);
      Cand b = cand_none(for_max);
      const int wl = for_max ? warp_argbest<true>(w.key, w.idx, b.key, b.idx) : warp_argbest<false>(w.key, w.idx, b.key, b.idx);
      b.y = __shfl_sync(0xffffffffu, w.y, wl < 0 ? 0 : wl);
      if (wl >= 0) {
        b.Y = s_Y[b.idx - lo];
        if (LAZY) b.slot = s_slot[b.idx - lo];
      }
      return b;
    }
    // cluster (warp 0 only): every lane reads the 8 records itself and selects in registers
    static_assert(kTrainWarps <= 8, "best_of8 covers the warp winners of one CTA");
    Cand e[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      e[w] = cand_none(for_max);
      if (w < kTrainWarps) {
        const WCand c = s_warp[q][w];
        e[w].key = c.key;
        e[w].idx = c.idx;
        e[w].y = c.y;
      }
    }
    Cand b = for_max ? best_of8<true>(e) : best_of8<false>(e);
#ifdef FASTRON_TRAIN_PROF
    if (b.idx == -12345) prof[11] += 1;  // the tree's result is needed here
    PROF_MARK(11);
#endif
    if (b.idx != kNone) {
      b.Y = s_Y[b.idx - lo];
      if (LAZY) b.slot = s_slot[b.idx - lo];
    }
    return b;
  };
  auto cluster_best = [&](const Cand& mine, bool for_max) -> Cand {  // mine: warp 0's CTA winner
    const int b = (int)(ex & 1u);
    if (warp == 0) {
      if (lane == 0) mbar_expect_tx(&s_inbar[b], (uint32_t)C * kCandMsgBytes);
      if (lane < C) {  // lane r delivers this CTA's winner to rank r
        const uint32_t dst = cluster_addr(&s_inbox[b][rank], lane);
        const uint32_t bar = cluster_addr(&s_inbar[b], lane);
        st_async_v2b64(dst, mine.key, (uint64_t)__double_as_longlong(mine.Y), bar);
        st_async_v2b64(dst + 16, ((uint64_t)(uint32_t)mine.y << 32) | (uint32_t)mine.idx,
                       (uint64_t)(uint32_t)mine.slot, bar);
      }
    }
    PROF_MARK(8);
    mbar_wait_cluster(&s_inbar[b], (ex >> 1) & 1u);
    PROF_MARK(9);
    ++ex;
    // the C CTA winners: REDUX argbest over (key, idx), the winner's payload by a broadcast
    // load. (A selection tree over entries every lane reads itself was measured slower here,
    // 295 -> 588 cycles: all 8 warps run this stage redundantly, so its ~140 instructions
    // per warp are issue-bound, while the REDUX path is ~20.)
    uint64_t key = for_max ? 0ull : ~0ull;
    int idx = kNone;
    if (lane < C) {
      key = s_inbox[b][lane].key;
      idx = s_inbox[b][lane].idx;
    }
    Cand best = cand_none(for_max);
    const int wl = for_max ? warp_argbest<true>(key, idx, best.key, best.idx) : warp_argbest<false>(key, idx, best.key, best.idx);
    if (wl >= 0) {
      best.Y = s_inbox[b][wl].Y;
      best.y = s_inbox[b][wl].y;
      best.slot = s_inbox[b][wl].slot;
    }
    PROF_MARK(10);
    return best;
  };

  int64_t iters = 0, n_add = 0, n_remove = 0;
  int upd_i = -1;  // row of the pending rank-one update of F
  double upd_delta = 0.0;
  int upd_slot = -1, upd_new_slot = -1;  // lazy mode: where column upd_i comes from / goes to
  int nfree = 0;                         // lazy mode: next free cache slot (uniform)
  int parity = 0;
  int converged = 0;

  for (;;) {
    // ---- 1. all loads of the pending K row, then the fused update + min scan ----
    float kr[EPT];
    const bool have_upd = upd_i >= 0;
    if (have_upd) {
      if (!LAZY || upd_slot >= 0) {
        const float* Krow = LAZY ? A.cache + (int64_t)upd_slot * A.n + lo : A.K + (int64_t)upd_i * A.ldk + lo;
#pragma unroll
        for (int k = 0; k < EPT; ++k) kr[k] = ld_evict_last<LAZY>(Krow + koff[k], pol);
      } else if (LAZY) {
#ifdef FASTRON_TRAIN_PROF
        const unsigned long long t_miss = clock64();
#endif
        // computeKernelMatrixColumn(i): K(X_j, X_i) for the thread's slots,
        // with the same term function and summation order as fastron_gram (bit-identical)
        const float* wr = A.packed + (int64_t)(upd_i / kTileSupports) * LTF + (upd_i % kTileSupports) * LNP * 8;
        f2 vx[LNP], vy[LNP], vz[LNP];
#pragma unroll
        for (int p = 0; p < LNP; ++p) {
          const float4 xy = __ldg(reinterpret_cast<const float4*>(wr + p * 8));
          const float2 zz = __ldg(reinterpret_cast<const float2*>(wr + p * 8 + 4));
          vx[p] = pk(xy.x, xy.y);
          vy[p] = pk(xy.z, xy.w);
          vz[p] = pk(zz.x, zz.y);
        }
        if (A.M < LMP) {  // odd M: x_i's padded point at 0 so the padded term is 0 (as in K3)
          vx[LNP - 1] &= 0xffffffffull;  // high lane (control point MP-1) := +0.0f
          vy[LNP - 1] &= 0xffffffffull;
          vz[LNP - 1] &= 0xffffffffull;
        }
        // split GPTS instance: the few planes that live in L2, for every live slot, in one
        // batch up front (the cache stores between the slots would otherwise fence each
        // slot's loads behind the previous slot's store: one L2 round trip per slot)
        constexpr int NG = (GPTS && NSPL > 0) ? LNP * 3 - NSPL : 0;
        f2 gq[NG > 0 ? EPT : 1][NG > 0 ? NG : 1];
        if (NG > 0) {
#pragma unroll
          for (int k = 0; k < EPT; ++k) {
            if (k * kTrainNT >= len) continue;
#pragma unroll
            for (int g = 0; g < NG; ++g) gq[k][g] = g_pts[(int64_t)(NSPL + g) * A.chunk + koff[k]];
          }
        }
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          // slots past the slice (whole rounds of 256: uniform over the CTA) hold G = +inf and
          // need no column entry; with the planes in global memory (GPTS: 8 slots per thread
          // for ~5 live ones at cfg5 scale) they were 3/8 of a computed column's time
          if (k * kTrainNT >= len) {
            kr[k] = 0.0f;
            continue;
          }
          // GPTS: all of the slot's plane reads first (L2 round trips: one batch per slot
          // instead of one per control-point pair), then the terms
          f2 acc;
          if (GPTS) {
            f2 ux[LNP], uy[LNP], uz[LNP];
#pragma unroll
            for (int p = 0; p < LNP; ++p) {
#define FASTRON_PL(pl)                                                                      \
  ((pl) < n_spl ? s_pts[(int64_t)(pl) * A.chunk + koff[k]]                                  \
                : NG > 0 ? gq[k][(pl) - n_spl < 0 ? 0 : (pl) - n_spl] : g_pts[(int64_t)(pl) * A.chunk + koff[k]])
              ux[p] = FASTRON_PL(p * 3 + 0);
              uy[p] = FASTRON_PL(p * 3 + 1);
              uz[p] = FASTRON_PL(p * 3 + 2);
#undef FASTRON_PL
            }
#pragma unroll
            for (int p = 0; p < LNP; ++p)
              accum_term<LKIND>(acc, sub2(ux[p], vx[p]), sub2(uy[p], vy[p]), sub2(uz[p], vz[p]), p == 0);
          } else {
#pragma unroll
            for (int p = 0; p < LNP; ++p) {
              const f2 ux = s_pts[(int64_t)(p * 3 + 0) * A.chunk + koff[k]];
              const f2 uy = s_pts[(int64_t)(p * 3 + 1) * A.chunk + koff[k]];
              const f2 uz = s_pts[(int64_t)(p * 3 + 2) * A.chunk + koff[k]];
              accum_term<LKIND>(acc, sub2(ux, vx[p]), sub2(uy, vy[p]), sub2(uz, vz[p]), p == 0);
            }
          }
          const float ks = pair_sum(acc);
          const float v = A.m_pow2 ? ks * A.inv_m : __fdiv_rn(ks, (float)A.M);
          kr[k] = v;
          const int j = k * kTrainNT + tid;
          if (upd_new_slot >= 0 && j < len) A.cache[(int64_t)upd_new_slot * A.n + lo + j] = v;
        }
#ifdef FASTRON_TRAIN_PROF
        {
          // force completion of the computed values before reading the clock
          float sink = 0.f;
#pragma unroll
          for (int k = 0; k < EPT; ++k) sink += kr[k];
          if (sink == -1.f) prof_miss += 1;
          prof_miss += clock64() - t_miss;
          ++n_miss;
        }
#endif
      }
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
    PROF_MARK(0);
    // merge (slot order == index order inside a thread; the lower slot wins ties)
    double mk = m0;
    int mkk = k0;
    if (m1 < m0 || (m1 == m0 && k1 >= 0 && k1 < k0)) { mk = m1; mkk = k1; }
    const int my_idx = (mkk >= 0 && mk != INFINITY) ? lo + mkk * kTrainNT + tid : kNone;
    {
      const uint64_t okey = order_key(mk);
      PROF_MARK(6);
      const int wl = warp_arglane<false>(okey, my_idx);
      PROF_MARK(7);
      if (lane == wl) {  // the owner lane writes the warp winner
        s_warp[parity][warp] = WCand{okey, my_idx, ((yneg >> mkk) & 1u) ? -1 : 1};
        if (ONE) {
          const int jw = mkk * kTrainNT + tid;
          s_wY[parity][warp] = s_Y[jw];
          if (LAZY) s_wslot[parity][warp] = s_slot[jw];
        }
      } else if (wl < 0 && lane == 0) {
        s_warp[parity][warp] = wcand_none(false);
      }
    }
    PROF_MARK(1);
    __syncthreads();
    PROF_MARK(2);

    // ---- 2. CTA (and cluster) reduction + the decision of Algorithm 1, taken redundantly
    //         by every warp (identical inputs -> identical decisions, no second barrier;
    //         the candidate buffers are double-buffered by parity) ----
    Decision d;
    if (C == 1) {
      d = decide_min(cta_best(parity, false), iters, nnz, nfree, A);
    } else {
      Cand mine = cand_none(false);
      if (warp == 0) mine = cta_best(parity, false);
      const Cand best = cluster_best(mine, false);
      d = decide_min(best, iters, nnz, nfree, A);
    }
    PROF_MARK(3);
    PROF_MARK(4);

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
        const uint64_t rkey = order_key(rk);
        const int wl = warp_arglane<true>(rkey, ridx);
        if (lane == wl) {
          s_warp[q][warp] = WCand{rkey, ridx, ((yneg >> rkk) & 1u) ? -1 : 1};
          if (ONE) {
            const int jw = rkk * kTrainNT + tid;
            s_wY[q][warp] = s_Y[jw];
            if (LAZY) s_wslot[q][warp] = s_slot[jw];
          }
        } else if (wl < 0 && lane == 0) {
          s_warp[q][warp] = wcand_none(true);
        }
      }
      __syncthreads();
      if (C == 1) {
        d = decide_removal(d, cta_best(q, true), nfree, A);
      } else {
        Cand mine = cand_none(true);
        if (warp == 0) mine = cta_best(q, true);
        const Cand best = cluster_best(mine, true);
        d = decide_removal(d, best, nfree, A);
      }
      parity = q;  // buffers of parity q were used last; the loop flips back below
    }

    if (d.action == ACT_STOP) {
      converged = d.converged;
      break;
    }
    PROF_MARK(5);
    // apply the step: the owner thread updates Y_i, everyone records the pending
    // rank-one update of G for the next pass
    if (d.idx >= lo && d.idx < hi && ((d.idx - lo) % kTrainNT) == tid) {
      s_Y[d.idx - lo] = d.newY;
      if (LAZY && d.new_slot >= 0) s_slot[d.idx - lo] = d.new_slot;
    }
    if (LAZY) {
      upd_slot = d.slot;
      upd_new_slot = d.new_slot;
      if (d.new_slot >= 0) nfree = d.new_slot + 1;
    }
    if (tid == 0 && rank == 0 && A.trace) A.trace[iters] = d.action == ACT_ADD ? d.idx : -(d.idx + 1);
    if (d.action == ACT_ADD) ++n_add;
    else ++n_remove;
    upd_i = d.idx;
    upd_delta = d.delta;
    nnz = d.nnz;
    ++iters;
    parity ^= 1;
  }

#ifdef FASTRON_TRAIN_PROF
  if (tid == 0 && rank == 0 && n_miss) printf("train prof computed columns %llu, %.0f cycles each\n", n_miss, (double)prof_miss / n_miss);
  if (tid == 0 && rank == 0)
    printf("train prof cycles/iter: scan %.0f merge+key %.0f argbest %.0f payload %.0f bar %.0f | cta-tree %.0f payload+send %.0f inbox-wait %.0f inbox-best %.0f decide %.0f - %.0f tail %.0f (iters %lld)\n",
           (double)prof[0] / iters, (double)prof[6] / iters, (double)prof[7] / iters, (double)prof[1] / iters,
           (double)prof[2] / iters, (double)prof[11] / iters, (double)prof[8] / iters, (double)prof[9] / iters,
           (double)prof[10] / iters,
           (double)prof[3] / iters, (double)prof[4] / iters, (double)prof[5] / iters, (long long)iters);
#endif
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

// Cluster size for n points when a CTA holds at most chunk_max. Up to 2,048 points one
// CTA (8 slots per thread) beats any cluster, whose winner exchange costs ~0.15 us per
// iteration; above, ~1,024 points per CTA (4 slots per thread) — measured at 256 threads
// (tools/train_sweep.py, us / iteration): N = 2,000 C = 1 0.98, C = 2 1.14; N = 3,000
// C = 1 1.16, C = 3 1.14; N = 5,000 C = 1 1.50, C = 4 1.31 (8 slots), C = 5 1.15,
// C = 8 1.16; N = 8,446 C = 9 1.30, C = 12 1.31. FASTRON_TRAIN_CLUSTER sets C (tuning and
// tests; never below the minimum that fits).
static int train_cluster_size(int64_t n, int64_t chunk_max) {
  int64_t C = (n + chunk_max - 1) / chunk_max;  // the minimum that fits
  if (C < 1) C = 1;
  const int64_t c_min = C;
  if (n > 2048) {
    int64_t c_small = (n + 1023) / 1024;
    if (c_small > kMaxCluster) c_small = kMaxCluster;
    if (c_small > C) C = c_small;
  }
  if (const char* env = getenv("FASTRON_TRAIN_CLUSTER")) {
    const int64_t c = atoi(env);
    C = c > c_min ? c : c_min;
  }
  return (int)C;
}

template <int EPT, int LMP = 0, int LKIND = 0, bool GPTS = false, bool ONE = false, int NSPL = 0>
static cudaError_t launch_ept(const TrainArgs& A, int C, cudaStream_t st, size_t smem) {
  static std::atomic<int> attr[kMaxDevices];
  const int dev = device_slot();
  if (!attr[dev].load()) {
    cudaFuncSetAttribute(train_kernel<EPT, LMP, LKIND, GPTS, ONE, NSPL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(train_kernel<EPT, LMP, LKIND, GPTS, ONE, NSPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr[dev].store(1);
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
  return cudaLaunchKernelEx(&cfg, train_kernel<EPT, LMP, LKIND, GPTS, ONE, NSPL>, A);
}

cudaError_t launch_train(const float* K, int64_t n, int64_t ldk, const int8_t* y, double beta, int64_t iter_max,
                         int64_t s_max, double* alpha, double* F, int32_t* support_idx, int32_t* trace, void* result,
                         cudaStream_t st) {
  const int C = train_cluster_size(n, kChunkMax);
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
  A.packed = nullptr;
  A.gpts = nullptr;
  A.cache = nullptr;
  A.cache_cols = 0;
  A.M = 1;
  A.m_pow2 = 1;
  A.inv_m = 1.0f;
  A.smem_planes = 0;
  const int64_t ept = (A.chunk + kTrainNT - 1) / kTrainNT;
  const size_t smem = (size_t)A.chunk * 8;
  cudaError_t e;
  // the smallest instance that covers the slice: dead slots still cost a load and an update
  // instances at sixths of the register budget (4, 8, ..., 24 slots at 256 threads)
  constexpr int E = kMaxEPT / 6;
  if (C == 1 && ept <= E) e = launch_ept<E, 0, 0, false, true>(A, C, st, smem);
  else if (C == 1 && ept <= 2 * E) e = launch_ept<2 * E, 0, 0, false, true>(A, C, st, smem);
  else if (ept <= E) e = launch_ept<E>(A, C, st, smem);
  else if (ept <= E + E / 2) e = launch_ept<E + E / 2>(A, C, st, smem);  // 6 slots: N = 20,000 on 16 CTAs (5 live)
  else if (ept <= 2 * E) e = launch_ept<2 * E>(A, C, st, smem);
  else if (ept <= 3 * E) e = launch_ept<3 * E>(A, C, st, smem);
  else if (ept <= 4 * E) e = launch_ept<4 * E>(A, C, st, smem);
  else if (ept <= 5 * E) e = launch_ept<5 * E>(A, C, st, smem);
  else e = launch_ept<6 * E>(A, C, st, smem);
  g_launches.fetch_add(1);
  return e;
}

// ---- lazy-column mode ----
constexpr int64_t kLazySmem = 200 * 1024;  // shared-memory budget per CTA
constexpr int kLazyMaxEPT = 8;             // slots per thread in the lazy mode
constexpr int64_t kLazySmemGpts = 217 * 1024;  // GPTS instances: shared memory for Y, slots and the first planes

static int64_t lazy_bytes_per_slot(int MP) { return 8 + 4 + (int64_t)(MP / 2) * 24; }

// slices up to this many points keep their planes in shared memory; larger ones (up to
// kLazyMaxEPT x 256 per CTA) use the GPTS instance with the planes in global memory
static int64_t lazy_smem_chunk(int MP) {
  int64_t chunk = kLazySmem / lazy_bytes_per_slot(MP);
  return chunk > kLazyMaxEPT * kTrainNT ? kLazyMaxEPT * kTrainNT : chunk;
}

int64_t train_lazy_max_n(int M) {
  (void)M;
  return (int64_t)kLazyMaxEPT * kTrainNT * kMaxCluster;
}

// FASTRON_LAZY_GPTS=1 (env, tests): global point planes even where shared memory suffices
static bool lazy_force_gpts() {
  const char* e = getenv("FASTRON_LAZY_GPTS");
  return e && e[0] == '1';
}

// bytes of global point planes fastron_train_lazy needs for n points (0: shared memory)
size_t train_lazy_plane_bytes(int64_t n, int M) {
  const int MP = padded_m(M);
  if (train_cluster_size(n, lazy_smem_chunk(MP)) <= kMaxCluster && !lazy_force_gpts()) return 0;
  const int C = train_cluster_size(n, (int64_t)kLazyMaxEPT * kTrainNT);
  const int64_t chunk = (n + C - 1) / C;
  return (size_t)C * chunk * (MP / 2) * 3 * sizeof(f2);
}

// planes a GPTS instance can keep in shared memory: 5/6 of the slice's (20 of 24 at M = 16:
// 1,250 points x 160 B + Y + slots = 215 KB), or none when the slice is too long for that
constexpr int gpts_split_planes(int mp) { return (mp / 2) * 3 * 5 / 6; }

template <int MP, int KIND>
static cudaError_t launch_lazy_mp(const TrainArgs& A, int C, cudaStream_t st, size_t smem) {
  const int64_t ept = (A.chunk + kTrainNT - 1) / kTrainNT;
  if (A.gpts && A.smem_planes > 0) {  // 6 slots where they cover the slice (cfg5 scale: 5 live)
    if (ept <= 6) return launch_ept<6, MP, KIND, true, false, gpts_split_planes(MP)>(A, C, st, smem);
    return launch_ept<kLazyMaxEPT, MP, KIND, true, false, gpts_split_planes(MP)>(A, C, st, smem);
  }
  if (A.gpts) return launch_ept<kLazyMaxEPT, MP, KIND, true>(A, C, st, smem);
  if (ept <= 2) return launch_ept<2, MP, KIND>(A, C, st, smem);
  if (ept <= 4) return launch_ept<4, MP, KIND>(A, C, st, smem);
  return launch_ept<kLazyMaxEPT, MP, KIND>(A, C, st, smem);
}

cudaError_t launch_train_lazy(const float* packed, int64_t n, int M, int kind, const int8_t* y, double beta,
                              int64_t iter_max, int64_t s_max, double* alpha, double* F, int32_t* support_idx,
                              int32_t* trace, void* result, float* cache, int64_t cache_cols, void* planes,
                              cudaStream_t st) {
  const int MP = padded_m(M);
  int C = train_cluster_size(n, lazy_smem_chunk(MP));  // as in launch_train (lazy cfg3: C = 5)
  const bool gpts = C > kMaxCluster || lazy_force_gpts();
  if (gpts) C = train_cluster_size(n, (int64_t)kLazyMaxEPT * kTrainNT);
  if (C > kMaxCluster || (gpts && !planes)) return cudaErrorInvalidValue;
  TrainArgs A;
  A.K = nullptr;
  A.n = n;
  A.ldk = n;
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
  A.packed = packed;
  A.gpts = gpts ? static_cast<f2*>(planes) : nullptr;
  A.smem_planes = 0;
  if (gpts) {  // the split instance when its planes fit, else every plane in L2
    const int64_t fixed = ((A.chunk * 8 + 15) & ~15ll) + A.chunk * 4;
    const int sp = gpts_split_planes(MP);
    const char* e = getenv("FASTRON_LAZY_SMEM_PLANES");  // "0": the all-L2 instance (tests, A/B)
    if (sp > 0 && fixed + A.chunk * 8 * sp <= kLazySmemGpts && !(e && e[0] == '0')) A.smem_planes = sp;
  }
  A.cache = cache;
  A.cache_cols = cache_cols;
  A.M = M;
  A.m_pow2 = (M & (M - 1)) == 0;
  A.inv_m = 1.0f / (float)M;
  const size_t smem = (size_t)((A.chunk * 8 + 15) & ~15ll) +
                      (gpts ? (size_t)A.chunk * 8 * A.smem_planes : (size_t)A.chunk * (MP / 2) * 24) +
                      (size_t)A.chunk * 4;
  cudaError_t e;
  switch (MP) {
#define FASTRON_LCASE(mp)                                                                              \
  case mp:                                                                                             \
    e = kind == kGaussian ? launch_lazy_mp<mp, kGaussian>(A, C, st, smem) : launch_lazy_mp<mp, kRQ>(A, C, st, smem); \
    break;
    FASTRON_LCASE(2)
    FASTRON_LCASE(4)
    FASTRON_LCASE(6)
    FASTRON_LCASE(8)
    FASTRON_LCASE(10)
    FASTRON_LCASE(12)
    FASTRON_LCASE(14)
    FASTRON_LCASE(16)
#undef FASTRON_LCASE
    default:
      return cudaErrorInvalidValue;
  }
  g_launches.fetch_add(1);
  return e;
}

}  // namespace fastron
