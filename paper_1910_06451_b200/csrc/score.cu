// score.cu — K2, Fastron scoring f(x) = sum_i alpha_i K_FK(S_i, x) with
// K_FK of Eq. 4, plus the fused edge-check rounds (K4) that reuse
// the same support-streaming loop with an interpolate+FK prologue and a warp-vote
// epilogue.
//
// Design:
//  * The support set is first packed once per call into tiles of 64 supports
//    (pre-scaled, control points paired (m, m+1), alpha appended), so one
//    cp.async.bulk (TMA bulk copy) moves a whole tile into shared memory; a
//    3-stage mbarrier ring overlaps the next tiles' copies with compute.
//  * Each thread owns QT queries whose scaled control points live in registers as
//    f32x2 pairs; every support record is a warp-broadcast LDS.128 + LDS.64 shared
//    by the QT queries. Per control-point pair: 3 FADD2 + FMUL2 + 2 FFMA2 +
//    2 MUFU (ex2 or rcp) + FADD2 — MUFU-bound (one SFU op per term).
//  * Accumulation: per support the M terms are summed in two fp32 lanes (even and odd
//    control points, fixed order); both lane sums go to fp64 on the ALU pipe and are
//    added to the query's fp64 score with alpha (stored as double) by DFMA — no fp32
//    rounding above the 4-term lane sums (DESIGN.md §5 error budget). 1/M is applied
//    once at the end in fp64.
//  * Grid = query blocks x support splits, the split count chosen to fill 148 SMs in
//    whole waves; splits > 1 write fp64 partials that a second kernel adds in a fixed
//    order (deterministic).
#include "fastron_device.cuh"
#include "internal.h"

namespace fastron {

#ifndef FASTRON_REORDER
#define FASTRON_REORDER 1
#endif
#ifndef FASTRON_ACC_SPLIT
#define FASTRON_ACC_SPLIT 1
#endif
#ifndef FASTRON_SUP_UNROLL
#define FASTRON_SUP_UNROLL 2
#endif
constexpr int kSupUnroll = FASTRON_SUP_UNROLL;  // supports per unrolled step of K2's inner loop

#ifndef FASTRON_SCORE_NT
#define FASTRON_SCORE_NT 128
#endif
#ifndef FASTRON_SCORE_STAGES
#define FASTRON_SCORE_STAGES 3
#endif
constexpr int kNT = FASTRON_SCORE_NT;  // threads per scoring CTA
constexpr int kStages = FASTRON_SCORE_STAGES;  // TMA ring depth

#ifndef FASTRON_QT4
#define FASTRON_QT4 4
#endif
#ifndef FASTRON_QT8
#define FASTRON_QT8 3
#endif
#ifndef FASTRON_QT16
#define FASTRON_QT16 3
#endif
// queries per thread (A/B on the B200, bit-identical scores): M = 8: QT = 3
// (122 registers, 4 resident CTAs) beats 4 (158, 3 CTAs) by 1.2 % on the headline, 2/5/6
// are slower; M = 16: 3 (244 registers, 2 CTAs) beats 2 by 2 % and 1 by 15 %; M = 4:
// 4 (94 registers, 5 CTAs) beats 8 by 3.5 %.
__host__ __device__ constexpr int qt_for(int mp) {
  return mp <= 4 ? FASTRON_QT4 : mp <= 8 ? FASTRON_QT8 : mp <= 16 ? FASTRON_QT16 : 1;
}

int padded_m(int M) { return (M + 1) & ~1; }
int64_t n_support_tiles(int64_t ns) { return (ns + kTileSupports - 1) / kTileSupports; }
size_t packed_bytes(int64_t ns, int M) { return (size_t)n_support_tiles(ns) * (size_t)tile_bytes(padded_m(M)); }
int score_queries_per_cta(int M) { return kNT * qt_for(padded_m(M)); }

// ---------------------------------------------------------------------------------
// pack: spos float4 [M][lds] + alpha -> scaled, paired tiles
// ---------------------------------------------------------------------------------
__global__ void pack_kernel(const float4* __restrict__ spos, int64_t lds, const float* __restrict__ alpha, int64_t ns,
                            int M, int MP, float scale, float pad, float* __restrict__ packed, int64_t n_slots) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_slots) return;
  const int64_t tile = i / kTileSupports;
  const int s = (int)(i % kTileSupports);
  float* T = packed + tile * tile_floats(MP);
  float* rec = T + (int64_t)s * (MP / 2) * 8;
  const bool live = i < ns;
  for (int p = 0; p < MP / 2; ++p) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    const int m0 = 2 * p, m1 = 2 * p + 1;
    if (live) a = spos[(int64_t)m0 * lds + i];
    if (live && m1 < M) b = spos[(int64_t)m1 * lds + i];
    float ax = __fmul_rn(a.x, scale), ay = __fmul_rn(a.y, scale), az = __fmul_rn(a.z, scale);
    float bx = __fmul_rn(b.x, scale), by = __fmul_rn(b.y, scale), bz = __fmul_rn(b.z, scale);
    if (m1 >= M) bx = by = bz = pad;  // padded control point: term exactly 0 (FK) / no distance (joint)
    reinterpret_cast<float4*>(rec + p * 8)[0] = make_float4(ax, bx, ay, by);
    reinterpret_cast<float4*>(rec + p * 8)[1] = make_float4(az, bz, 0.f, 0.f);
  }
  reinterpret_cast<double*>(T + tile_record_floats(MP))[s] = (live && alpha) ? (double)alpha[i] : 0.0;
}

cudaError_t launch_pack(const float4* spos, int64_t lds, const float* alpha, int64_t ns, int M, float scale,
                        float* packed, cudaStream_t st, bool joint) {
  const int64_t slots = n_support_tiles(ns) * kTileSupports;
  if (slots == 0) return cudaSuccess;
  const int threads = 256;
  g_launches.fetch_add(1);
  return launch_pdl(pack_kernel, dim3((unsigned)((slots + threads - 1) / threads)), dim3(threads), 0, st, spos, lds,
                    alpha, ns, M, padded_m(M), scale, joint ? 0.0f : kPadCoord, packed, slots);
}

// ---------------------------------------------------------------------------------
// the scoring kernel (positions mode and fused edge mode)
// ---------------------------------------------------------------------------------
// MODE_POS: FK-kernel score of control-point positions (Eq. 4); MODE_EDGE: fused edge
// rounds; MODE_JOINT: the joint-space RBF kernel of the paper's "Fastron RBF" baseline
// (Table I): one RBF term of the whole joint-vector distance,
// with the joint vector laid out as ceil(D/3) zero-padded pseudo "control points".
enum { MODE_POS = 0, MODE_EDGE = 1, MODE_JOINT = 2 };

struct ScoreArgs {
  const float4* qpos;
  int64_t ldq;
  int64_t nq;  // number of (virtual) queries the grid covers
  const float* packed;
  int64_t n_tiles;
  int32_t tiles_per_split;
  int32_t n_splits;
  int32_t M;
  float scale;
  float* score;
  int8_t* label;
  double* partial;
  // edge mode
  const float* qa;
  const float* qb;
  int64_t ldqe;
  int32_t n_interp;
  int32_t round;
  const int32_t* active;
  const int32_t* active_count;
  int32_t* next_active;
  int32_t* next_count;
  uint8_t* in_collision;
  int32_t* hit_index;
  double denom;  // M for the FK kernel's 1/M mean (Eq. 4), 1 for the joint-space kernel
  double* score64;  // optional fp64 scores (margins for a warm start)
  int64_t plan_nq;  // host only: batch size the split count is planned for (0: nq)
  const float* qcfg;  // small fused query: configurations [nq][ldqc] (FK in the kernel)
  int64_t ldqc;
  // RQ refinement: pass 1 (fast term) appends the queries whose score lies
  // within refine_tau of 0 to refine_list; pass 2 (precise term) scores exactly those:
  // query vq of pass 2 is query qidx[vq] of the batch, for vq < *qcount
  int32_t* refine_list;
  int32_t* refine_count;
  double refine_tau;
  const int32_t* qidx;
  const int32_t* qcount;
};

// |f| below which a fast RQ score is recomputed with the precise term. The fast term's
// error at the headline size is rms 3.0e-6, max ~1.1e-5 (5.5 sigma over 1M queries ~1.7e-5);
// at |f| >= 0.5 the tolerance is >= 5e-5, a 3x margin, and ~0.9 % of the headline's
// queries fall below it.
constexpr double kRefineTau = 0.5;

__device__ __forceinline__ void maybe_refine(const ScoreArgs& A, int64_t vq, double fm) {
  if (A.refine_list && fabs(fm) < A.refine_tau) A.refine_list[atomicAdd(A.refine_count, 1)] = (int32_t)vq;
}

// pass 2: the batch index of (virtual) query vq
__device__ __forceinline__ int64_t batch_query(const ScoreArgs& A, int64_t vq) { return A.qidx ? A.qidx[vq] : vq; }

// Final write of one query's fp64 sum: 1/denom, fp64 / fp32 score, label (R8).
__device__ __forceinline__ void write_score(const ScoreArgs& A, int64_t vq, double f) {
  const double fm = f / A.denom;
  if (A.score64) A.score64[vq] = fm;
  if (A.score) A.score[vq] = (float)fm;
  if (A.label) A.label[vq] = fm > 0.0 ? 1 : -1;
}

// Position k of the visiting order of round r, lane l: evens first, then odds (R11).
__device__ __forceinline__ int edge_point(int n_interp, int o) {
  const int n_even = (n_interp + 1) >> 1;
  return o < n_even ? 2 * o : 2 * (o - n_even) + 1;
}

__device__ __forceinline__ int64_t edge_active_queries(const ScoreArgs& A) {
  return A.active_count ? (int64_t)(*A.active_count) * 32 : A.nq;
}

// Warp vote over the 32 lanes that hold one (edge, round) item; called by full warps.
__device__ __forceinline__ void edge_vote(const ScoreArgs& A, int64_t vq, double f) {
  const int lane = threadIdx.x & 31;
  const int64_t slot = vq >> 5;
  const int64_t n_active = edge_active_queries(A) >> 5;
  const bool in_range = slot < n_active;  // warp-uniform
  const int o = A.round * 32 + lane;
  const bool valid = in_range && o < A.n_interp;
  const bool hit = valid && f > 0.0;
  const unsigned ballot = __ballot_sync(0xffffffffu, hit);
  const int k = valid ? edge_point(A.n_interp, o) : 0x7fffffff;
  const int kmin = __reduce_min_sync(0xffffffffu, hit ? k : 0x7fffffff);
  if (!in_range || lane != 0) return;
  const int32_t e = A.active ? A.active[slot] : (int32_t)slot;
  if (ballot) {
    A.in_collision[e] = 1;
    if (A.hit_index) A.hit_index[e] = kmin;
  } else if ((A.round + 1) * 32 >= A.n_interp) {
    A.in_collision[e] = 0;
    if (A.hit_index) A.hit_index[e] = -1;
  } else {
    A.next_active[atomicAdd(A.next_count, 1)] = e;
  }
}

// K4 prologue, once per round: virtual query vq = (active slot vq / 32, lane vq % 32) ->
// interpolated configuration q_k = qa + t_k (qb - qa) in fp32 (R11) -> fp64 FK chain ->
// fp32 control points, SoA float4 [M][nq] (the layout the score kernel reads). Lanes past
// n_interp get zeros (they never vote). Computed once instead of in every support split.
__global__ void __launch_bounds__(256) edge_fk_kernel(const __grid_constant__ ScoreArgs A,
                                                      const __grid_constant__ FkParams P, float4* __restrict__ pos) {
  pdl_trigger();
  pdl_wait();
  const int64_t vq = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (vq >= edge_active_queries(A)) return;
  const int64_t slot = vq >> 5;
  const int o = A.round * 32 + (int)(vq & 31);
  if (o >= A.n_interp) {
    for (int m = 0; m < A.M; ++m) pos[(int64_t)m * A.nq + vq] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int32_t e = A.active ? A.active[slot] : (int32_t)slot;
  const int k = edge_point(A.n_interp, o);
  const float t = A.n_interp > 1 ? __fdiv_rn((float)k, (float)(A.n_interp - 1)) : 0.0f;
  const float* qa = A.qa + (int64_t)e * A.ldqe;
  const float* qb = A.qb + (int64_t)e * A.ldqe;
  fk_chain(
      P,
      [&](int jj) {
        const float a = __ldg(qa + jj), b = __ldg(qb + jj);
        return (double)__fadd_rn(a, __fmul_rn(t, __fsub_rn(b, a)));
      },
      [&](int m, double x, double y, double z) {
        pos[(int64_t)m * A.nq + vq] =
            make_float4(__double2float_rn(x), __double2float_rn(y), __double2float_rn(z), 0.0f);
      });
}

// QTO > 0 overrides the queries per thread: small and mid-size batches use QT = 1 (more,
// shorter CTAs and no dead query slots; the summation order per query, hence every bit,
// is the same for any QT)
template <int MP, int KIND, int MODE, int QTO = 0>
// (no min-blocks argument: with one, ptxas allocates more registers and fewer CTAs fit
// per SM — measured slower)
__global__ void __launch_bounds__(kNT) score_kernel(const __grid_constant__ ScoreArgs A,
                                                    const __grid_constant__ FkParams P) {
  constexpr int QT = QTO > 0 ? QTO : qt_for(MP);
  constexpr int NP = MP / 2;
  constexpr int64_t TF = tile_floats(MP);
  constexpr uint32_t TB = (uint32_t)tile_bytes(MP);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  float* stages = reinterpret_cast<float*>(smem_raw + 128);

  const int tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();  // before any global access (the counts, the packed tiles, the positions)
  const int64_t qb = blockIdx.x / A.n_splits;
  const int split = blockIdx.x % A.n_splits;
  const int64_t q_base = qb * (int64_t)(kNT * QT);
  const int64_t nq_live = MODE == MODE_EDGE ? edge_active_queries(A) : (A.qcount ? (int64_t)*A.qcount : A.nq);
  if (q_base >= nq_live) return;  // uniform: whole CTA idle (edge rounds / refinement: worst-case grids)

  const int64_t t0 = (int64_t)split * A.tiles_per_split;
  const int64_t t1 = min(t0 + (int64_t)A.tiles_per_split, A.n_tiles);
  const int nt = (int)max(t1 - t0, (int64_t)0);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages && s < nt; ++s) {
      mbar_expect_tx(&bars[s], TB);
      tma_bulk_g2s(stages + s * TF, A.packed + (t0 + s) * TF, TB, &bars[s]);
    }
  }

  // ---- queries -> scaled control points in registers (f32x2 pairs over m) ----
  f2 ux[QT][NP], uy[QT][NP], uz[QT][NP];
#pragma unroll
  for (int j = 0; j < QT; ++j) {
    const int64_t vq = q_base + j * kNT + tid;
    float px[MP], py[MP], pz[MP];
#pragma unroll
    for (int m = 0; m < MP; ++m) px[m] = py[m] = pz[m] = 0.0f;
    if (vq < nq_live) {
      // positions of the query (MODE_EDGE: of the interpolated configuration, written by
      // edge_fk_kernel for this round)
      const int64_t bq = batch_query(A, vq);
#pragma unroll
      for (int m = 0; m < MP; ++m) {
        if (m < A.M) {
          const float4 v = __ldg(A.qpos + (int64_t)m * A.ldq + bq);
          px[m] = v.x; py[m] = v.y; pz[m] = v.z;
        }
      }
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      ux[j][p] = pk(__fmul_rn(px[2 * p], A.scale), __fmul_rn(px[2 * p + 1], A.scale));
      uy[j][p] = pk(__fmul_rn(py[2 * p], A.scale), __fmul_rn(py[2 * p + 1], A.scale));
      uz[j][p] = pk(__fmul_rn(pz[2 * p], A.scale), __fmul_rn(pz[2 * p + 1], A.scale));
    }
  }

  double f[QT];
#pragma unroll
  for (int j = 0; j < QT; ++j) f[j] = 0.0;
  // RQ lanes start from -OFF (rq_lane_offset); 2 OFF sum(alpha) is added back at the end
  constexpr float OFF = MODE == MODE_JOINT ? 0.0f : rq_lane_offset<KIND, NP>();
  const f2 lane0 = OFF != 0.0f ? pk(-OFF, -OFF) : 0ull;
  double asum = 0.0;

  // ---- stream the support tiles ----
  for (int it = 0; it < nt; ++it) {
    const int st = it % kStages;
    mbar_wait(&bars[st], (uint32_t)((it / kStages) & 1));
    const float* T = stages + st * TF;
    const double* alpha = reinterpret_cast<const double*>(T + tile_record_floats(MP));
#pragma unroll kSupUnroll
    for (int s = 0; s < kTileSupports; ++s) {
      const float* rec = T + s * NP * 8;
      const double a = alpha[s];
      if (OFF != 0.0f) asum += a;
      if (MODE == MODE_JOINT) {
        // joint-space RBF: accumulate the squared distance over all pseudo points, one MUFU
        f2 s2[QT];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const float4 xy = *reinterpret_cast<const float4*>(rec + p * 8);
          const float2 zz = *reinterpret_cast<const float2*>(rec + p * 8 + 4);
          const f2 vx = pk(xy.x, xy.y), vy = pk(xy.z, xy.w), vz = pk(zz.x, zz.y);
#pragma unroll
          for (int j = 0; j < QT; ++j) {
            const f2 dx = sub2(ux[j][p], vx), dy = sub2(uy[j][p], vy), dz = sub2(uz[j][p], vz);
            s2[j] = p == 0 ? mul2(dx, dx) : fma2(dx, dx, s2[j]);
            s2[j] = fma2(dy, dy, s2[j]);
            s2[j] = fma2(dz, dz, s2[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          const float d2 = lo(s2[j]) + hi(s2[j]);
          float t;
          if (KIND == kGaussian) {
            t = ex2_neg(d2);
          } else {
            const float w = 1.0f + d2;
            t = rcp_approx(w * w);
          }
          f[j] = fma(a, nonneg_f32_to_f64(t), f[j]);
        }
        continue;
      }
      f2 acc[QT];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float4 xy = *reinterpret_cast<const float4*>(rec + p * 8);
        const float2 zz = *reinterpret_cast<const float2*>(rec + p * 8 + 4);
        const f2 vx = pk(xy.x, xy.y), vy = pk(xy.z, xy.w), vz = pk(zz.x, zz.y);
#if FASTRON_REORDER
        // coordinate-major order: consecutive instructions share the support operand,
        // letting the operand-reuse cache absorb one register-bank read per FADD2
        f2 dx[QT], dy[QT], dz[QT];
#pragma unroll
        for (int j = 0; j < QT; ++j) dx[j] = sub2(ux[j][p], vx);
#pragma unroll
        for (int j = 0; j < QT; ++j) dy[j] = sub2(uy[j][p], vy);
#pragma unroll
        for (int j = 0; j < QT; ++j) dz[j] = sub2(uz[j][p], vz);
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          accum_term<KIND>(acc[j], dx[j], dy[j], dz[j], p == 0, lane0);
        }
#else
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          accum_term<KIND>(acc[j], sub2(ux[j][p], vx), sub2(uy[j][p], vy), sub2(uz[j][p], vz), p == 0, lane0);
        }
#endif
      }
#pragma unroll
      for (int j = 0; j < QT; ++j) {
#if FASTRON_ACC_SPLIT
        if (KIND == kRQPrecise && MODE != MODE_JOINT) {  // offset lanes can be negative
          f[j] = fma(a, rq_lane_to_f64(lo(acc[j])), f[j]);
          f[j] = fma(a, rq_lane_to_f64(hi(acc[j])), f[j]);
        } else {
          f[j] = fma(a, nonneg_f32_to_f64(lo(acc[j])), f[j]);
          f[j] = fma(a, nonneg_f32_to_f64(hi(acc[j])), f[j]);
        }
#else
        f[j] = fma(a, nonneg_f32_to_f64(pair_sum(acc[j])), f[j]);
#endif
      }
    }
    __syncthreads();  // every thread is done with stage st
    if (tid == 0 && it + kStages < nt) {
      fence_proxy_async();
      mbar_expect_tx(&bars[st], TB);
      tma_bulk_g2s(stages + st * TF, A.packed + (t0 + it + kStages) * TF, TB, &bars[st]);
    }
  }

  // ---- epilogue ----
  if (OFF != 0.0f) {
#pragma unroll
    for (int j = 0; j < QT; ++j) f[j] = fma(2.0 * (double)OFF, asum, f[j]);
  }
#pragma unroll
  for (int j = 0; j < QT; ++j) {
    const int64_t vq = q_base + j * kNT + tid;
    if (A.n_splits > 1) {
      if (vq < nq_live) A.partial[(int64_t)split * A.nq + vq] = f[j];
    } else if (MODE == MODE_POS || MODE == MODE_JOINT) {
      if (vq < nq_live) {
        const double fm = f[j] / A.denom;
        const int64_t bq = batch_query(A, vq);
        if (A.score64) A.score64[bq] = fm;
        if (A.score) A.score[bq] = (float)fm;
        if (A.label) A.label[bq] = fm > 0.0 ? 1 : -1;
        maybe_refine(A, vq, fm);
      }
    } else {
      edge_vote(A, vq, f[j] / A.denom);
    }
  }
}

// Fixed-order reduction of the split partials (deterministic), then 1/M, score, label / vote.
template <int MODE>
__global__ void __launch_bounds__(256) finalize_kernel(const __grid_constant__ ScoreArgs A) {
  pdl_trigger();
  pdl_wait();
  const int64_t vq = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nq_live = MODE == MODE_EDGE ? edge_active_queries(A) : (A.qcount ? (int64_t)*A.qcount : A.nq);
  if (MODE == MODE_EDGE) {
    if ((vq & ~(int64_t)31) >= nq_live) return;  // warp-uniform
  } else if (vq >= nq_live) {
    return;
  }
  double f = 0.0;
  if (vq < nq_live)
    for (int s = 0; s < A.n_splits; ++s) f += A.partial[(int64_t)s * A.nq + vq];
  const double fm = f / A.denom;
  if (MODE == MODE_POS || MODE == MODE_JOINT) {
    const int64_t bq = batch_query(A, vq);
    if (A.score64) A.score64[bq] = fm;
    if (A.score) A.score[bq] = (float)fm;
    if (A.label) A.label[bq] = fm > 0.0 ? 1 : -1;
    maybe_refine(A, vq, fm);
  } else {
    edge_vote(A, vq, fm);
  }
}

// The same for many splits (> kSeqSplits): a CTA of 8 warps owns 32 consecutive queries;
// warp w adds the w-th contiguous eighth of the splits in order, then warp 0 adds the 8
// group sums in order — a fixed order (deterministic), 8x shorter dependency chains and
// 8x more CTAs than the sequential kernel, which left a 4,096-query batch against 20k
// supports (313 splits) 38 us in its finalize.
constexpr int kSeqSplits = 16;
template <int MODE>
__global__ void __launch_bounds__(256) finalize_grouped_kernel(const __grid_constant__ ScoreArgs A) {
  __shared__ double part[8][32];
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t vq = (int64_t)blockIdx.x * 32 + lane;
  const int64_t nq_live = MODE == MODE_EDGE ? edge_active_queries(A) : (A.qcount ? (int64_t)*A.qcount : A.nq);
  if ((int64_t)blockIdx.x * 32 >= nq_live) return;  // CTA-uniform
  const int per = (A.n_splits + 7) / 8;
  const int s0 = w * per, s1 = min(A.n_splits, s0 + per);
  double f = 0.0;
  if (vq < nq_live)
    for (int sp = s0; sp < s1; ++sp) f += A.partial[(int64_t)sp * A.nq + vq];
  part[w][lane] = f;
  __syncthreads();
  if (w != 0) return;
  f = part[0][lane];
#pragma unroll
  for (int g = 1; g < 8; ++g) f += part[g][lane];
  const double fm = f / A.denom;
  if (MODE == MODE_POS || MODE == MODE_JOINT) {
    if (vq < nq_live) {
      const int64_t bq = batch_query(A, vq);
      if (A.score64) A.score64[bq] = fm;
      if (A.score) A.score[bq] = (float)fm;
      if (A.label) A.label[bq] = fm > 0.0 ? 1 : -1;
      maybe_refine(A, vq, fm);
    }
  } else {
    edge_vote(A, vq, fm);
  }
}

// ---------------------------------------------------------------------------------
// small batches (nq <= kSmallQ): support-parallel scoring
// ---------------------------------------------------------------------------------
// The tile kernel gives every CTA 128*QT query slots, so a planner asking for one
// configuration would run 512 slots per CTA for one live query. Here each thread owns
// supports (grid-stride), the <= 32 queries sit in shared memory, and every thread keeps
// one fp64 partial per query; the CTA reduces them in a fixed order, and the last CTA to
// finish (ticket counter) adds the CTA partials in CTA order: one launch, deterministic.
// Terms, lane sums and fp64 accumulation are those of K2 (same tolerance).
constexpr int kSmallQ = 32;
constexpr int kSmallNT = 256;
constexpr int kSmallChunk = 32;  // CTA partials fetched per round by the last CTA
constexpr int64_t kSmallOneCtaTerms = 32768;  // nq * ns * M up to which one CTA scores the batch

// FUSED_FK: the queries arrive as configurations and thread q runs the D-H chain of
// query q (fk_chain, the FK kernel's arithmetic and rounding: the same positions), so a
// small fastron_query is one launch.
template <int MP, int KIND, bool FUSED_FK>
__global__ void __launch_bounds__(kSmallNT) score_small_kernel(const __grid_constant__ ScoreArgs A,
                                                               const __grid_constant__ FkParams P, int64_t ns,
                                                               unsigned int* __restrict__ ticket) {
  constexpr int NP = MP / 2;
  constexpr int64_t TF = tile_floats(MP);
  __shared__ f2 sq[kSmallQ][NP][3];
  __shared__ double s_red[kSmallNT / 32][kSmallQ];
  __shared__ double s_fin[kSmallChunk][kSmallQ];
  __shared__ float s_pos[FUSED_FK ? kSmallQ : 1][FUSED_FK ? MP : 1][3];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_trigger();
  pdl_wait();
  const int nq = (int)A.nq;
  if (FUSED_FK) {
    // the thread's first support record travels to L1 while the D-H chains run
    const int64_t sup0 = (int64_t)blockIdx.x * kSmallNT + tid;
    if (sup0 < ns) {
      const float* r0 = A.packed + (sup0 / kTileSupports) * TF + (sup0 % kTileSupports) * NP * 8;
#pragma unroll
      for (int p = 0; p < NP; ++p) asm volatile("prefetch.global.L1 [%0];" ::"l"(r0 + p * 8));
    }
    if (tid < nq) {
      const float* qk = A.qcfg + (int64_t)tid * A.ldqc;
      fk_chain(
          P, [&](int j) { return (double)__ldg(qk + j); },
          [&](int m, double x, double y, double z) {
            s_pos[tid][m][0] = __double2float_rn(x);
            s_pos[tid][m][1] = __double2float_rn(y);
            s_pos[tid][m][2] = __double2float_rn(z);
          });
    }
    __syncthreads();
  }
  for (int i = tid; i < nq * NP; i += kSmallNT) {  // queries -> scaled pairs (padded point: 0)
    const int q = i / NP, p = i % NP;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (FUSED_FK) {
      if (2 * p < A.M) a = make_float4(s_pos[q][2 * p][0], s_pos[q][2 * p][1], s_pos[q][2 * p][2], 0.f);
      if (2 * p + 1 < A.M) b = make_float4(s_pos[q][2 * p + 1][0], s_pos[q][2 * p + 1][1], s_pos[q][2 * p + 1][2], 0.f);
    } else {
      if (2 * p < A.M) a = __ldg(A.qpos + (int64_t)(2 * p) * A.ldq + q);
      if (2 * p + 1 < A.M) b = __ldg(A.qpos + (int64_t)(2 * p + 1) * A.ldq + q);
    }
    sq[q][p][0] = pk(__fmul_rn(a.x, A.scale), __fmul_rn(b.x, A.scale));
    sq[q][p][1] = pk(__fmul_rn(a.y, A.scale), __fmul_rn(b.y, A.scale));
    sq[q][p][2] = pk(__fmul_rn(a.z, A.scale), __fmul_rn(b.z, A.scale));
  }
  __syncthreads();
  double f[kSmallQ];
#pragma unroll
  for (int q = 0; q < kSmallQ; ++q) f[q] = 0.0;
  constexpr float OFF = rq_lane_offset<KIND, NP>();  // as in score_kernel
  const f2 lane0 = OFF != 0.0f ? pk(-OFF, -OFF) : 0ull;
  double asum = 0.0;
  for (int64_t sup = (int64_t)blockIdx.x * kSmallNT + tid; sup < ns; sup += (int64_t)gridDim.x * kSmallNT) {
    const float* T = A.packed + (sup / kTileSupports) * TF;
    const float* rec = T + (sup % kTileSupports) * NP * 8;
    const double a = reinterpret_cast<const double*>(T + tile_record_floats(MP))[sup % kTileSupports];
    if (OFF != 0.0f) asum += a;
    f2 vx[NP], vy[NP], vz[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float4 xy = __ldg(reinterpret_cast<const float4*>(rec + p * 8));
      const float2 zz = __ldg(reinterpret_cast<const float2*>(rec + p * 8 + 4));
      vx[p] = pk(xy.x, xy.y);
      vy[p] = pk(xy.z, xy.w);
      vz[p] = pk(zz.x, zz.y);
    }
#pragma unroll
    for (int q = 0; q < kSmallQ; ++q) {
      if (q < nq) {  // uniform
        f2 acc;
#pragma unroll
        for (int p = 0; p < NP; ++p)
          accum_term<KIND>(acc, sub2(sq[q][p][0], vx[p]), sub2(sq[q][p][1], vy[p]), sub2(sq[q][p][2], vz[p]), p == 0,
                           lane0);
        if (KIND == kRQPrecise) {  // offset lanes can be negative
          f[q] = fma(a, rq_lane_to_f64(lo(acc)), f[q]);
          f[q] = fma(a, rq_lane_to_f64(hi(acc)), f[q]);
        } else {
          f[q] = fma(a, nonneg_f32_to_f64(lo(acc)), f[q]);
          f[q] = fma(a, nonneg_f32_to_f64(hi(acc)), f[q]);
        }
      }
    }
  }
  if (OFF != 0.0f) {
#pragma unroll
    for (int q = 0; q < kSmallQ; ++q) f[q] = fma(2.0 * (double)OFF, asum, f[q]);
  }
#pragma unroll
  for (int q = 0; q < kSmallQ; ++q) {
    if (q < nq) {
      double v = f[q];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
      if (lane == 0) s_red[warp][q] = v;
    }
  }
  __syncthreads();
  if (tid < nq) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kSmallNT / 32; ++w) v += s_red[w][tid];
    if (gridDim.x == 1) {
      write_score(A, tid, 0.0 + v);  // the multi-CTA path's sum over one partial, same bits
      return;
    }
    A.partial[(int64_t)blockIdx.x * kSmallQ + tid] = v;
  }
  if (gridDim.x == 1) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last CTA adds the CTA partials in CTA order; all its threads fetch a chunk of them at
  // once into shared memory first (one L2 round trip per 64 CTAs instead of one per CTA on
  // a serial chain: 1 query x 20k supports, 79 CTAs: 18.3 us before), same order, same bits
  double v = 0.0;
  for (unsigned c0 = 0; c0 < gridDim.x; c0 += kSmallChunk) {
    const unsigned cn = min((unsigned)kSmallChunk, gridDim.x - c0);
    for (unsigned i = tid; i < cn * kSmallQ; i += kSmallNT)
      s_fin[i / kSmallQ][i % kSmallQ] = __ldcg(A.partial + (int64_t)(c0 + i / kSmallQ) * kSmallQ + i % kSmallQ);
    __syncthreads();
    if (tid < nq)
      for (unsigned c = 0; c < cn; ++c) v += s_fin[c][tid];
    __syncthreads();
  }
  if (tid < nq) write_score(A, tid, v);
  if (tid == 0) *ticket = 0u;  // reset for the next call on this workspace
}

template <int MP, int KIND, bool FUSED_FK = false>
static cudaError_t run_score_small(const ScoreArgs& A, int64_t ns, cudaStream_t st, const FkParams& P = FkParams{}) {
  // one CTA when the whole batch is a few thousand terms (a planner's single query against
  // a Table-I-size model): no cross-CTA partials, ticket or memset
  const bool one_cta = A.nq * ns * (int64_t)A.M <= kSmallOneCtaTerms;
  const int64_t want = one_cta ? 1 : (ns + kSmallNT - 1) / kSmallNT;
  const int64_t grid = want < 1 ? 1 : (want > device_info().sms ? device_info().sms : want);
  // partials: [grid][kSmallQ] doubles; the ticket counter follows them
  unsigned int* ticket = reinterpret_cast<unsigned int*>(A.partial + (int64_t)device_info().sms * kSmallQ);
  if (grid > 1) {
    cudaError_t e = cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return e;
  }
  g_launches.fetch_add(1);
  return launch_pdl(score_small_kernel<MP, KIND, FUSED_FK>, dim3((unsigned)grid), dim3(kSmallNT), 0, st, A, P, ns,
                    ticket);
}

size_t score_small_bytes() { return (size_t)device_info().sms * kSmallQ * sizeof(double) + 256; }

// ---------------------------------------------------------------------------------
// planning + dispatch
// ---------------------------------------------------------------------------------
// Support splits. Measured on the headline (tools/split_probe.sh): the time falls as the
// per-CTA work shrinks — 2 splits 41.7 ms, 4: 40.9, 8: 40.9, 16: 40.8 — because the
// last partial wave costs about one CTA's work, and the hardware block scheduler balances
// many short CTAs well. The plan therefore aims at ~kTargetWaves waves of CTAs, bounded
// by the tile count and by the fp64 partial buffer (s * nq doubles <= kPartialBudget).
constexpr int64_t kTargetWaves = 32;
constexpr int64_t kPartialBudget = (int64_t)1 << 23;  // doubles (64 MB)

static int64_t split_env() {
  const char* e = getenv("FASTRON_SCORE_SPLITS");  // experiments: force a split count
  return e ? atoll(e) : 0;
}

int score_max_splits(int64_t nq, int64_t ns, int M) {
  const int64_t qblocks = (nq + score_queries_per_cta(M) - 1) / score_queries_per_cta(M);
  const int64_t tiles = n_support_tiles(ns);
  if (qblocks <= 0 || tiles <= 1) return 1;
  const int64_t slots_max = (int64_t)device_info().sms * 4;  // >= any resident-CTA count of K2
  int64_t cap = (kTargetWaves * slots_max + qblocks - 1) / qblocks;
  const int64_t budget = kPartialBudget / (nq > 0 ? nq : 1);
  if (cap > budget) cap = budget;
  const int64_t forced = split_env();
  if (forced > cap) cap = forced;
  if (cap > tiles) cap = tiles;
  return (int)(cap < 1 ? 1 : cap);
}

// The partial region: split partials (or the small kernel's CTA partials), then the RQ
// refinement list (nq int32) and its counter.
static size_t score_partial_core_bytes(int64_t nq, int64_t ns, int M) {
  const int s = score_max_splits(nq, ns, M);
  const size_t tiles = s > 1 ? (size_t)s * (size_t)nq * sizeof(double) : 0;
  const size_t small = (nq > 0 && nq <= kSmallQ && M <= 16) ? score_small_bytes() : 0;
  return ((tiles > small ? tiles : small) + 255) & ~(size_t)255;
}

size_t score_partial_bytes(int64_t nq, int64_t ns, int M) {
  return score_partial_core_bytes(nq, ns, M) + (((size_t)(nq > 0 ? nq : 0) * 4 + 255) & ~(size_t)255) + 256;
}

template <int MP, int KIND, int MODE>
static int score_ctas_per_sm() {
  static std::atomic<int> cached[kMaxDevices];
  const int dev = device_slot();
  int v = cached[dev].load();
  if (v == 0) {
    const size_t smem = 128 + kStages * tile_bytes(MP);
    int n = 0;
    cudaFuncSetAttribute(score_kernel<MP, KIND, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, score_kernel<MP, KIND, MODE>, kNT, smem);
    v = n > 0 ? n : 1;
    cached[dev].store(v);
  }
  return v;
}

// Largest batch scored with one query per thread (QT = 1), measured per M:
// M = 8: 2,048; M = 16: 512; M <= 4: 16,384 (cfg1, 10k x 1k: 28.2 -> 26.6 us as a graph
// replay of FK + score; the 128 of round 1 was never measured). FASTRON_ONEQ_MAX (env)
// overrides all three for experiments.
#ifndef FASTRON_ONEQ_MAX4
#define FASTRON_ONEQ_MAX4 16384
#endif
static int64_t oneq_max(int mp) {
  if (const char* e = getenv("FASTRON_ONEQ_MAX")) return atoll(e);  // experiments
  return mp <= 4 ? FASTRON_ONEQ_MAX4 : mp <= 8 ? 2048 : 512;
}

static ScorePlan make_plan(int64_t nq, int64_t ns, int M, int ctas_per_sm) {
  ScorePlan p;
  const int qpc = score_queries_per_cta(M);
  p.n_qblocks = (nq + qpc - 1) / qpc;
  p.n_tiles = n_support_tiles(ns);
  const int64_t slots = (int64_t)device_info().sms * ctas_per_sm;
  const int max_s = score_max_splits(nq, ns, M);
  // the smallest split count reaching ~kTargetWaves waves (capped by max_s), moved to a
  // count whose splits are all non-empty
  int64_t want = p.n_qblocks > 0 ? (kTargetWaves * slots + p.n_qblocks - 1) / p.n_qblocks : 1;
  if (const int64_t forced = split_env()) want = forced;
  if (want > max_s) want = max_s;
  if (want < 1) want = 1;
  int best = (int)want;
  for (int s = (int)want; s >= 1; --s) {
    const int64_t tps = (p.n_tiles + s - 1) / s;
    const int64_t s_eff = tps > 0 ? (p.n_tiles + tps - 1) / tps : 1;
    if (s_eff == s) { best = s; break; }
  }
  p.n_splits = best;
  p.tiles_per_split = (int32_t)(p.n_tiles > 0 ? (p.n_tiles + best - 1) / best : 0);
  return p;
}

template <int MP, int KIND, int MODE>
static cudaError_t run_score(const ScoreArgs& base, const FkParams& P, int64_t nq, int64_t ns, cudaStream_t st) {
  // the split count (and so the fp64 summation order) follows the whole batch: a chunk of
  // a larger batch is planned like the batch, so chunked and single-launch scores agree
  // bit for bit
  ScorePlan plan = make_plan(base.plan_nq > nq ? base.plan_nq : nq, ns, base.M, score_ctas_per_sm<MP, KIND, MODE>());
  plan.n_qblocks = (nq + score_queries_per_cta(base.M) - 1) / score_queries_per_cta(base.M);
  ScoreArgs A = base;
  A.n_tiles = plan.n_tiles;
  A.n_splits = plan.n_splits;
  A.tiles_per_split = plan.tiles_per_split;
  const size_t smem = 128 + kStages * tile_bytes(MP);
  // one query per thread up to a batch size measured per M (A/B, 20k supports, same bits):
  // M = 8 up to 2,048 queries (512: 58 -> 46 us, 1,024: 73 -> 68, 2,048: 118 -> 113; 4,096
  // slower), M = 16 up to 512 (256: 66 -> 58 us, 512: 97 -> 82; 1,024 slower)
  const bool one_q = MODE != MODE_EDGE && nq <= oneq_max(MP) && qt_for(MP) > 1;
  if (one_q) plan.n_qblocks = (nq + kNT - 1) / kNT;
  const int64_t grid = plan.n_qblocks * plan.n_splits;
  if (grid > 0x7fffffff) return cudaErrorInvalidValue;
  if (one_q) {
    static std::atomic<int> attr[kMaxDevices];
    const int dev = device_slot();
    if (!attr[dev].load()) {
      cudaFuncSetAttribute(score_kernel<MP, KIND, MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr[dev].store(1);
    }
  }
  cudaError_t e;
  if (one_q) {
    e = launch_pdl(score_kernel<MP, KIND, MODE, 1>, dim3((unsigned)grid), dim3(kNT), smem, st, A, P);
  } else {
    e = launch_pdl(score_kernel<MP, KIND, MODE>, dim3((unsigned)grid), dim3(kNT), smem, st, A, P);
  }
  g_launches.fetch_add(1);
  if (e != cudaSuccess || plan.n_splits == 1) return e;
  if (plan.n_splits > kSeqSplits) {
    e = launch_pdl(finalize_grouped_kernel<MODE>, dim3((unsigned)((nq + 31) / 32)), dim3(256), 0, st, A);
  } else {
    e = launch_pdl(finalize_kernel<MODE>, dim3((unsigned)((nq + 255) / 256)), dim3(256), 0, st, A);
  }
  g_launches.fetch_add(1);
  return e;
}

template <int MODE>
static cudaError_t dispatch(const ScoreArgs& A, const FkParams& P, int64_t nq, int64_t ns, int kind, cudaStream_t st) {
  const int MP = padded_m(A.M);
  // kind: kGaussian, kRQ (fast) or, for MODE_POS only, kRQPrecise (refinement pass 2)
#define FASTRON_CASE(mp)                                                                   \
  case mp:                                                                                 \
    if (MODE == MODE_POS && kind == kRQPrecise) return run_score<mp, kRQPrecise, MODE_POS>(A, P, nq, ns, st); \
    return kind == kGaussian ? run_score<mp, kGaussian, MODE>(A, P, nq, ns, st)            \
                             : run_score<mp, kRQ, MODE>(A, P, nq, ns, st);
  switch (MP) {
    FASTRON_CASE(2)
    FASTRON_CASE(4)
    FASTRON_CASE(6)
    FASTRON_CASE(8)
    FASTRON_CASE(10)
    FASTRON_CASE(12)
    FASTRON_CASE(14)
    FASTRON_CASE(16)
    FASTRON_CASE(18)
    FASTRON_CASE(20)
    FASTRON_CASE(22)
    FASTRON_CASE(24)
    FASTRON_CASE(26)
    FASTRON_CASE(28)
    FASTRON_CASE(30)
    FASTRON_CASE(32)
    default:
      return cudaErrorInvalidValue;
  }
#undef FASTRON_CASE
}

// joint vectors [n][ldx] (D dims) -> pseudo points float4 [ceil(D/3)][n], zero padded
__global__ void joint_points_kernel(const float* __restrict__ x, int64_t n, int64_t ldx, int D, float4* __restrict__ out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const float* xk = x + k * ldx;
  const int Mj = (D + 2) / 3;
  for (int m = 0; m < Mj; ++m) {
    const int d = 3 * m;
    out[(int64_t)m * n + k] = make_float4(__ldg(xk + d), d + 1 < D ? __ldg(xk + d + 1) : 0.0f,
                                          d + 2 < D ? __ldg(xk + d + 2) : 0.0f, 0.0f);
  }
}

int joint_points(int D) { return (D + 2) / 3; }

cudaError_t launch_joint_points(const float* x, int64_t n, int64_t ldx, int D, float4* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  joint_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, n, ldx, D, out);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

cudaError_t launch_score_joint(const float4* qpts, int64_t nq, const float* packed, int64_t ns, int D, int kind,
                               float scale, float* score, int8_t* label, double* partial, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  ScoreArgs A = {};
  A.qpos = qpts;
  A.ldq = nq;
  A.nq = nq;
  A.packed = packed;
  A.M = joint_points(D);
  A.scale = scale;
  A.score = score;
  A.label = label;
  A.partial = partial;
  A.denom = 1.0;
  FkParams P = {};
  const int MP = padded_m(A.M);
  switch (MP) {
    case 2:
      return kind == kGaussian ? run_score<2, kGaussian, MODE_JOINT>(A, P, nq, ns, st)
                               : run_score<2, kRQ, MODE_JOINT>(A, P, nq, ns, st);
    case 4:
      return kind == kGaussian ? run_score<4, kGaussian, MODE_JOINT>(A, P, nq, ns, st)
                               : run_score<4, kRQ, MODE_JOINT>(A, P, nq, ns, st);
    case 6:
      return kind == kGaussian ? run_score<6, kGaussian, MODE_JOINT>(A, P, nq, ns, st)
                               : run_score<6, kRQ, MODE_JOINT>(A, P, nq, ns, st);
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_score(const float4* qpos, int64_t nq, int64_t ldq, const float* packed, int64_t ns, int M, int kind,
                         float scale, float* score, int8_t* label, double* partial, cudaStream_t st,
                         double* score64, int64_t plan_nq) {
  if (nq <= 0) return cudaSuccess;
  ScoreArgs A = {};
  A.plan_nq = plan_nq;
  A.score64 = score64;
  A.qpos = qpos;
  A.ldq = ldq;
  A.nq = nq;
  A.packed = packed;
  A.M = M;
  A.scale = scale;
  A.score = score;
  A.label = label;
  A.partial = partial;
  A.denom = (double)M;
  FkParams P = {};
  // a small batch (planned as a whole) takes the support-parallel kernel
  const int64_t batch = plan_nq > nq ? plan_nq : nq;
  if (batch <= kSmallQ && ns > 0 && M <= 16 && partial) {
    switch (padded_m(M)) {
#define FASTRON_SCASE(mp)                                                                            \
  case mp:                                                                                           \
    return kind == kGaussian ? run_score_small<mp, kGaussian>(A, ns, st) : run_score_small<mp, kRQPrecise>(A, ns, st);
      FASTRON_SCASE(2)
      FASTRON_SCASE(4)
      FASTRON_SCASE(6)
      FASTRON_SCASE(8)
      FASTRON_SCASE(10)
      FASTRON_SCASE(12)
      FASTRON_SCASE(14)
      FASTRON_SCASE(16)
#undef FASTRON_SCASE
      default:
        break;
    }
  }
  if (kind == kRQ && ns > 0 && partial) {
    // RQ in two passes: the fast term for every query, then the precise
    // (Newton + offset lanes) term for the queries whose fast score lies within
    // kRefineTau of 0 — found by pass 1's epilogue, scored by pass 2 over a worst-case grid
    // whose CTAs beyond the device-side count exit at once (no host synchronisation)
    // (laid out for this call's nq: a chunk of a larger batch gets a region sized for the
    // chunk capacity, and core(nq) + list(nq) is monotone in nq)
    char* region = reinterpret_cast<char*>(partial) + score_partial_core_bytes(nq, ns, M);
    int32_t* list = reinterpret_cast<int32_t*>(region);
    int32_t* count = reinterpret_cast<int32_t*>(region + (((size_t)nq * 4 + 255) & ~(size_t)255));
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    ScoreArgs A1 = A;
    A1.refine_list = list;
    A1.refine_count = count;
    A1.refine_tau = kRefineTau;
    e = dispatch<MODE_POS>(A1, P, nq, ns, kRQ, st);
    if (e != cudaSuccess) return e;
    ScoreArgs A2 = A;
    A2.qidx = list;
    A2.qcount = count;
    return dispatch<MODE_POS>(A2, P, nq, ns, kRQPrecise, st);
  }
  return dispatch<MODE_POS>(A, P, nq, ns, kind, st);
}

bool query_small_ok(int64_t nq, int64_t ns, int M) { return nq > 0 && nq <= kSmallQ && ns > 0 && M <= 16; }

cudaError_t launch_query_small(const FkParams& P, const float* q, int64_t nq, int64_t ldq, const float* packed,
                               int64_t ns, int M, int kind, float scale, float* score, int8_t* label,
                               double* partial, cudaStream_t st) {
  ScoreArgs A = {};
  A.qcfg = q;
  A.ldqc = ldq;
  A.nq = nq;
  A.packed = packed;
  A.M = M;
  A.scale = scale;
  A.score = score;
  A.label = label;
  A.partial = partial;
  A.denom = (double)M;
  switch (padded_m(M)) {
#define FASTRON_QCASE(mp)                                                                   \
  case mp:                                                                                  \
    return kind == kGaussian ? run_score_small<mp, kGaussian, true>(A, ns, st, P)           \
                             : run_score_small<mp, kRQPrecise, true>(A, ns, st, P);
    FASTRON_QCASE(2)
    FASTRON_QCASE(4)
    FASTRON_QCASE(6)
    FASTRON_QCASE(8)
    FASTRON_QCASE(10)
    FASTRON_QCASE(12)
    FASTRON_QCASE(14)
    FASTRON_QCASE(16)
#undef FASTRON_QCASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_edge_round(const FkParams& P, const EdgeRound& R, const float* packed, int64_t ns, int M, int kind,
                              float scale, double* partial, float4* pos, cudaStream_t st) {
  if (R.n_edges <= 0) return cudaSuccess;
  ScoreArgs A = {};
  A.nq = R.n_edges * 32;
  A.qpos = pos;
  A.ldq = A.nq;
  A.packed = packed;
  A.M = M;
  A.scale = scale;
  A.partial = partial;
  A.qa = R.qa;
  A.qb = R.qb;
  A.ldqe = R.ldq;
  A.n_interp = R.n_interp;
  A.round = R.round;
  A.active = R.active;
  A.active_count = R.active_count;
  A.next_active = R.next_active;
  A.next_count = R.next_count;
  A.in_collision = R.in_collision;
  A.hit_index = R.hit_index;
  A.denom = (double)M;
  g_launches.fetch_add(1);
  cudaError_t e = launch_pdl(edge_fk_kernel, dim3((unsigned)((A.nq + 255) / 256)), dim3(256), 0, st, A, P, pos);
  if (e != cudaSuccess) return e;
  return dispatch<MODE_EDGE>(A, P, A.nq, ns, kind, st);
}

}  // namespace fastron
