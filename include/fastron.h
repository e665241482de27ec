/*
 * fastron.h — C ABI of the B200-native Fastron FK hot path (arXiv 1910.06451,
 * "Forward Kinematics Kernel for Improved Proxy Collision Checking").
 *
 * Library: paper_1910_06451_b200/libfastron_b200.so (hand-written sm_100a CUDA).
 * Citations: PAPER.md:<line> (§, Eq./Alg.) of /root/reference/PAPER.md; readings
 * R<n> are listed in DESIGN.md §3.
 *
 * Conventions for every call
 * --------------------------
 *  - Pointers are DEVICE pointers unless the argument says "host" (or "host or
 *    device" for fastron_query). The caller owns every buffer; the library never
 *    allocates or frees caller memory and keeps no state besides a per-device cache
 *    of cudaDeviceProp/occupancy. Scratch memory is passed in through `workspace`.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls enqueue work on it and return without synchronising (except where noted);
 *    asynchronous device faults surface at the caller's next synchronisation.
 *  - Host-checkable argument errors return FASTRON_ERR_INVALID_ARG before any launch:
 *    null pointers with a non-zero size, negative sizes, leading dimensions smaller
 *    than the row length, gamma <= 0 or non-finite, unknown kernel kind, dof outside
 *    [1,16], n_cp outside [1,32], cp_frame outside [0,dof], non-finite robot data,
 *    beta < 1, n_interp < 1. A short workspace returns FASTRON_ERR_WORKSPACE. A
 *    CUDA launch/runtime failure returns FASTRON_ERR_CUDA. fastron_last_error()
 *    returns a thread-local message for the last non-OK status of the calling thread.
 *  - Device array CONTENTS (NaN joint values, labels outside {-1,+1}) are not
 *    checked on the hot path. With validation on (fastron_set_validation(1), or the
 *    environment variable FASTRON_VALIDATE=1 at the first call) every entry point
 *    first counts non-finite values in its float inputs and labels outside {-1,+1},
 *    synchronising `stream` to read the count, and returns FASTRON_ERR_INVALID_ARG if
 *    any is found (SURVEY §8(b) conventions). A debugging aid, off by default.
 *  - There is no CPU fallback: every computation runs in this library's kernels.
 *
 * Data layouts
 * ------------
 *  Configurations q: row-major float [n][ldq], columns 0..dof-1 used.
 *  Control-point positions: SoA float4 [n_cp][ldpos] = (x, y, z, 0) in metres,
 *    i.e. element (m, k) at pos + 4*(m*ldpos + k) (Eq. 2).
 *  Gram matrix: row-major float [n][ldk].
 */
#ifndef FASTRON_H_
#define FASTRON_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FASTRON_MAX_DOF 16
#define FASTRON_MAX_CP 32

typedef enum {
  FASTRON_OK = 0,
  FASTRON_ERR_INVALID_ARG = 1,
  FASTRON_ERR_CUDA = 2,
  FASTRON_ERR_WORKSPACE = 3,
  FASTRON_ERR_UNSUPPORTED = 4
} fastron_status;

/* Shape of the per-control-point RBF term (R1/R2). Both are combined by
 * the 1/M mean of Eq. 4, so k(x, x) = 1 for both. */
typedef enum {
  FASTRON_RBF_GAUSSIAN = 0, /* exp(-gamma d^2): BASELINE.json north_star term (headline)  */
  FASTRON_RBF_RQ = 1        /* (1 + gamma/2 d^2)^-2: Eq. 3               */
} fastron_rbf;

typedef struct {
  int32_t kind; /* fastron_rbf */
  float gamma;  /* > 0 and finite */
} fastron_kernel;

/* Serial manipulator in the standard D-H convention with its
 * control points. Host struct; copied by value into kernel parameters. */
typedef struct {
  int32_t dof;                  /* D in [1, 16]; all joints revolute (R6)             */
  int32_t n_cp;                 /* M in [1, 32]                                        */
  float dh[FASTRON_MAX_DOF][4]; /* per joint: theta_offset, d, a, alpha (Eq. 1);
                                   theta_i = q_i + theta_offset_i                     */
  float base[3][4];             /* wA_0 as a row-major 3x4 affine       */
  int32_t cp_frame[FASTRON_MAX_CP];     /* j_m in [0, D]: 0 = base frame, i = frame
                                           after joint i (Eq. 2)                       */
  float cp_offset[FASTRON_MAX_CP][3];   /* translation of the static T_m in frame j_m
                                           (T_m = I <=> 0)               */
} fastron_robot;

typedef struct {
  int64_t iterations; /* add/adjust + remove steps taken (R10)                      */
  int64_t n_add;      /* add/adjust steps (Eq. 6-8)                                  */
  int64_t n_remove;   /* redundant-support removals (Alg. 1 lines PAPER.md:235-239) */
  int32_t converged;  /* 1 iff min_i y_i F_i > 0 at exit (Claim 2)     */
  int32_t n_support;  /* |S| = count(alpha != 0) after removeNonsupportPoints         */
} fastron_train_result;

/*
 * fastron_fk — batched forward kinematics, Eq. 1-2.
 * For k < n: theta_i = q[k*ldq + i] + theta_offset_i, wA_i = wA_0 0A_1 ... (i-1)A_i,
 * pos(m, k) = pos(wA_{j_m} T_m). Arithmetic is fp64 inside (sincos, chain), rounded
 * once to fp32 on store. One thread per configuration.
 *   robot: host. q: device float [n][ldq], ldq >= dof. pos: device float4 [n_cp][ldpos],
 *   ldpos >= n, 16-byte aligned. n == 0 is a no-op.
 */
fastron_status fastron_fk(const fastron_robot* robot, const float* q, int64_t n, int64_t ldq, float* pos,
                          int64_t ldpos, void* stream);

/*
 * fastron_score — Fastron model evaluation f(x) = sum_i K_FK(S_i, x) alpha_i and its
 * sign, K_FK of Eq. 4 with the term of k.kind.
 *   qpos: device float4 [n_cp][ldq] query control points (from fastron_fk), ldq >= nq,
 *   16-byte aligned (as spos).
 *   spos: device float4 [n_cp][lds] support control points, lds >= ns. alpha: device float [ns].
 *   score: device float [nq] (nullable): f rounded to fp32 (accumulated in fp64).
 *   label: device int8 [nq] (nullable): +1 iff f > 0 else -1 (R8).
 *   workspace: device scratch of >= fastron_score_workspace_bytes(nq, ns, n_cp) bytes,
 *   256-byte aligned; contents are overwritten.
 * ns == 0 gives f = 0, label -1. nq == 0 is a no-op.
 * Results are deterministic (fixed-order reductions) for a given device and batch size;
 * the fp64 summation order follows the batch: nq <= 32 (n_cp <= 16) runs a
 * support-parallel kernel, larger batches split the supports over a number of CTAs
 * chosen from nq, so the same query may differ in the last fp32 bit between batches of
 * different sizes (always within the tolerance of DESIGN.md R16). The workspace also
 * carries a completion counter: one call at a time per workspace.
 */
size_t fastron_score_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp);
fastron_status fastron_score(const float* qpos, int64_t nq, int64_t ldq, const float* spos, const float* alpha,
                             int64_t ns, int64_t lds, int32_t n_cp, fastron_kernel k, float* score, int8_t* label,
                             void* workspace, size_t workspace_bytes, void* stream);

/*
 * fastron_model_pack / fastron_score_packed — the same evaluation as fastron_score, split
 * so that a model (support positions + alpha, "support set") is packed once
 * per model update and then scored against many query batches.
 *   fastron_model_pack: spos/alpha as fastron_score; packed: device buffer of
 *   fastron_model_bytes(ns, n_cp) bytes, 256-byte aligned, holding the supports
 *   pre-scaled for kernel k (its contents are only meaningful to fastron_score_packed
 *   with the same ns, n_cp and k).
 *   fastron_score_packed: qpos/score/label as fastron_score (qpos 16-byte aligned);
 *   packed as written by fastron_model_pack (256-byte aligned, checked); workspace >=
 *   fastron_score_packed_workspace_bytes(nq, ns, n_cp) (may be 0 bytes), 256-byte aligned
 *   when non-empty (checked: misaligned buffers return INVALID_ARG, never a fault).
 */
size_t fastron_model_bytes(int64_t ns, int32_t n_cp);
/* fastron_score_packed_f64: the same scores in fp64 (before the fp32 rounding). score64:
 * device double [nq]. (The packed alpha is fp32 and the sums follow the scoring order, so
 * these are NOT the margins F = K alpha of Algorithm 1: use fastron_kernel_matvec or
 * fastron_kernel_matvec_lazy for a warm start.) */
fastron_status fastron_score_packed_f64(const float* qpos, int64_t nq, int64_t ldq, const void* packed, int64_t ns,
                                        int32_t n_cp, fastron_kernel k, double* score64, void* workspace,
                                        size_t workspace_bytes, void* stream);
fastron_status fastron_model_pack(const float* spos, const float* alpha, int64_t ns, int64_t lds, int32_t n_cp,
                                  fastron_kernel k, void* packed, size_t packed_bytes, void* stream);
size_t fastron_score_packed_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp);
fastron_status fastron_score_packed(const float* qpos, int64_t nq, int64_t ldq, const void* packed, int64_t ns,
                                    int32_t n_cp, fastron_kernel k, float* score, int8_t* label, void* workspace,
                                    size_t workspace_bytes, void* stream);

/*
 * fastron_gram — FK-kernel Gram matrix K_ij = K_FK(X_i, X_j),
 * written in full (both triangles; computed once per unordered pair and mirrored,
 * so K is exactly symmetric), K_ii = 1 exactly. For n_cp a power of two the values are
 * bit-identical to fastron_score with alpha = e_i.
 *   pos: device float4 [n_cp][ldp], ldp >= n. K: device float [n][ldk], ldk >= n.
 *   workspace: >= fastron_gram_workspace_bytes(n, n_cp).
 */
size_t fastron_gram_workspace_bytes(int64_t n, int32_t n_cp);
fastron_status fastron_gram(const float* pos, int64_t n, int64_t ldp, int32_t n_cp, fastron_kernel k, float* K,
                            int64_t ldk, void* workspace, size_t workspace_bytes, void* stream);

/*
 * fastron_train — Algorithm 1, "Fastron Model Update Algorithm" (PAPER.md:206-252,
 * Eq. 6-9), run entirely on the device in one persistent cluster kernel (one CTA up to
 * 2,048 points; above, a cluster of ~n/1024 CTAs up to 16, chosen by the library).
 *   K: device float [n][ldk] Gram (from fastron_gram; promoted to fp64 on read).
 *   y: device int8 [n], +1 = C_obs, -1 = C_free.
 *   beta >= 1: conditional bias, b_i = beta^(0.5 (y_i + 1)).
 *   iter_max >= 0, s_max >= 0.
 *   alpha_inout, F_inout: device double [n]; on entry the previous model
 *     (loadPreviousModel; zeros = cold start; F must equal K alpha),
 *     on exit the updated alpha and F.
 *   support_idx: device int32 [n] (nullable): ascending indices with alpha != 0
 *     (removeNonsupportPoints); result->n_support entries are valid.
 *   trace: device int32 [iter_max] (nullable): i for an add/adjust of i, -(i+1) for a
 *     removal of i, one entry per iteration.
 *   result: device fastron_train_result.
 * Ties in argmin/argmax go to the lowest index (R9); an iteration is one add/adjust
 * or remove (R10); non-convergence is reported in result->converged, not as an error.
 * All alpha/F arithmetic is fp64 with separately rounded multiply and add, so the
 * trace is bit-identical to the oracle's on the same K (R13).
 * n <= fastron_train_max_n() (state is held on chip); larger n returns ERR_UNSUPPORTED.
 */
int64_t fastron_train_max_n(void);
fastron_status fastron_train(const float* K, int64_t n, int64_t ldk, const int8_t* y, double beta, int64_t iter_max,
                             int64_t s_max, double* alpha_inout, double* F_inout, int32_t* support_idx,
                             int32_t* trace, fastron_train_result* result, void* stream);

/*
 * fastron_train_lazy — Algorithm 1 with lazy kernel-matrix columns ("a column
 * of K can be computed and stored only when needed", :225 computeKernelMatrixColumn):
 * no Gram matrix is formed. The column of the selected index is computed inside the
 * persistent cluster kernel from the pre-scaled training points (held in shared memory,
 * or — for slices beyond the shared-memory budget, e.g. n = 20,000 at n_cp = 16 — in an
 * L2-resident part of the workspace) and stored in a column cache of cache_cols columns;
 * later steps on the same index
 * read it back. Columns are bit-identical to fastron_gram's, so the result equals
 * fastron_train(fastron_gram(pos)) exactly.
 *   pos: device float4 [n_cp][ldp] control points of the n training configurations;
 *   k: the FK-kernel term; n_cp <= 16 (odd n_cp padded as in fastron_score);
 *   y, beta, iter_max, s_max, alpha_inout, F_inout, support_idx, trace, result: as
 *   fastron_train. cache_cols >= 0 (columns beyond the cache are recomputed).
 *   workspace: >= fastron_train_lazy_workspace_bytes(n, n_cp, cache_cols).
 * n <= fastron_train_lazy_max_n(n_cp) (32,768: 16 CTAs x 2,048 slots), else
 * FASTRON_ERR_UNSUPPORTED.
 */
int64_t fastron_train_lazy_max_n(int32_t n_cp);
size_t fastron_train_lazy_workspace_bytes(int64_t n, int32_t n_cp, int64_t cache_cols);
fastron_status fastron_train_lazy(const float* pos, int64_t n, int64_t ldp, int32_t n_cp, fastron_kernel k,
                                  const int8_t* y, double beta, int64_t iter_max, int64_t s_max,
                                  double* alpha_inout, double* F_inout, int32_t* support_idx, int32_t* trace,
                                  fastron_train_result* result, int64_t cache_cols, void* workspace,
                                  size_t workspace_bytes, void* stream);

/*
 * Model-update cycle (PAPER.md:272, "two-stage active learning"; :219 loadPreviousModel).
 *
 * fastron_active_samples — stage 1: n_near samples around each of the ns support points,
 *   clamp(S_i + sigma * z, lo, hi); stage 2: n_uniform samples lo + u (hi - lo). The random
 *   numbers are inputs: z device float [ns*n_near][dof] ~ N(0,1), u device float
 *   [n_uniform][dof] ~ U[0,1). sigma, lo, hi: device float [dof]. out: device float
 *   [ns*n_near + n_uniform][ldo], stage-1 rows first (support-major), ldo >= dof.
 * fastron_label_capsules — the geometric check that labels samples and re-labels supports
 *   (the paper uses FCL; here capsules vs axis-aligned boxes, R12): capsules of
 *   `radius` on the segments between consecutive entries of chain (host int32 [n_chain],
 *   control-point indices, -1 = the base origin), boxes host double [n_cubes][6] (lo xyz,
 *   hi xyz), n_cubes <= 64, n_chain <= 33. pos: device float4 [n_cp][ldp]. label: device
 *   int8 [n], +1 iff any capsule touches any box (tangency counts).
 * fastron_kernel_matvec — F = K alpha (fp64, index order over alpha != 0), the margin
 *   vector a warm start needs when the dataset changed around a loaded alpha.
 * fastron_kernel_matvec_lazy — the same F = K alpha for the lazy Algorithm 1, without the
 *   Gram: every K entry is computed from the control points pos (device float4
 *   [n_cp][ldp], ldp >= n) exactly as fastron_gram computes it, so F equals
 *   fastron_kernel_matvec(fastron_gram(pos), alpha) bit for bit.
 *   alpha, F: device double [n]. workspace (256-byte aligned):
 *   >= fastron_kernel_matvec_lazy_workspace_bytes(n, n_cp). Cost: n x nnz(alpha) entries.
 */
fastron_status fastron_active_samples(const float* S, int64_t ns, int64_t lds, int32_t dof, int32_t n_near,
                                      const float* z, const float* sigma, const float* u, int64_t n_uniform,
                                      const float* lo, const float* hi, float* out, int64_t ldo, void* stream);
fastron_status fastron_label_capsules(const float* pos, int64_t ldp, int64_t n, const int32_t* chain, int32_t n_chain,
                                      const double* boxes, int32_t n_cubes, float radius, int8_t* label, void* stream);
fastron_status fastron_kernel_matvec(const float* K, int64_t n, int64_t ldk, const double* alpha, double* F,
                                     void* stream);
size_t fastron_kernel_matvec_lazy_workspace_bytes(int64_t n, int32_t n_cp);
fastron_status fastron_kernel_matvec_lazy(const float* pos, int64_t n, int64_t ldp, int32_t n_cp, fastron_kernel k,
                                          const double* alpha, double* F, void* workspace, size_t workspace_bytes,
                                          void* stream);

/*
 * fastron_edge_check — discrete motion-planning edge check (BASELINE.json cfg4,
 * SPEC.md:379-387, R11): for edge e and k = 0..n_interp-1,
 * q_k = qa + t_k (qb - qa) with t_k = k / (n_interp - 1) in fp32 (t = 0 if n_interp = 1),
 * each q_k goes through FK (Eq. 1-2) and the Fastron score;
 * in_collision[e] = 1 iff some f(q_k) > 0. Points are visited in rounds of 32 in the
 * order k = 0, 2, 4, ..., then 1, 3, 5, ...; an edge stops after the first round that
 * contains a hit (warp vote).
 *   robot: host. qa, qb: device float [n_edges][ldq]. spos/alpha as fastron_score.
 *   in_collision: device uint8 [n_edges]. hit_index: device int32 [n_edges] (nullable):
 *   the lowest k with f(q_k) > 0 inside the first round that had a hit, else -1.
 *   workspace: >= fastron_edge_workspace_bytes(n_edges, ns, robot->n_cp).
 */
size_t fastron_edge_workspace_bytes(int64_t n_edges, int64_t ns, int32_t n_cp);
/* fastron_edge_check_packed — the same check against a model packed once by
 * fastron_model_pack (e.g. replicated to every GPU by one broadcast of the packed buffer,
 * DESIGN.md §8): the same rounds, the same results. packed: device, 256-byte aligned;
 * n_cp == robot->n_cp. workspace (256-byte aligned):
 * >= fastron_edge_packed_workspace_bytes(n_edges, ns, n_cp). */
size_t fastron_edge_packed_workspace_bytes(int64_t n_edges, int64_t ns, int32_t n_cp);
fastron_status fastron_edge_check_packed(const fastron_robot* robot, const float* qa, const float* qb,
                                         int64_t n_edges, int64_t ldq, int32_t n_interp, const void* packed,
                                         int64_t ns, int32_t n_cp, fastron_kernel k, uint8_t* in_collision,
                                         int32_t* hit_index, void* workspace, size_t workspace_bytes, void* stream);
fastron_status fastron_edge_check(const fastron_robot* robot, const float* qa, const float* qb, int64_t n_edges,
                                  int64_t ldq, int32_t n_interp, const float* spos, const float* alpha, int64_t ns,
                                  int64_t lds, fastron_kernel k, uint8_t* in_collision, int32_t* hit_index,
                                  void* workspace, size_t workspace_bytes, void* stream);

/*
 * fastron_score_joint / fastron_gram_joint — the joint-space RBF kernel of the paper's
 * "Fastron RBF" baseline (Eq. 3, Table I): K(x, x') is ONE RBF term
 * of the joint-vector distance ||x - x'||^2 (no forward kinematics, no mean), with the
 * term of k.kind. Inputs are configurations, not positions.
 *   q: device float [nq][ldq], s: device float [ns][lds], x: device float [n][ldx];
 *   dof in [1, 16] (ldq, lds, ldx >= dof). alpha, score, label, K: as fastron_score /
 *   fastron_gram. workspace: >= the matching *_workspace_bytes (256-byte aligned).
 * fastron_train accepts the resulting K unchanged (the Alg. 1 update is kernel-agnostic).
 */
size_t fastron_score_joint_workspace_bytes(int64_t nq, int64_t ns, int32_t dof);
fastron_status fastron_score_joint(const float* q, int64_t nq, int64_t ldq, const float* s, const float* alpha,
                                   int64_t ns, int64_t lds, int32_t dof, fastron_kernel k, float* score,
                                   int8_t* label, void* workspace, size_t workspace_bytes, void* stream);
size_t fastron_gram_joint_workspace_bytes(int64_t n, int32_t dof);
fastron_status fastron_gram_joint(const float* x, int64_t n, int64_t ldx, int32_t dof, fastron_kernel k, float* K,
                                  int64_t ldk, void* workspace, size_t workspace_bytes, void* stream);

/*
 * fastron_query — the configuration-level proxy collision check, fastron_fk followed
 * by fastron_score on the same stream ("query").
 *   q: float [nq][ldq], HOST (pageable or pinned) or DEVICE. score (nullable) and
 *   label (nullable): HOST or DEVICE. spos/alpha: device, as fastron_score.
 *   When q / score / label are host memory the call streams them in chunks through the
 *   workspace (H2D of chunk c+1 and D2H of chunk c-1, on two library-owned copy
 *   streams, overlap the compute of chunk c on `stream`) and returns after the
 *   results are in host memory (it synchronises `stream`). With device pointers it is
 *   asynchronous like the other calls.
 *   workspace: >= fastron_query_workspace_bytes(nq, ns, robot->n_cp, robot->dof).
 */
size_t fastron_query_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp, int32_t dof);
fastron_status fastron_query(const fastron_robot* robot, const float* q, int64_t nq, int64_t ldq, const float* spos,
                             const float* alpha, int64_t ns, int64_t lds, fastron_kernel k, float* score,
                             int8_t* label, void* workspace, size_t workspace_bytes, void* stream);

/*
 * fastron_query_packed — the proxy collision check of configurations against a model
 * packed once by fastron_model_pack (the planner's call: configurations
 * in, scores and labels out, one API call per batch). DEVICE buffers only (fastron_query
 * streams host buffers). For nq <= 32 (n_cp <= 16) it is one launch of the
 * support-parallel kernel with the D-H chain inside; otherwise fastron_fk +
 * fastron_score_packed on the workspace. Every path gives the bits of fastron_fk +
 * fastron_score_packed on the same batch.
 *   robot: host; n_cp must equal robot->n_cp and the packing's n_cp. q: device float
 *   [nq][ldq], ldq >= dof. packed: device, 256-byte aligned (fastron_model_pack).
 *   score / label: device, nullable (not both). workspace (256-byte aligned):
 *   >= fastron_query_packed_workspace_bytes(nq, ns, n_cp, dof).
 *   Errors: host pointers -> INVALID_ARG.
 */
size_t fastron_query_packed_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp, int32_t dof);
fastron_status fastron_query_packed(const fastron_robot* robot, const float* q, int64_t nq, int64_t ldq,
                                    const void* packed, int64_t ns, int32_t n_cp, fastron_kernel k, float* score,
                                    int8_t* label, void* workspace, size_t workspace_bytes, void* stream);

/*
 * The fp64 path for ill-conditioned models (R25). A model trained by
 * Algorithm 1 has weights of both signs up to ~200, so its score
 * cancels and the fp32 path's rounding (~1e-5..1e-4) can exceed the 1e-5
 * floor near the decision boundary. These calls keep the positions, the weights, every
 * term of Eq. 3/4 and every sum in fp64.
 * fastron_fk64 — fastron_fk with unrounded fp64 positions: pos device double4
 *   [n_cp][ldpos] = (x, y, z, 0), 32-byte aligned, ldpos >= n.
 * fastron_score_precise — f(q) = sum_i alpha_i (1/M) sum_m t_m in fp64 (Gaussian exp, RQ
 *   by division), support order. qpos: double4 [n_cp][ldq] (fastron_fk64), spos: double4
 *   [n_cp][lds], alpha: device double [ns] (e.g. fastron_train's alpha), score: device
 *   double [nq] (nullable), label: int8 [nq] (nullable; +1 iff f > 0). n_cp <= 16 (else
 *   UNSUPPORTED). No workspace. Roughly 10x the fp32 path's time per term.
 */
fastron_status fastron_fk64(const fastron_robot* robot, const float* q, int64_t n, int64_t ldq, double* pos,
                            int64_t ldpos, void* stream);
fastron_status fastron_score_precise(const double* qpos, int64_t nq, int64_t ldq, const double* spos,
                                     const double* alpha, int64_t ns, int64_t lds, int32_t n_cp, fastron_kernel k,
                                     double* score, int8_t* label, void* stream);

/* Thread-local message for the last non-OK status returned on this thread. */
const char* fastron_last_error(void);

/* Library version string and the number of kernel launches issued by this process
 * (a counter for the bench's gpu_launches claim). */
const char* fastron_version(void);
int64_t fastron_launch_count(void);

/* Content validation switch (see Conventions): on != 0 enables it for the process,
 * 0 disables it; fastron_validation() returns the current setting. */
void fastron_set_validation(int32_t on);
int32_t fastron_validation(void);

#ifdef __cplusplus
}
#endif

#endif /* FASTRON_H_ */
