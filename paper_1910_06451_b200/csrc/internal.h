// internal.h — host-side launchers of the sm_100a kernels (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "fk_device.cuh"

namespace fastron {

extern std::atomic<int64_t> g_launches;  // kernels launched by this process (bench gpu_launches)

struct DeviceInfo {
  int device;
  int sms;
  int max_smem_optin;
};
const DeviceInfo& device_info();

// Function attributes and occupancy are per device: kernels keep one cached value per
// device ordinal (0 = not yet computed).
constexpr int kMaxDevices = 64;
inline int device_slot() {
  const int d = device_info().device;
  return d >= 0 && d < kMaxDevices ? d : 0;
}

// Programmatic dependent launch (PDL): the query-path kernels (FK, pack, scoring, finalize,
// edge FK, small batches) are launched with programmatic stream serialisation, so a kernel
// is scheduled while its predecessor drains; each one calls pdl_wait() (griddepcontrol.wait:
// the predecessor has completed and its memory is visible) before its first global-memory
// access and pdl_trigger() at its start. Off by default (measured slower on the headline
// and on cfg1 graph replays); FASTRON_PDL=1 (env) turns it on.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// K1: control-point positions, float4 [M][ldpos]
cudaError_t launch_fk(const FkParams& P, const float* q, int64_t n, int64_t ldq, float4* pos, int64_t ldpos,
                      cudaStream_t st);

// Padded, scaled support tiles (see fastron_device.cuh for the layout).
int padded_m(int M);
int64_t n_support_tiles(int64_t ns);
size_t packed_bytes(int64_t ns, int M);
cudaError_t launch_pack(const float4* spos, int64_t lds, const float* alpha, int64_t ns, int M, float scale,
                        float* packed, cudaStream_t st, bool joint = false);

// K2: scoring. Plan = grid decomposition (query blocks x support splits).
struct ScorePlan {
  int64_t n_qblocks;
  int32_t n_splits;
  int32_t tiles_per_split;
  int64_t n_tiles;
};
int score_queries_per_cta(int M);
int score_max_splits(int64_t nq, int64_t ns, int M);
size_t score_partial_bytes(int64_t nq, int64_t ns, int M);

cudaError_t launch_score(const float4* qpos, int64_t nq, int64_t ldq, const float* packed, int64_t ns, int M, int kind,
                         float scale, float* score, int8_t* label, double* partial, cudaStream_t st,
                         double* score64 = nullptr, int64_t plan_nq = 0);

// Small fastron_query (nq <= 32, M <= 16): FK of the configurations inside the
// support-parallel scoring kernel, one launch. partial: >= score_partial_bytes(nq, ..).
bool query_small_ok(int64_t nq, int64_t ns, int M);
cudaError_t launch_query_small(const FkParams& P, const float* q, int64_t nq, int64_t ldq, const float* packed,
                               int64_t ns, int M, int kind, float scale, float* score, int8_t* label,
                               double* partial, cudaStream_t st);

// K4: one round of the fused edge check (interpolate -> FK -> score -> warp vote).
struct EdgeRound {
  const float* qa;
  const float* qb;
  int64_t ldq;
  int64_t n_edges;
  int32_t n_interp;
  int32_t round;
  const int32_t* active;  // round > 0: edges still undecided
  const int32_t* active_count;
  int32_t* next_active;
  int32_t* next_count;
  uint8_t* in_collision;
  int32_t* hit_index;
};
// pos: workspace for the round's control points, float4 [M][32 * n_edges]
cudaError_t launch_edge_round(const FkParams& P, const EdgeRound& R, const float* packed, int64_t ns, int M, int kind,
                              float scale, double* partial, float4* pos, cudaStream_t st);

// Joint-space RBF baseline ("Fastron RBF"): joint vectors as zero-padded pseudo points.
int joint_points(int D);
cudaError_t launch_joint_points(const float* x, int64_t n, int64_t ldx, int D, float4* out, cudaStream_t st);
cudaError_t launch_score_joint(const float4* qpts, int64_t nq, const float* packed, int64_t ns, int D, int kind,
                               float scale, float* score, int8_t* label, double* partial, cudaStream_t st);
cudaError_t launch_gram_joint(float* packed, const float4* pts, float scale, int64_t n, int D, int kind, float* K,
                              int64_t ldk, cudaStream_t st);

// Model-update cycle pieces (update.cu)
constexpr int kMaxCubes = 64;
cudaError_t launch_active_samples(const float* S, int64_t ns, int64_t lds, int D, int n_near, const float* z,
                                  const float* sigma, const float* u, int64_t n_uniform, const float* lo,
                                  const float* hi, float* out, int64_t ldo, cudaStream_t st);
cudaError_t launch_label_capsules(const float4* pos, int64_t ldp, int64_t n, const int32_t* chain, int n_chain,
                                  const double* boxes, int n_cubes, float radius, int8_t* label, cudaStream_t st);
cudaError_t launch_matvec(const float* K, int64_t n, int64_t ldk, const double* alpha, double* F, cudaStream_t st);
cudaError_t launch_matvec_lazy(const float* packed, int64_t n, int M, int kind, const double* alpha, double* F,
                               cudaStream_t st);

// fp64 path for ill-conditioned (trained) models (precise.cu)
cudaError_t launch_fk64(const FkParams& P, const float* q, int64_t n, int64_t ldq, double4* pos, int64_t ldpos,
                        cudaStream_t st);
cudaError_t launch_score64(const double4* qpos, int64_t nq, int64_t ldq, const double4* spos, const double* alpha,
                           int64_t ns, int64_t lds, int M, int kind, double gamma, double* score, int8_t* label,
                           cudaStream_t st);

// Optional content checks (validate.cu): counts are read back synchronously.
cudaError_t count_nonfinite(const float* a, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st,
                            unsigned long long* out);
cudaError_t count_nonfinite_f64(const double* a, int64_t n, cudaStream_t st, unsigned long long* out);
cudaError_t count_bad_labels(const int8_t* y, int64_t n, cudaStream_t st, unsigned long long* out);

// K3: Gram of the points pos (float4 [M][ldp]) with the kernel scale `scale`. packed: workspace
// for packed support tiles (packed_bytes(n, M)), filled only when the tile form runs.
cudaError_t launch_gram(float* packed, const float4* pos, int64_t ldp, float scale, int64_t n, int M, int kind,
                        float* K, int64_t ldk, cudaStream_t st);

// K5: Algorithm 1
struct TrainOut;
int64_t train_max_n();
cudaError_t launch_train(const float* K, int64_t n, int64_t ldk, const int8_t* y, double beta, int64_t iter_max,
                         int64_t s_max, double* alpha, double* F, int32_t* support_idx, int32_t* trace, void* result,
                         cudaStream_t st);
int64_t train_lazy_max_n(int M);
size_t train_lazy_plane_bytes(int64_t n, int M);  // global point planes needed (0: shared memory)
cudaError_t launch_train_lazy(const float* packed, int64_t n, int M, int kind, const int8_t* y, double beta,
                              int64_t iter_max, int64_t s_max, double* alpha, double* F, int32_t* support_idx,
                              int32_t* trace, void* result, float* cache, int64_t cache_cols, void* planes,
                              cudaStream_t st);

}  // namespace fastron
