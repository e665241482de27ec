// abi.cu — the C ABI of include/fastron.h: argument validation, status codes,
// workspace carving and kernel selection. No computation happens on the host except
// the per-call robot constants (cos/sin of the fixed D-H twist angles, the pre-scale
// constant); every step of the hot path runs in the kernels of fk.cu / score.cu /
// gram.cu / train.cu.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges are free unless a profiler attaches

#include "../../include/fastron.h"
#include "fastron_device.cuh"
#include "internal.h"

namespace fastron {

std::atomic<int64_t> g_launches{0};

// Off by default: measured A/B on the B200 (same box, bench --rows): headline 40.13 ->
// 40.48 ms with PDL, cfg1 graph replay 24.6 -> 28.7 us, small batches 0-2 us faster
// (DESIGN.md §6). FASTRON_PDL=1 turns it on.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FASTRON_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

// Per-device properties, queried once. The fast path is a lock-free acquire load of the
// device's ready flag (the mutex only serialises the first query per device).
const DeviceInfo& device_info() {
  static DeviceInfo infos[64];
  static std::atomic<bool> ready[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (ready[dev].load(std::memory_order_acquire)) return infos[dev];
  std::lock_guard<std::mutex> g(mu);
  if (!ready[dev].load(std::memory_order_relaxed)) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) == cudaSuccess) {
      infos[dev] = DeviceInfo{dev, p.multiProcessorCount, (int)p.sharedMemPerBlockOptin};
    } else {
      infos[dev] = DeviceInfo{dev, 148, 227 * 1024};
    }
    ready[dev].store(true, std::memory_order_release);
  }
  return infos[dev];
}

}  // namespace fastron

using namespace fastron;

namespace {

thread_local std::string t_last_error;

fastron_status fail(fastron_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return s;
}

fastron_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FASTRON_OK;
  return fail(FASTRON_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define FASTRON_REQUIRE(cond, ...) \
  do {                             \
    if (!(cond)) return fail(FASTRON_ERR_INVALID_ARG, __VA_ARGS__); \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// One NVTX range per ABI call (host-side enqueue span), named after the entry point.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// ---- optional content validation (fastron_set_validation, FASTRON_VALIDATE=1) ----
std::atomic<int> g_validate{-1};

bool validation_on() {
  int v = g_validate.load();
  if (v < 0) {
    const char* e = getenv("FASTRON_VALIDATE");
    v = (e && e[0] == '1') ? 1 : 0;
    g_validate.store(v);
  }
  return v == 1;
}

fastron_status vcheck_f32(const float* a, int64_t rows, int64_t cols, int64_t ld, void* stream, const char* what) {
  if (!a) return FASTRON_OK;
  unsigned long long bad = 0;
  const cudaError_t e = count_nonfinite(a, rows, cols, ld, S(stream), &bad);
  if (e != cudaSuccess) return fail(FASTRON_ERR_CUDA, "validation of %s: %s", what, cudaGetErrorString(e));
  if (bad) return fail(FASTRON_ERR_INVALID_ARG, "validation: %s holds %llu non-finite values", what, bad);
  return FASTRON_OK;
}

fastron_status vcheck_f64(const double* a, int64_t n, void* stream, const char* what) {
  if (!a) return FASTRON_OK;
  unsigned long long bad = 0;
  const cudaError_t e = count_nonfinite_f64(a, n, S(stream), &bad);
  if (e != cudaSuccess) return fail(FASTRON_ERR_CUDA, "validation of %s: %s", what, cudaGetErrorString(e));
  if (bad) return fail(FASTRON_ERR_INVALID_ARG, "validation: %s holds %llu non-finite values", what, bad);
  return FASTRON_OK;
}

fastron_status vcheck_labels(const int8_t* y, int64_t n, void* stream) {
  if (!y) return FASTRON_OK;
  unsigned long long bad = 0;
  const cudaError_t e = count_bad_labels(y, n, S(stream), &bad);
  if (e != cudaSuccess) return fail(FASTRON_ERR_CUDA, "validation of y: %s", cudaGetErrorString(e));
  if (bad) return fail(FASTRON_ERR_INVALID_ARG, "validation: y holds %llu labels outside {-1, +1}", bad);
  return FASTRON_OK;
}

#define FASTRON_VALIDATE(expr)                  \
  do {                                          \
    if (validation_on()) {                      \
      const fastron_status vs_ = (expr);        \
      if (vs_ != FASTRON_OK) return vs_;        \
    }                                           \
  } while (0)

fastron_status check_kernel(const fastron_kernel& k) {
  FASTRON_REQUIRE(k.kind == FASTRON_RBF_GAUSSIAN || k.kind == FASTRON_RBF_RQ, "kernel kind %d is not a fastron_rbf", k.kind);
  FASTRON_REQUIRE(std::isfinite(k.gamma) && k.gamma > 0.0f, "gamma must be finite and > 0 (PAPER.md:118), got %g",
                  (double)k.gamma);
  return FASTRON_OK;
}

// Pre-scale so that the kernels evaluate 2^-(c d)^2 = exp(-gamma d^2) (Gaussian) or
// 1/(1 + (c d)^2)^2 = (1 + gamma/2 d^2)^-2 (RQ, Eq. 3).
float kernel_scale(const fastron_kernel& k) {
  const double g = (double)k.gamma;
  const double c = k.kind == FASTRON_RBF_GAUSSIAN ? std::sqrt(g * 1.4426950408889634074) : std::sqrt(0.5 * g);
  return (float)c;
}

fastron_status check_robot(const fastron_robot* r) {
  FASTRON_REQUIRE(r != nullptr, "robot is NULL");
  FASTRON_REQUIRE(r->dof >= 1 && r->dof <= FASTRON_MAX_DOF, "dof must be in [1,16], got %d", r->dof);
  FASTRON_REQUIRE(r->n_cp >= 1 && r->n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", r->n_cp);
  for (int i = 0; i < r->dof; ++i)
    for (int c = 0; c < 4; ++c) FASTRON_REQUIRE(std::isfinite(r->dh[i][c]), "dh[%d][%d] is not finite", i, c);
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 4; ++c) FASTRON_REQUIRE(std::isfinite(r->base[i][c]), "base[%d][%d] is not finite", i, c);
  for (int m = 0; m < r->n_cp; ++m) {
    FASTRON_REQUIRE(r->cp_frame[m] >= 0 && r->cp_frame[m] <= r->dof, "cp_frame[%d] = %d outside [0, dof]", m,
                    r->cp_frame[m]);
    for (int c = 0; c < 3; ++c) FASTRON_REQUIRE(std::isfinite(r->cp_offset[m][c]), "cp_offset[%d][%d] is not finite", m, c);
  }
  return FASTRON_OK;
}

FkParams make_fk_params(const fastron_robot& r) {
  FkParams P;
  memset(&P, 0, sizeof(P));
  P.dof = r.dof;
  P.n_cp = r.n_cp;
  for (int i = 0; i < r.dof; ++i) {
    P.theta_off[i] = (double)r.dh[i][0];
    P.d[i] = (double)r.dh[i][1];
    P.a[i] = (double)r.dh[i][2];
    P.ca[i] = std::cos((double)r.dh[i][3]);
    P.sa[i] = std::sin((double)r.dh[i][3]);
  }
  for (int c = 0; c < 3; ++c) {
    for (int rr = 0; rr < 3; ++rr) P.base_c[c][rr] = (double)r.base[rr][c];
    P.base_p[c] = (double)r.base[c][3];
  }
  int n = 0;
  for (int j = 0; j <= r.dof; ++j) {
    P.frame_begin[j] = n;
    for (int m = 0; m < r.n_cp; ++m)
      if (r.cp_frame[m] == j) P.frame_list[n++] = m;
  }
  for (int j = r.dof + 1; j <= FASTRON_MAX_DOF + 1; ++j) P.frame_begin[j] = n;  // ends of frames dof..16
  for (int m = 0; m < r.n_cp; ++m)
    for (int c = 0; c < 3; ++c) P.cp_off[m][c] = (double)r.cp_offset[m][c];
  return P;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr int64_t kQueryChunk = 1 << 18;  // queries per pipelined chunk of fastron_query



// One non-blocking copy stream per device for fastron_query's host<->device pipeline.
// which = 0: host-to-device copies, 1: device-to-host copies, 2: the second compute stream.
cudaStream_t query_copy_stream(int which) {
  static cudaStream_t streams[64][3] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> g(mu);
  if (!streams[dev][which]) cudaStreamCreateWithFlags(&streams[dev][which], cudaStreamNonBlocking);
  return streams[dev][which];
}

bool is_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

}  // namespace

extern "C" {

const char* fastron_last_error(void) { return t_last_error.c_str(); }

const char* fastron_version(void) { return "fastron_b200 0.1.0 (sm_100a)"; }

int64_t fastron_launch_count(void) { return g_launches.load(); }

void fastron_set_validation(int32_t on) { g_validate.store(on ? 1 : 0); }

int32_t fastron_validation(void) { return validation_on() ? 1 : 0; }

fastron_status fastron_fk(const fastron_robot* robot, const float* q, int64_t n, int64_t ldq, float* pos, int64_t ldpos,
                          void* stream) {
  NvtxRange nvtx_range_("fastron_fk");
  fastron_status s = check_robot(robot);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(q && pos, "q and pos must be non-NULL");
  FASTRON_REQUIRE(ldq >= robot->dof, "ldq (%lld) < dof (%d)", (long long)ldq, robot->dof);
  FASTRON_REQUIRE(ldpos >= n, "ldpos (%lld) < n (%lld)", (long long)ldpos, (long long)n);
  FASTRON_REQUIRE(((uintptr_t)pos & 15) == 0, "pos must be 16-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(q, n, robot->dof, ldq, stream, "q"));
  return cuda_status(launch_fk(make_fk_params(*robot), q, n, ldq, reinterpret_cast<float4*>(pos), ldpos, S(stream)),
                     "fastron_fk");
}

size_t fastron_score_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp) {
  if (nq < 0 || ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  return align_up(packed_bytes(ns, n_cp)) + align_up(score_partial_bytes(nq, ns, n_cp));
}

fastron_status fastron_score(const float* qpos, int64_t nq, int64_t ldq, const float* spos, const float* alpha,
                             int64_t ns, int64_t lds, int32_t n_cp, fastron_kernel k, float* score, int8_t* label,
                             void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_score");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(qpos != nullptr, "qpos is NULL");
  FASTRON_REQUIRE(ldq >= nq, "ldq (%lld) < nq (%lld)", (long long)ldq, (long long)nq);
  FASTRON_REQUIRE(((uintptr_t)qpos & 15) == 0, "qpos must be 16-byte aligned (float4 records)");
  FASTRON_REQUIRE(score || label, "score and label are both NULL");
  if (ns > 0) {
    FASTRON_REQUIRE(spos && alpha, "spos and alpha must be non-NULL when ns > 0");
    FASTRON_REQUIRE(lds >= ns, "lds (%lld) < ns (%lld)", (long long)lds, (long long)ns);
    FASTRON_REQUIRE(((uintptr_t)spos & 15) == 0, "spos must be 16-byte aligned (float4 records)");
  }
  const size_t need = fastron_score_workspace_bytes(nq, ns, n_cp);
  if (workspace_bytes < need || (need > 0 && !workspace))
    return fail(FASTRON_ERR_WORKSPACE, "fastron_score needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(qpos, n_cp, 4 * nq, 4 * ldq, stream, "qpos"));
  if (ns > 0) {
    FASTRON_VALIDATE(vcheck_f32(spos, n_cp, 4 * ns, 4 * lds, stream, "spos"));
    FASTRON_VALIDATE(vcheck_f32(alpha, 1, ns, ns, stream, "alpha"));
  }
  char* ws = static_cast<char*>(workspace);
  float* packed = reinterpret_cast<float*>(ws);
  double* partial = reinterpret_cast<double*>(ws + align_up(packed_bytes(ns, n_cp)));
  const float c = kernel_scale(k);
  cudaError_t e = launch_pack(reinterpret_cast<const float4*>(spos), lds, alpha, ns, n_cp, c, packed, S(stream));
  if (e != cudaSuccess) return cuda_status(e, "fastron_score(pack)");
  e = launch_score(reinterpret_cast<const float4*>(qpos), nq, ldq, packed, ns, n_cp, k.kind, c, score, label, partial,
                   S(stream));
  return cuda_status(e, "fastron_score");
}

size_t fastron_model_bytes(int64_t ns, int32_t n_cp) {
  if (ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  return align_up(packed_bytes(ns, n_cp));
}

fastron_status fastron_model_pack(const float* spos, const float* alpha, int64_t ns, int64_t lds, int32_t n_cp,
                                  fastron_kernel k, void* packed, size_t packed_bytes_given, void* stream) {
  NvtxRange nvtx_range_("fastron_model_pack");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(ns >= 0, "ns must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (ns == 0) return FASTRON_OK;
  FASTRON_REQUIRE(spos && alpha, "spos and alpha must be non-NULL when ns > 0");
  FASTRON_REQUIRE(lds >= ns, "lds (%lld) < ns (%lld)", (long long)lds, (long long)ns);
  const size_t need = fastron_model_bytes(ns, n_cp);
  if (packed_bytes_given < need || !packed)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_model_pack needs %zu bytes, got %zu", need, packed_bytes_given);
  FASTRON_REQUIRE(((uintptr_t)packed & 255) == 0, "packed must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(spos, n_cp, 4 * ns, 4 * lds, stream, "spos"));
  FASTRON_VALIDATE(vcheck_f32(alpha, 1, ns, ns, stream, "alpha"));
  return cuda_status(launch_pack(reinterpret_cast<const float4*>(spos), lds, alpha, ns, n_cp, kernel_scale(k),
                                 static_cast<float*>(packed), S(stream)),
                     "fastron_model_pack");
}

size_t fastron_score_packed_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp) {
  if (nq < 0 || ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  return align_up(score_partial_bytes(nq, ns, n_cp));
}

fastron_status fastron_score_packed(const float* qpos, int64_t nq, int64_t ldq, const void* packed, int64_t ns,
                                    int32_t n_cp, fastron_kernel k, float* score, int8_t* label, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_score_packed");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(qpos != nullptr, "qpos is NULL");
  FASTRON_REQUIRE(ldq >= nq, "ldq (%lld) < nq (%lld)", (long long)ldq, (long long)nq);
  FASTRON_REQUIRE(score || label, "score and label are both NULL");
  FASTRON_REQUIRE(ns == 0 || packed, "packed is NULL");
  FASTRON_REQUIRE(((uintptr_t)qpos & 15) == 0, "qpos must be 16-byte aligned (float4 records)");
  FASTRON_REQUIRE(ns == 0 || ((uintptr_t)packed & 255) == 0, "packed must be 256-byte aligned (fastron_model_pack)");
  const size_t need = fastron_score_packed_workspace_bytes(nq, ns, n_cp);
  if (workspace_bytes < need || (need > 0 && !workspace))
    return fail(FASTRON_ERR_WORKSPACE, "fastron_score_packed needs %zu workspace bytes, got %zu", need,
                workspace_bytes);
  FASTRON_REQUIRE(need == 0 || ((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(qpos, n_cp, 4 * nq, 4 * ldq, stream, "qpos"));
  return cuda_status(launch_score(reinterpret_cast<const float4*>(qpos), nq, ldq, static_cast<const float*>(packed), ns,
                                  n_cp, k.kind, kernel_scale(k), score, label, static_cast<double*>(workspace),
                                  S(stream)),
                     "fastron_score_packed");
}

fastron_status fastron_fk64(const fastron_robot* robot, const float* q, int64_t n, int64_t ldq, double* pos,
                            int64_t ldpos, void* stream) {
  NvtxRange nvtx_range_("fastron_fk64");
  fastron_status s = check_robot(robot);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(q && pos, "q and pos must be non-NULL");
  FASTRON_REQUIRE(ldq >= robot->dof, "ldq (%lld) < dof (%d)", (long long)ldq, robot->dof);
  FASTRON_REQUIRE(ldpos >= n, "ldpos (%lld) < n (%lld)", (long long)ldpos, (long long)n);
  FASTRON_REQUIRE(((uintptr_t)pos & 31) == 0, "pos must be 32-byte aligned (double4 records)");
  FASTRON_VALIDATE(vcheck_f32(q, n, robot->dof, ldq, stream, "q"));
  return cuda_status(launch_fk64(make_fk_params(*robot), q, n, ldq, reinterpret_cast<double4*>(pos), ldpos, S(stream)),
                     "fastron_fk64");
}

fastron_status fastron_score_precise(const double* qpos, int64_t nq, int64_t ldq, const double* spos,
                                     const double* alpha, int64_t ns, int64_t lds, int32_t n_cp, fastron_kernel k,
                                     double* score, int8_t* label, void* stream) {
  NvtxRange nvtx_range_("fastron_score_precise");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (n_cp > 16) return fail(FASTRON_ERR_UNSUPPORTED, "fastron_score_precise supports n_cp <= 16, got %d", n_cp);
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(qpos != nullptr && ldq >= nq, "qpos must be non-NULL and ldq >= nq");
  FASTRON_REQUIRE(score || label, "score and label are both NULL");
  FASTRON_REQUIRE(((uintptr_t)qpos & 31) == 0, "qpos must be 32-byte aligned (double4 records)");
  if (ns > 0) {
    FASTRON_REQUIRE(spos && alpha, "spos and alpha must be non-NULL when ns > 0");
    FASTRON_REQUIRE(lds >= ns, "lds (%lld) < ns (%lld)", (long long)lds, (long long)ns);
    FASTRON_REQUIRE(((uintptr_t)spos & 31) == 0, "spos must be 32-byte aligned (double4 records)");
  }
  FASTRON_VALIDATE(vcheck_f64(qpos, 4 * ldq * n_cp, stream, "qpos"));
  if (ns > 0) {
    FASTRON_VALIDATE(vcheck_f64(spos, 4 * lds * n_cp, stream, "spos"));
    FASTRON_VALIDATE(vcheck_f64(alpha, ns, stream, "alpha"));
  }
  return cuda_status(launch_score64(reinterpret_cast<const double4*>(qpos), nq, ldq,
                                    reinterpret_cast<const double4*>(spos), alpha, ns, lds, n_cp, k.kind,
                                    (double)k.gamma, score, label, S(stream)),
                     "fastron_score_precise");
}

fastron_status fastron_score_packed_f64(const float* qpos, int64_t nq, int64_t ldq, const void* packed, int64_t ns,
                                        int32_t n_cp, fastron_kernel k, double* score64, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_score_packed_f64");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(qpos && score64 && ldq >= nq, "qpos and score64 must be non-NULL and ldq >= nq");
  FASTRON_REQUIRE(ns == 0 || packed, "packed is NULL");
  FASTRON_REQUIRE(((uintptr_t)qpos & 15) == 0, "qpos must be 16-byte aligned (float4 records)");
  FASTRON_REQUIRE(ns == 0 || ((uintptr_t)packed & 255) == 0, "packed must be 256-byte aligned (fastron_model_pack)");
  const size_t need = fastron_score_packed_workspace_bytes(nq, ns, n_cp);
  if (workspace_bytes < need || (need > 0 && !workspace))
    return fail(FASTRON_ERR_WORKSPACE, "fastron_score_packed_f64 needs %zu workspace bytes, got %zu", need,
                workspace_bytes);
  FASTRON_REQUIRE(need == 0 || ((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(qpos, n_cp, 4 * nq, 4 * ldq, stream, "qpos"));
  return cuda_status(launch_score(reinterpret_cast<const float4*>(qpos), nq, ldq, static_cast<const float*>(packed), ns,
                                  n_cp, k.kind, kernel_scale(k), nullptr, nullptr, static_cast<double*>(workspace),
                                  S(stream), score64),
                     "fastron_score_packed_f64");
}

size_t fastron_gram_workspace_bytes(int64_t n, int32_t n_cp) {
  if (n < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  // the Gram kernel reads column tiles in pairs: round the packed buffer to an even tile count
  const int64_t tiles = n_support_tiles(n);
  return align_up(packed_bytes((tiles + 1) / 2 * 2 * kTileSupports, n_cp));
}

fastron_status fastron_gram(const float* pos, int64_t n, int64_t ldp, int32_t n_cp, fastron_kernel k, float* K,
                            int64_t ldk, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_gram");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(pos && K, "pos and K must be non-NULL");
  FASTRON_REQUIRE(ldp >= n && ldk >= n, "ldp and ldk must be >= n");
  const size_t need = fastron_gram_workspace_bytes(n, n_cp);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_gram needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(pos, n_cp, 4 * n, 4 * ldp, stream, "pos"));
  float* packed = static_cast<float*>(workspace);
  const float c = kernel_scale(k);
  return cuda_status(launch_gram(packed, reinterpret_cast<const float4*>(pos), ldp, c, n, n_cp, k.kind, K, ldk, S(stream)),
                     "fastron_gram");
}

int64_t fastron_train_max_n(void) { return train_max_n(); }

fastron_status fastron_train(const float* K, int64_t n, int64_t ldk, const int8_t* y, double beta, int64_t iter_max,
                             int64_t s_max, double* alpha_inout, double* F_inout, int32_t* support_idx, int32_t* trace,
                             fastron_train_result* result, void* stream) {
  NvtxRange nvtx_range_("fastron_train");
  FASTRON_REQUIRE(n >= 0 && iter_max >= 0 && s_max >= 0, "n, iter_max and s_max must be >= 0");
  FASTRON_REQUIRE(std::isfinite(beta) && beta >= 1.0, "beta must be >= 1 (PAPER.md:189), got %g", beta);
  FASTRON_REQUIRE(result != nullptr, "result is NULL");
  if (n > fastron_train_max_n())
    return fail(FASTRON_ERR_UNSUPPORTED, "n = %lld exceeds fastron_train_max_n() = %lld", (long long)n,
                (long long)fastron_train_max_n());
  if (n > 0x7fffffffLL) return fail(FASTRON_ERR_UNSUPPORTED, "n too large");
  if (n == 0) return cuda_status(cudaMemsetAsync(result, 0, sizeof(*result), S(stream)), "fastron_train");
  FASTRON_REQUIRE(K && y && alpha_inout && F_inout, "K, y, alpha_inout and F_inout must be non-NULL");
  FASTRON_REQUIRE(ldk >= n, "ldk (%lld) < n (%lld)", (long long)ldk, (long long)n);
  FASTRON_VALIDATE(vcheck_f32(K, n, n, ldk, stream, "K"));
  FASTRON_VALIDATE(vcheck_labels(y, n, stream));
  FASTRON_VALIDATE(vcheck_f64(alpha_inout, n, stream, "alpha_inout"));
  FASTRON_VALIDATE(vcheck_f64(F_inout, n, stream, "F_inout"));
  return cuda_status(launch_train(K, n, ldk, y, beta, iter_max, s_max, alpha_inout, F_inout, support_idx, trace, result,
                                  S(stream)),
                     "fastron_train");
}

int64_t fastron_train_lazy_max_n(int32_t n_cp) {
  if (n_cp < 1 || n_cp > 16) return 0;
  return train_lazy_max_n(n_cp);
}

size_t fastron_train_lazy_workspace_bytes(int64_t n, int32_t n_cp, int64_t cache_cols) {
  if (n < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP || cache_cols < 0) return 0;
  return align_up(packed_bytes(n, n_cp)) + align_up((size_t)cache_cols * (size_t)n * 4) +
         align_up(n_cp <= 16 ? train_lazy_plane_bytes(n, n_cp) : 0);
}

fastron_status fastron_train_lazy(const float* pos, int64_t n, int64_t ldp, int32_t n_cp, fastron_kernel k,
                                  const int8_t* y, double beta, int64_t iter_max, int64_t s_max,
                                  double* alpha_inout, double* F_inout, int32_t* support_idx, int32_t* trace,
                                  fastron_train_result* result, int64_t cache_cols, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_train_lazy");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n >= 0 && iter_max >= 0 && s_max >= 0 && cache_cols >= 0, "sizes must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  FASTRON_REQUIRE(std::isfinite(beta) && beta >= 1.0, "beta must be >= 1 (PAPER.md:189), got %g", beta);
  FASTRON_REQUIRE(result != nullptr, "result is NULL");
  if (n_cp > 16) return fail(FASTRON_ERR_UNSUPPORTED, "fastron_train_lazy supports n_cp <= 16, got %d", n_cp);
  if (n > fastron_train_lazy_max_n(n_cp))
    return fail(FASTRON_ERR_UNSUPPORTED, "n = %lld exceeds fastron_train_lazy_max_n = %lld", (long long)n,
                (long long)fastron_train_lazy_max_n(n_cp));
  if (n == 0) return cuda_status(cudaMemsetAsync(result, 0, sizeof(*result), S(stream)), "fastron_train_lazy");
  FASTRON_REQUIRE(pos && y && alpha_inout && F_inout, "pos, y, alpha_inout and F_inout must be non-NULL");
  FASTRON_REQUIRE(ldp >= n, "ldp (%lld) < n (%lld)", (long long)ldp, (long long)n);
  const size_t need = fastron_train_lazy_workspace_bytes(n, n_cp, cache_cols);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_train_lazy needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(pos, n_cp, 4 * n, 4 * ldp, stream, "pos"));
  FASTRON_VALIDATE(vcheck_labels(y, n, stream));
  FASTRON_VALIDATE(vcheck_f64(alpha_inout, n, stream, "alpha_inout"));
  FASTRON_VALIDATE(vcheck_f64(F_inout, n, stream, "F_inout"));
  char* ws = static_cast<char*>(workspace);
  float* packed = reinterpret_cast<float*>(ws);
  float* cache = reinterpret_cast<float*>(ws + align_up(packed_bytes(n, n_cp)));
  void* planes = ws + align_up(packed_bytes(n, n_cp)) + align_up((size_t)cache_cols * (size_t)n * 4);
  cudaStream_t st = S(stream);
  cudaError_t e =
      launch_pack(reinterpret_cast<const float4*>(pos), ldp, nullptr, n, n_cp, kernel_scale(k), packed, st);
  if (e == cudaSuccess)
    e = launch_train_lazy(packed, n, n_cp, k.kind, y, beta, iter_max, s_max, alpha_inout, F_inout, support_idx, trace,
                          result, cache, cache_cols, planes, st);
  return cuda_status(e, "fastron_train_lazy");
}

fastron_status fastron_active_samples(const float* sup, int64_t ns, int64_t lds, int32_t dof, int32_t n_near,
                                      const float* z, const float* sigma, const float* u, int64_t n_uniform,
                                      const float* lo, const float* hi, float* out, int64_t ldo, void* stream) {
  NvtxRange nvtx_range_("fastron_active_samples");
  FASTRON_REQUIRE(ns >= 0 && n_near >= 0 && n_uniform >= 0, "sizes must be >= 0");
  FASTRON_REQUIRE(dof >= 1 && dof <= FASTRON_MAX_DOF, "dof must be in [1,16], got %d", dof);
  if (ns * n_near + n_uniform == 0) return FASTRON_OK;
  FASTRON_REQUIRE(lo && hi && out && ldo >= dof, "lo, hi, out must be non-NULL and ldo >= dof");
  if (ns * n_near > 0) FASTRON_REQUIRE(sup && z && sigma && lds >= dof, "S, z, sigma needed for stage-1 samples");
  if (n_uniform > 0) FASTRON_REQUIRE(u != nullptr, "u needed for stage-2 samples");
  return cuda_status(launch_active_samples(sup, ns, lds, dof, n_near, z, sigma, u, n_uniform, lo, hi, out, ldo, S(stream)),
                     "fastron_active_samples");
}

fastron_status fastron_label_capsules(const float* pos, int64_t ldp, int64_t n, const int32_t* chain, int32_t n_chain,
                                      const double* boxes, int32_t n_cubes, float radius, int8_t* label, void* stream) {
  NvtxRange nvtx_range_("fastron_label_capsules");
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  FASTRON_REQUIRE(n_chain >= 0 && n_chain <= 33 && n_cubes >= 0 && n_cubes <= kMaxCubes,
                  "n_chain must be in [0,33] and n_cubes in [0,64]");
  FASTRON_REQUIRE(std::isfinite(radius) && radius >= 0.0f, "radius must be finite and >= 0");
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(pos && label && ldp >= n, "pos and label must be non-NULL and ldp >= n");
  FASTRON_REQUIRE(n_chain == 0 || chain, "chain is NULL");
  FASTRON_REQUIRE(n_cubes == 0 || boxes, "boxes is NULL");
  for (int c = 0; c < n_chain; ++c) FASTRON_REQUIRE(chain[c] >= -1 && chain[c] < FASTRON_MAX_CP, "chain[%d] invalid", c);
  for (int b = 0; b < 6 * n_cubes; ++b) FASTRON_REQUIRE(std::isfinite(boxes[b]), "boxes contain a non-finite value");
  return cuda_status(launch_label_capsules(reinterpret_cast<const float4*>(pos), ldp, n, chain, n_chain, boxes, n_cubes,
                                           radius, label, S(stream)),
                     "fastron_label_capsules");
}

fastron_status fastron_kernel_matvec(const float* K, int64_t n, int64_t ldk, const double* alpha, double* F,
                                     void* stream) {
  NvtxRange nvtx_range_("fastron_kernel_matvec");
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(K && alpha && F && ldk >= n, "K, alpha, F must be non-NULL and ldk >= n");
  return cuda_status(launch_matvec(K, n, ldk, alpha, F, S(stream)), "fastron_kernel_matvec");
}

size_t fastron_kernel_matvec_lazy_workspace_bytes(int64_t n, int32_t n_cp) {
  if (n < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  return align_up(packed_bytes(n, n_cp));
}

fastron_status fastron_kernel_matvec_lazy(const float* pos, int64_t n, int64_t ldp, int32_t n_cp, fastron_kernel k,
                                          const double* alpha, double* F, void* workspace, size_t workspace_bytes,
                                          void* stream) {
  NvtxRange nvtx_range_("fastron_kernel_matvec_lazy");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  FASTRON_REQUIRE(n_cp >= 1 && n_cp <= FASTRON_MAX_CP, "n_cp must be in [1,32], got %d", n_cp);
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(pos && alpha && F && ldp >= n, "pos, alpha, F must be non-NULL and ldp >= n");
  FASTRON_REQUIRE(((uintptr_t)pos & 15) == 0, "pos must be 16-byte aligned (float4 records)");
  const size_t need = fastron_kernel_matvec_lazy_workspace_bytes(n, n_cp);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_kernel_matvec_lazy needs %zu workspace bytes, got %zu", need,
                workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(pos, n_cp, 4 * n, 4 * ldp, stream, "pos"));
  FASTRON_VALIDATE(vcheck_f64(alpha, n, stream, "alpha"));
  float* packed = static_cast<float*>(workspace);
  cudaStream_t st = S(stream);
  cudaError_t e = launch_pack(reinterpret_cast<const float4*>(pos), ldp, nullptr, n, n_cp, kernel_scale(k), packed, st);
  if (e == cudaSuccess) e = launch_matvec_lazy(packed, n, n_cp, k.kind, alpha, F, st);
  return cuda_status(e, "fastron_kernel_matvec_lazy");
}

size_t fastron_edge_packed_workspace_bytes(int64_t n_edges, int64_t ns, int32_t n_cp) {
  if (n_edges < 0 || ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  const size_t lists = 2 * align_up((size_t)n_edges * 4) + 256;  // two active lists + two counters
  const size_t pos = align_up((size_t)n_edges * 32 * n_cp * 16);  // a round's control points
  return align_up(score_partial_bytes(n_edges * 32, ns, n_cp)) + lists + pos;
}

size_t fastron_edge_workspace_bytes(int64_t n_edges, int64_t ns, int32_t n_cp) {
  if (n_edges < 0 || ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP) return 0;
  return align_up(packed_bytes(ns, n_cp)) + fastron_edge_packed_workspace_bytes(n_edges, ns, n_cp);
}

}  // extern "C"

namespace {

// the rounds of the edge check against a packed model; ws: fastron_edge_packed_workspace_bytes
fastron_status edge_rounds(const fastron_robot* robot, const float* qa, const float* qb, int64_t n_edges, int64_t ldq,
                           int32_t n_interp, const float* packed, int64_t ns, fastron_kernel k, uint8_t* in_collision,
                           int32_t* hit_index, char* ws, cudaStream_t st) {
  const int M = robot->n_cp;
  double* partial = reinterpret_cast<double*>(ws);
  ws += align_up(score_partial_bytes(n_edges * 32, ns, M));
  int32_t* counts = reinterpret_cast<int32_t*>(ws);  // [2] live counters (256 B reserved)
  ws += 256;
  int32_t* lists[2] = {reinterpret_cast<int32_t*>(ws), reinterpret_cast<int32_t*>(ws + align_up((size_t)n_edges * 4))};
  ws += 2 * align_up((size_t)n_edges * 4);
  float4* epos = reinterpret_cast<float4*>(ws);
  const float c = kernel_scale(k);
  const FkParams P = make_fk_params(*robot);
  const int rounds = (n_interp + 31) / 32;
  for (int r = 0; r < rounds; ++r) {
    EdgeRound R;
    R.qa = qa;
    R.qb = qb;
    R.ldq = ldq;
    R.n_edges = n_edges;
    R.n_interp = n_interp;
    R.round = r;
    R.active = r == 0 ? nullptr : lists[(r - 1) & 1];
    R.active_count = r == 0 ? nullptr : counts + ((r - 1) & 1);
    R.next_active = lists[r & 1];
    R.next_count = counts + (r & 1);
    R.in_collision = in_collision;
    R.hit_index = hit_index;
    cudaError_t e = cudaMemsetAsync(R.next_count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return cuda_status(e, "fastron_edge_check(memset)");
    e = launch_edge_round(P, R, packed, ns, M, k.kind, c, partial, epos, st);
    if (e != cudaSuccess) return cuda_status(e, "fastron_edge_check");
  }
  return FASTRON_OK;
}

fastron_status edge_common_checks(const fastron_robot* robot, const float* qa, const float* qb, int64_t n_edges,
                                  int64_t ldq, int32_t n_interp, int64_t ns, fastron_kernel k, uint8_t* in_collision) {
  fastron_status s = check_robot(robot);
  if (s != FASTRON_OK) return s;
  s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n_edges >= 0 && ns >= 0, "n_edges and ns must be >= 0");
  FASTRON_REQUIRE(n_interp >= 1, "n_interp must be >= 1, got %d", n_interp);
  if (n_edges == 0) return FASTRON_OK;
  FASTRON_REQUIRE(n_edges <= (int64_t)1 << 26, "n_edges too large for one call (max 2^26)");
  FASTRON_REQUIRE(qa && qb && in_collision, "qa, qb and in_collision must be non-NULL");
  FASTRON_REQUIRE(ldq >= robot->dof, "ldq (%lld) < dof (%d)", (long long)ldq, robot->dof);
  return FASTRON_OK;
}

}  // namespace

extern "C" {

fastron_status fastron_edge_check(const fastron_robot* robot, const float* qa, const float* qb, int64_t n_edges,
                                  int64_t ldq, int32_t n_interp, const float* spos, const float* alpha, int64_t ns,
                                  int64_t lds, fastron_kernel k, uint8_t* in_collision, int32_t* hit_index,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_edge_check");
  fastron_status s = edge_common_checks(robot, qa, qb, n_edges, ldq, n_interp, ns, k, in_collision);
  if (s != FASTRON_OK || n_edges == 0) return s;
  if (ns > 0) {
    FASTRON_REQUIRE(spos && alpha, "spos and alpha must be non-NULL when ns > 0");
    FASTRON_REQUIRE(lds >= ns, "lds (%lld) < ns (%lld)", (long long)lds, (long long)ns);
  }
  const size_t need = fastron_edge_workspace_bytes(n_edges, ns, robot->n_cp);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_edge_check needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  const int M = robot->n_cp;
  FASTRON_VALIDATE(vcheck_f32(qa, n_edges, robot->dof, ldq, stream, "qa"));
  FASTRON_VALIDATE(vcheck_f32(qb, n_edges, robot->dof, ldq, stream, "qb"));
  if (ns > 0) {
    FASTRON_VALIDATE(vcheck_f32(spos, M, 4 * ns, 4 * lds, stream, "spos"));
    FASTRON_VALIDATE(vcheck_f32(alpha, 1, ns, ns, stream, "alpha"));
  }
  char* ws = static_cast<char*>(workspace);
  float* packed = reinterpret_cast<float*>(ws);
  cudaStream_t st = S(stream);
  cudaError_t e = launch_pack(reinterpret_cast<const float4*>(spos), lds, alpha, ns, M, kernel_scale(k), packed, st);
  if (e != cudaSuccess) return cuda_status(e, "fastron_edge_check(pack)");
  return edge_rounds(robot, qa, qb, n_edges, ldq, n_interp, packed, ns, k, in_collision, hit_index,
                     ws + align_up(packed_bytes(ns, M)), st);
}

fastron_status fastron_edge_check_packed(const fastron_robot* robot, const float* qa, const float* qb,
                                         int64_t n_edges, int64_t ldq, int32_t n_interp, const void* packed,
                                         int64_t ns, int32_t n_cp, fastron_kernel k, uint8_t* in_collision,
                                         int32_t* hit_index, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_edge_check_packed");
  fastron_status s = edge_common_checks(robot, qa, qb, n_edges, ldq, n_interp, ns, k, in_collision);
  if (s != FASTRON_OK || n_edges == 0) return s;
  FASTRON_REQUIRE(n_cp == robot->n_cp, "n_cp (%d) differs from robot->n_cp (%d)", n_cp, robot->n_cp);
  FASTRON_REQUIRE(ns == 0 || packed, "packed is NULL");
  FASTRON_REQUIRE(ns == 0 || ((uintptr_t)packed & 255) == 0, "packed must be 256-byte aligned (fastron_model_pack)");
  const size_t need = fastron_edge_packed_workspace_bytes(n_edges, ns, n_cp);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_edge_check_packed needs %zu workspace bytes, got %zu", need,
                workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(qa, n_edges, robot->dof, ldq, stream, "qa"));
  FASTRON_VALIDATE(vcheck_f32(qb, n_edges, robot->dof, ldq, stream, "qb"));
  return edge_rounds(robot, qa, qb, n_edges, ldq, n_interp, static_cast<const float*>(packed), ns, k, in_collision,
                     hit_index, static_cast<char*>(workspace), S(stream));
}

size_t fastron_score_joint_workspace_bytes(int64_t nq, int64_t ns, int32_t dof) {
  if (nq < 0 || ns < 0 || dof < 1 || dof > FASTRON_MAX_DOF) return 0;
  const int Mj = joint_points(dof);
  return align_up((size_t)(nq + ns) * Mj * 16) + align_up(packed_bytes(ns, Mj)) +
         align_up(score_partial_bytes(nq, ns, Mj));
}

fastron_status fastron_score_joint(const float* q, int64_t nq, int64_t ldq, const float* sx, const float* alpha,
                                   int64_t ns, int64_t lds, int32_t dof, fastron_kernel k, float* score,
                                   int8_t* label, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_score_joint");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  FASTRON_REQUIRE(dof >= 1 && dof <= FASTRON_MAX_DOF, "dof must be in [1,16], got %d", dof);
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(q != nullptr && ldq >= dof, "q must be non-NULL with ldq >= dof");
  FASTRON_REQUIRE(score || label, "score and label are both NULL");
  if (ns > 0) FASTRON_REQUIRE(sx && alpha && lds >= dof, "s and alpha must be non-NULL with lds >= dof when ns > 0");
  const size_t need = fastron_score_joint_workspace_bytes(nq, ns, dof);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_score_joint needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(q, nq, dof, ldq, stream, "q"));
  if (ns > 0) {
    FASTRON_VALIDATE(vcheck_f32(sx, ns, dof, lds, stream, "s"));
    FASTRON_VALIDATE(vcheck_f32(alpha, 1, ns, ns, stream, "alpha"));
  }
  const int Mj = joint_points(dof);
  char* ws = static_cast<char*>(workspace);
  float4* qpts = reinterpret_cast<float4*>(ws);
  float4* spts = qpts + (size_t)nq * Mj;
  ws += align_up((size_t)(nq + ns) * Mj * 16);
  float* packed = reinterpret_cast<float*>(ws);
  ws += align_up(packed_bytes(ns, Mj));
  double* partial = reinterpret_cast<double*>(ws);
  cudaStream_t st = S(stream);
  const float c = kernel_scale(k);
  cudaError_t e = launch_joint_points(q, nq, ldq, dof, qpts, st);
  if (e == cudaSuccess) e = launch_joint_points(sx, ns, lds, dof, spts, st);
  if (e == cudaSuccess) e = launch_pack(spts, ns, alpha, ns, Mj, c, packed, st, true);
  if (e == cudaSuccess) e = launch_score_joint(qpts, nq, packed, ns, dof, k.kind, c, score, label, partial, st);
  return cuda_status(e, "fastron_score_joint");
}

size_t fastron_gram_joint_workspace_bytes(int64_t n, int32_t dof) {
  if (n < 0 || dof < 1 || dof > FASTRON_MAX_DOF) return 0;
  const int Mj = joint_points(dof);
  const int64_t tiles = n_support_tiles(n);
  return align_up((size_t)n * Mj * 16) + align_up(packed_bytes((tiles + 1) / 2 * 2 * kTileSupports, Mj));
}

fastron_status fastron_gram_joint(const float* x, int64_t n, int64_t ldx, int32_t dof, fastron_kernel k, float* K,
                                  int64_t ldk, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_gram_joint");
  fastron_status s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(n >= 0, "n must be >= 0");
  FASTRON_REQUIRE(dof >= 1 && dof <= FASTRON_MAX_DOF, "dof must be in [1,16], got %d", dof);
  if (n == 0) return FASTRON_OK;
  FASTRON_REQUIRE(x && K, "x and K must be non-NULL");
  FASTRON_REQUIRE(ldx >= dof && ldk >= n, "ldx must be >= dof and ldk >= n");
  const size_t need = fastron_gram_joint_workspace_bytes(n, dof);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_gram_joint needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(x, n, dof, ldx, stream, "x"));
  const int Mj = joint_points(dof);
  char* ws = static_cast<char*>(workspace);
  float4* pts = reinterpret_cast<float4*>(ws);
  float* packed = reinterpret_cast<float*>(ws + align_up((size_t)n * Mj * 16));
  cudaStream_t st = S(stream);
  const float c = kernel_scale(k);
  cudaError_t e = launch_joint_points(x, n, ldx, dof, pts, st);
  if (e == cudaSuccess) e = launch_gram_joint(packed, pts, c, n, dof, k.kind, K, ldk, st);
  return cuda_status(e, "fastron_gram_joint");
}

size_t fastron_query_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp, int32_t dof) {
  if (nq < 0 || ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP || dof < 1 || dof > FASTRON_MAX_DOF) return 0;
  const int64_t chunk = nq < kQueryChunk ? nq : kQueryChunk;
  // per in-flight chunk: q (dof floats), positions (n_cp float4), score (float), label (int8); two chunks
  const size_t per = align_up((size_t)chunk * dof * 4) + align_up((size_t)chunk * n_cp * 16) +
                     align_up((size_t)chunk * 4) + align_up((size_t)chunk);
  return align_up(packed_bytes(ns, n_cp)) + 2 * align_up(score_partial_bytes(chunk, ns, n_cp)) + 2 * per;
}

fastron_status fastron_query(const fastron_robot* robot, const float* q, int64_t nq, int64_t ldq, const float* spos,
                             const float* alpha, int64_t ns, int64_t lds, fastron_kernel k, float* score,
                             int8_t* label, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_query");
  fastron_status s = check_robot(robot);
  if (s != FASTRON_OK) return s;
  s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(q != nullptr, "q is NULL");
  FASTRON_REQUIRE(score || label, "score and label are both NULL");
  FASTRON_REQUIRE(ldq >= robot->dof, "ldq (%lld) < dof (%d)", (long long)ldq, robot->dof);
  if (ns > 0) {
    FASTRON_REQUIRE(spos && alpha, "spos and alpha must be non-NULL when ns > 0");
    FASTRON_REQUIRE(lds >= ns, "lds (%lld) < ns (%lld)", (long long)lds, (long long)ns);
  }
  const int M = robot->n_cp, D = robot->dof;
  const size_t need = fastron_query_workspace_bytes(nq, ns, M, D);
  if (workspace_bytes < need || !workspace)
    return fail(FASTRON_ERR_WORKSPACE, "fastron_query needs %zu workspace bytes, got %zu", need, workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  const bool q_host = is_host_ptr(q), s_host = is_host_ptr(score), l_host = is_host_ptr(label);
  if (validation_on()) {
    if (q_host) {
      for (int64_t i = 0; i < nq; ++i)
        for (int j = 0; j < D; ++j)
          FASTRON_REQUIRE(std::isfinite(q[i * ldq + j]), "validation: q[%lld][%d] is not finite", (long long)i, j);
    } else {
      FASTRON_VALIDATE(vcheck_f32(q, nq, D, ldq, stream, "q"));
    }
    if (ns > 0) {
      FASTRON_VALIDATE(vcheck_f32(spos, M, 4 * ns, 4 * lds, stream, "spos"));
      FASTRON_VALIDATE(vcheck_f32(alpha, 1, ns, ns, stream, "alpha"));
    }
  }
  const int64_t chunk = nq < kQueryChunk ? nq : kQueryChunk;
  char* ws = static_cast<char*>(workspace);
  float* packed = reinterpret_cast<float*>(ws);
  ws += align_up(packed_bytes(ns, M));
  double* partials[2];
  for (int b = 0; b < 2; ++b) {
    partials[b] = reinterpret_cast<double*>(ws);
    ws += align_up(score_partial_bytes(chunk, ns, M));
  }
  double* partial = partials[0];
  struct Buf { float* q; float* pos; float* sc; int8_t* lb; } buf[2];
  for (int b = 0; b < 2; ++b) {
    buf[b].q = reinterpret_cast<float*>(ws); ws += align_up((size_t)chunk * D * 4);
    buf[b].pos = reinterpret_cast<float*>(ws); ws += align_up((size_t)chunk * M * 16);
    buf[b].sc = reinterpret_cast<float*>(ws); ws += align_up((size_t)chunk * 4);
    buf[b].lb = reinterpret_cast<int8_t*>(ws); ws += align_up((size_t)chunk);
  }
  cudaStream_t st = S(stream);
  const float c = kernel_scale(k);
  const FkParams P = make_fk_params(*robot);
  cudaError_t e = launch_pack(reinterpret_cast<const float4*>(spos), lds, alpha, ns, M, c, packed, st);
  if (e != cudaSuccess) return cuda_status(e, "fastron_query(pack)");
  const bool any_host = q_host || s_host || l_host;
  if (!any_host) {
    // device pointers: FK of the whole batch through the positions buffer in chunks
    for (int64_t off = 0; off < nq; off += chunk) {
      const int64_t n = nq - off < chunk ? nq - off : chunk;
      if (query_small_ok(nq, ns, M)) {  // one launch: FK inside the small-batch kernel
        e = launch_query_small(P, q, nq, ldq, packed, ns, M, k.kind, c, score, label, partial, st);
      } else {
        e = launch_fk(P, q + off * ldq, n, ldq, reinterpret_cast<float4*>(buf[0].pos), chunk, st);
        if (e == cudaSuccess)
          e = launch_score(reinterpret_cast<const float4*>(buf[0].pos), n, chunk, packed, ns, M, k.kind, c,
                           score ? score + off : nullptr, label ? label + off : nullptr, partial, st, nullptr, nq);
      }
      if (e != cudaSuccess) return cuda_status(e, "fastron_query");
    }
    return FASTRON_OK;
  }
  // host buffers: H2D(chunk c+1) on one copy stream and D2H(chunk c-1) on another overlap
  // FK+score(chunk c); chunks alternate between two buffer sets and two compute streams
  // (`stream` and a library stream), so chunk c+1's kernels fill the SMs that chunk c's
  // last wave leaves idle, and chunk c+2 reuses chunk c's buffers
  cudaStream_t h2d = query_copy_stream(0), d2h = query_copy_stream(1);
  cudaStream_t cs[2] = {st, query_copy_stream(2)};
  // the pipeline's 6 events are created once per host thread and device (a call ends with
  // a synchronisation, so the next call on this thread may reuse them)
  static thread_local cudaEvent_t t_events[64][6] = {};
  int evdev = 0;
  cudaGetDevice(&evdev);
  if (evdev < 0 || evdev >= 64) evdev = 0;
  cudaEvent_t* evs = t_events[evdev];
  if (!evs[0])
    for (int i = 0; i < 6; ++i) cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
  cudaEvent_t* ev_in = evs;
  cudaEvent_t* ev_used = evs + 2;
  cudaEvent_t* ev_out = evs + 4;
  for (int b = 0; b < 2; ++b) {
    cudaEventRecord(ev_used[b], st);  // ordered after the model pack and earlier work on `stream`
    cudaEventRecord(ev_out[b], st);
  }
  int64_t idx = 0;
  for (int64_t off = 0; off < nq && e == cudaSuccess; off += chunk, ++idx) {
    const int b = (int)(idx & 1);
    const int64_t n = nq - off < chunk ? nq - off : chunk;
    // stage q once chunk idx-2 (the last user of buffer b) has been computed
    const float* qsrc = q + off * ldq;
    float* qdev = q_host ? buf[b].q : const_cast<float*>(qsrc);
    int64_t ldq_dev = q_host ? D : ldq;
    cudaStreamWaitEvent(h2d, ev_used[b], 0);
    if (q_host) {
      if (ldq == D) e = cudaMemcpyAsync(qdev, qsrc, (size_t)n * D * 4, cudaMemcpyHostToDevice, h2d);
      else e = cudaMemcpy2DAsync(qdev, (size_t)D * 4, qsrc, (size_t)ldq * 4, (size_t)D * 4, (size_t)n,
                                 cudaMemcpyHostToDevice, h2d);
    }
    cudaEventRecord(ev_in[b], h2d);
    // compute once q is staged and chunk idx-2's results have left buffer b
    cudaStreamWaitEvent(cs[b], ev_in[b], 0);
    cudaStreamWaitEvent(cs[b], ev_out[b], 0);
    float* sdev = score ? (s_host ? buf[b].sc : score + off) : nullptr;
    int8_t* ldev = label ? (l_host ? buf[b].lb : label + off) : nullptr;
    if (e == cudaSuccess && query_small_ok(nq, ns, M)) {  // one launch: FK inside the small-batch kernel
      e = launch_query_small(P, qdev, n, ldq_dev, packed, ns, M, k.kind, c, sdev, ldev, partials[b], cs[b]);
    } else {
      if (e == cudaSuccess) e = launch_fk(P, qdev, n, ldq_dev, reinterpret_cast<float4*>(buf[b].pos), chunk, cs[b]);
      if (e == cudaSuccess)
        e = launch_score(reinterpret_cast<const float4*>(buf[b].pos), n, chunk, packed, ns, M, k.kind, c, sdev, ldev,
                         partials[b], cs[b], nullptr, nq);
    }
    cudaEventRecord(ev_used[b], cs[b]);
    // results out
    cudaStreamWaitEvent(d2h, ev_used[b], 0);
    if (e == cudaSuccess && score && s_host) e = cudaMemcpyAsync(score + off, sdev, (size_t)n * 4, cudaMemcpyDeviceToHost, d2h);
    if (e == cudaSuccess && label && l_host) e = cudaMemcpyAsync(label + off, ldev, (size_t)n, cudaMemcpyDeviceToHost, d2h);
    cudaEventRecord(ev_out[b], d2h);
  }
  cudaStreamWaitEvent(st, ev_used[1], 0);  // `stream` ends after both compute streams
  cudaError_t e2 = cudaStreamSynchronize(h2d);
  cudaError_t e3 = cudaStreamSynchronize(d2h);
  cudaError_t e4 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = e3;
  if (e == cudaSuccess) e = e4;
  return cuda_status(e, "fastron_query");
}

size_t fastron_query_packed_workspace_bytes(int64_t nq, int64_t ns, int32_t n_cp, int32_t dof) {
  if (nq < 0 || ns < 0 || n_cp < 1 || n_cp > FASTRON_MAX_CP || dof < 1 || dof > FASTRON_MAX_DOF) return 0;
  const int64_t chunk = nq < kQueryChunk ? nq : kQueryChunk;
  return align_up(score_partial_bytes(chunk, ns, n_cp)) + align_up((size_t)chunk * n_cp * 16);
}

fastron_status fastron_query_packed(const fastron_robot* robot, const float* q, int64_t nq, int64_t ldq,
                                    const void* packed, int64_t ns, int32_t n_cp, fastron_kernel k, float* score,
                                    int8_t* label, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range_("fastron_query_packed");
  fastron_status s = check_robot(robot);
  if (s != FASTRON_OK) return s;
  s = check_kernel(k);
  if (s != FASTRON_OK) return s;
  FASTRON_REQUIRE(nq >= 0 && ns >= 0, "nq and ns must be >= 0");
  FASTRON_REQUIRE(n_cp == robot->n_cp, "n_cp (%d) differs from robot->n_cp (%d)", n_cp, robot->n_cp);
  if (nq == 0) return FASTRON_OK;
  FASTRON_REQUIRE(q != nullptr, "q is NULL");
  FASTRON_REQUIRE(!is_host_ptr(q) && !is_host_ptr(score) && !is_host_ptr(label),
                  "fastron_query_packed takes device buffers (fastron_query streams host buffers)");
  FASTRON_REQUIRE(score || label, "score and label are both NULL");
  FASTRON_REQUIRE(ldq >= robot->dof, "ldq (%lld) < dof (%d)", (long long)ldq, robot->dof);
  FASTRON_REQUIRE(ns == 0 || packed, "packed is NULL");
  FASTRON_REQUIRE(ns == 0 || ((uintptr_t)packed & 255) == 0, "packed must be 256-byte aligned (fastron_model_pack)");
  const int M = robot->n_cp, D = robot->dof;
  const size_t need = fastron_query_packed_workspace_bytes(nq, ns, M, D);
  if (workspace_bytes < need || (need > 0 && !workspace))
    return fail(FASTRON_ERR_WORKSPACE, "fastron_query_packed needs %zu workspace bytes, got %zu", need,
                workspace_bytes);
  FASTRON_REQUIRE(((uintptr_t)workspace & 255) == 0, "workspace must be 256-byte aligned");
  FASTRON_VALIDATE(vcheck_f32(q, nq, D, ldq, stream, "q"));
  const int64_t chunk = nq < kQueryChunk ? nq : kQueryChunk;
  double* partial = static_cast<double*>(workspace);
  float4* pos = reinterpret_cast<float4*>(static_cast<char*>(workspace) + align_up(score_partial_bytes(chunk, ns, M)));
  cudaStream_t st = S(stream);
  const float c = kernel_scale(k);
  const FkParams P = make_fk_params(*robot);
  const float* pk = static_cast<const float*>(packed);
  cudaError_t e = cudaSuccess;
  if (query_small_ok(nq, ns, M))
    return cuda_status(launch_query_small(P, q, nq, ldq, pk, ns, M, k.kind, c, score, label, partial, st),
                       "fastron_query_packed");
  for (int64_t off = 0; off < nq && e == cudaSuccess; off += chunk) {
    const int64_t n = nq - off < chunk ? nq - off : chunk;
    e = launch_fk(P, q + off * ldq, n, ldq, pos, chunk, st);
    if (e == cudaSuccess)
      e = launch_score(pos, n, chunk, pk, ns, M, k.kind, c, score ? score + off : nullptr,
                       label ? label + off : nullptr, partial, st, nullptr, nq);
  }
  return cuda_status(e, "fastron_query_packed");
}

}  // extern "C"
