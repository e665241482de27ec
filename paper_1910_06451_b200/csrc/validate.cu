// validate.cu — the optional content checks of the ABI (include/fastron.h,
// fastron_set_validation / FASTRON_VALIDATE=1). Hot-path calls do not inspect device
// array contents; with validation on, each entry point first counts non-finite values in
// its float inputs and labels outside {-1, +1}, synchronising the stream to read the
// count, and fails with FASTRON_ERR_INVALID_ARG if any is found. A debugging aid.
#include "internal.h"

namespace fastron {

__global__ void count_nonfinite_kernel(const float* __restrict__ a, int64_t rows, int64_t cols, int64_t ld,
                                       unsigned long long* __restrict__ bad) {
  unsigned long long n = 0;
  const int64_t total = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = a[(i / cols) * ld + i % cols];
    n += isfinite(v) ? 0 : 1;
  }
  if (n) atomicAdd(bad, n);
}

__global__ void count_nonfinite_f64_kernel(const double* __restrict__ a, int64_t n_el, unsigned long long* __restrict__ bad) {
  unsigned long long n = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_el; i += (int64_t)gridDim.x * blockDim.x)
    n += isfinite(a[i]) ? 0 : 1;
  if (n) atomicAdd(bad, n);
}

__global__ void count_bad_labels_kernel(const int8_t* __restrict__ y, int64_t n_el, unsigned long long* __restrict__ bad) {
  unsigned long long n = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_el; i += (int64_t)gridDim.x * blockDim.x)
    n += (y[i] == 1 || y[i] == -1) ? 0 : 1;
  if (n) atomicAdd(bad, n);
}

template <class Launch>
static cudaError_t run_count(cudaStream_t st, unsigned long long* out, Launch launch) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(*d), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(d, 0, sizeof(*d), st);
  if (e == cudaSuccess) {
    launch(d);
    g_launches.fetch_add(1);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, sizeof(*d), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}

static unsigned grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (unsigned)(b < 1 ? 1 : b > 4096 ? 4096 : b);
}

cudaError_t count_nonfinite(const float* a, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st,
                            unsigned long long* out) {
  *out = 0;
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  return run_count(st, out, [&](unsigned long long* d) {
    count_nonfinite_kernel<<<grid_for(rows * cols), 256, 0, st>>>(a, rows, cols, ld, d);
  });
}

cudaError_t count_nonfinite_f64(const double* a, int64_t n, cudaStream_t st, unsigned long long* out) {
  *out = 0;
  if (n <= 0) return cudaSuccess;
  return run_count(st, out, [&](unsigned long long* d) { count_nonfinite_f64_kernel<<<grid_for(n), 256, 0, st>>>(a, n, d); });
}

cudaError_t count_bad_labels(const int8_t* y, int64_t n, cudaStream_t st, unsigned long long* out) {
  *out = 0;
  if (n <= 0) return cudaSuccess;
  return run_count(st, out, [&](unsigned long long* d) { count_bad_labels_kernel<<<grid_for(n), 256, 0, st>>>(y, n, d); });
}

}  // namespace fastron
