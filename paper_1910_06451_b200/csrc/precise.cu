// precise.cu — the fp64 scoring path for ill-conditioned models (R25).
//
// A model trained by Algorithm 1 has weights of both signs and
// magnitudes up to ~200, so f(x) = sum_i alpha_i K_FK(S_i, x) is a
// cancelling sum: fp32 positions and fp32 terms perturb it by ~1e-5..1e-4, above the
// 1e-5 floor near the decision boundary — exactly where a collision checker needs the sign.
// This path keeps everything in fp64: the D-H chain's positions are stored unrounded
// (fk64_kernel, SoA double4 [M][ldpos] = (x, y, z, 0)), the weights stay fp64 (as
// Algorithm 1 produced them), and every term of Eq. 3/4 and every sum is fp64:
//   Gaussian  exp(-gamma d^2)          (CUDA's fp64 exp)
//   RQ        (1 + gamma/2 d^2)^-2      (fp64 division)
// score64_kernel: one query per thread with its M control points in registers; supports
// stream through shared memory in tiles of 64 (structure of arrays, warp-broadcast reads);
// the score is sum_i alpha_i ((1/M) sum_m t_m) in support order. The fp64 pipe
// (~40 DFMA/clk/SM measured) bounds it: ~25 fp64 operations per term against one MUFU
// op per term on the fp32 path — an opt-in accuracy mode, not the hot path.
#include "fastron_device.cuh"
#include "internal.h"

namespace fastron {

__global__ void __launch_bounds__(128) fk64_kernel(const __grid_constant__ FkParams P, const float* __restrict__ q,
                                                   int64_t n, int64_t ldq, double4* __restrict__ pos, int64_t ldpos) {
  const int64_t k = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (k >= n) return;
  const float* qk = q + k * ldq;
  fk_chain(
      P, [&](int j) { return (double)__ldg(qk + j); },
      [&](int m, double x, double y, double z) { pos[(int64_t)m * ldpos + k] = make_double4(x, y, z, 0.0); });
}

cudaError_t launch_fk64(const FkParams& P, const float* q, int64_t n, int64_t ldq, double4* pos, int64_t ldpos,
                        cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fk64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(P, q, n, ldq, pos, ldpos);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

constexpr int kP64NT = 128;
constexpr int kP64Tile = 64;

template <int MMAX, int KIND>
__global__ void __launch_bounds__(kP64NT) score64_kernel(const double4* __restrict__ qpos, int64_t nq, int64_t ldq,
                                                         const double4* __restrict__ spos, const double* __restrict__ alpha,
                                                         int64_t ns, int64_t lds, int M, double gamma,
                                                         double* __restrict__ score, int8_t* __restrict__ label) {
  __shared__ double s_sup[MMAX * 3][kP64Tile];  // structure of arrays: [m * 3 + c][support]
  __shared__ double s_alpha[kP64Tile];
  const int tid = threadIdx.x;
  const int64_t q = (int64_t)blockIdx.x * kP64NT + tid;
  double ux[MMAX], uy[MMAX], uz[MMAX];
#pragma unroll
  for (int m = 0; m < MMAX; ++m) {
    double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
    if (m < M && q < nq) v = qpos[(int64_t)m * ldq + q];
    ux[m] = v.x; uy[m] = v.y; uz[m] = v.z;
  }
  const double hg = 0.5 * gamma;
  const double inv_m = 1.0 / (double)M;
  double f = 0.0;
  for (int64_t t0 = 0; t0 < ns; t0 += kP64Tile) {
    const int nt = (int)min((int64_t)kP64Tile, ns - t0);
    __syncthreads();  // the previous tile is consumed
    for (int i = tid; i < M * nt; i += kP64NT) {
      const int m = i / nt, s = i % nt;
      const double4 v = spos[(int64_t)m * lds + t0 + s];
      s_sup[m * 3 + 0][s] = v.x;
      s_sup[m * 3 + 1][s] = v.y;
      s_sup[m * 3 + 2][s] = v.z;
    }
    for (int s = tid; s < nt; s += kP64NT) s_alpha[s] = alpha[t0 + s];
    __syncthreads();
    for (int s = 0; s < nt; ++s) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < MMAX; ++m) {
        if (m < M) {
          const double dx = ux[m] - s_sup[m * 3 + 0][s];
          const double dy = uy[m] - s_sup[m * 3 + 1][s];
          const double dz = uz[m] - s_sup[m * 3 + 2][s];
          const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
          double t;
          if (KIND == kGaussian) {
            t = exp(-gamma * d2);
          } else {
            const double w = fma(hg, d2, 1.0);
            t = 1.0 / (w * w);
          }
          acc += t;
        }
      }
      f = fma(s_alpha[s], acc * inv_m, f);
    }
  }
  if (q < nq) {
    if (score) score[q] = f;
    if (label) label[q] = f > 0.0 ? 1 : -1;
  }
}

cudaError_t launch_score64(const double4* qpos, int64_t nq, int64_t ldq, const double4* spos, const double* alpha,
                           int64_t ns, int64_t lds, int M, int kind, double gamma, double* score, int8_t* label,
                           cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((nq + kP64NT - 1) / kP64NT);
#define FASTRON_P64(mm)                                                                                          \
  if (M <= mm) {                                                                                                 \
    if (kind == kGaussian)                                                                                       \
      score64_kernel<mm, kGaussian><<<grid, kP64NT, 0, st>>>(qpos, nq, ldq, spos, alpha, ns, lds, M, gamma, score, \
                                                             label);                                            \
    else                                                                                                         \
      score64_kernel<mm, kRQ><<<grid, kP64NT, 0, st>>>(qpos, nq, ldq, spos, alpha, ns, lds, M, gamma, score, label); \
    g_launches.fetch_add(1);                                                                                     \
    return cudaGetLastError();                                                                                   \
  }
  FASTRON_P64(4)
  FASTRON_P64(8)
  FASTRON_P64(16)
#undef FASTRON_P64
  return cudaErrorInvalidValue;
}

}  // namespace fastron
