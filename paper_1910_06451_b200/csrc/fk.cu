// fk.cu — K1, batched forward kinematics (Eq. 1-2).
//
// One thread per configuration, the fp64 chain of fk_device.cuh in registers, and
// coalesced SoA float4 stores pos[m][k] = (x, y, z, 0): for a fixed m consecutive
// threads write consecutive 16-byte elements. The roofline is HBM: per configuration
// 4*D bytes in + 16*M bytes out.
#include "internal.h"

namespace fastron {

#ifndef FASTRON_FK_THREADS
#define FASTRON_FK_THREADS 128
#endif
constexpr int kFkThreads = FASTRON_FK_THREADS;
#ifndef FASTRON_FK_CPT
#define FASTRON_FK_CPT 2
#endif
constexpr int kFkCpt = FASTRON_FK_CPT;  // configurations per thread

__global__ void __launch_bounds__(kFkThreads) fk_kernel(const __grid_constant__ FkParams P, const float* __restrict__ q,
                                                        int64_t n, int64_t ldq, float4* __restrict__ pos,
                                                        int64_t ldpos) {
  pdl_trigger();
  pdl_wait();
  if (kFkCpt == 1) {
    const int64_t k = (int64_t)blockIdx.x * kFkThreads + threadIdx.x;
    if (k >= n) return;
    const float* qk = q + k * ldq;
    fk_chain(
        P, [&](int j) { return (double)__ldg(qk + j); },
        [&](int m, double x, double y, double z) {
          pos[(int64_t)m * ldpos + k] =
              make_float4(__double2float_rn(x), __double2float_rn(y), __double2float_rn(z), 0.0f);
        });
  } else {
    // configuration c of this thread: k0 + c * kFkThreads (coalesced stores for each c);
    // slots past n recompute configuration n - 1 and store nothing
    const int64_t k0 = (int64_t)blockIdx.x * (kFkThreads * kFkCpt) + threadIdx.x;
    if (k0 >= n) return;
    fk_chain_multi<kFkCpt>(
        P,
        [&](int c, int j) {
          const int64_t k = min(k0 + (int64_t)c * kFkThreads, n - 1);
          return (double)__ldg(q + k * ldq + j);
        },
        [&](int c, int m, double x, double y, double z) {
          const int64_t k = k0 + (int64_t)c * kFkThreads;
          if (k < n)
            pos[(int64_t)m * ldpos + k] =
                make_float4(__double2float_rn(x), __double2float_rn(y), __double2float_rn(z), 0.0f);
        });
  }
}

cudaError_t launch_fk(const FkParams& P, const float* q, int64_t n, int64_t ldq, float4* pos, int64_t ldpos,
                      cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + kFkThreads * kFkCpt - 1) / (kFkThreads * kFkCpt);
  g_launches.fetch_add(1);
  return launch_pdl(fk_kernel, dim3((unsigned)blocks), dim3(kFkThreads), 0, st, P, q, n, ldq, pos, ldpos);
}

}  // namespace fastron
