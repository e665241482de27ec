// fk.cu — K1, batched forward kinematics (Eq. 1-2).
//
// One thread per configuration, the fp64 chain of fk_device.cuh in registers, and
// coalesced SoA float4 stores pos[m][k] = (x, y, z, 0): for a fixed m consecutive
// threads write consecutive 16-byte elements. The roofline is HBM: per configuration
// 4*D bytes in + 16*M bytes out.
#include "internal.h"

namespace fastron {

constexpr int kFkThreads = 256;

__global__ void __launch_bounds__(kFkThreads) fk_kernel(const __grid_constant__ FkParams P, const float* __restrict__ q,
                                                        int64_t n, int64_t ldq, float4* __restrict__ pos,
                                                        int64_t ldpos) {
  const int64_t k = (int64_t)blockIdx.x * kFkThreads + threadIdx.x;
  if (k >= n) return;
  const float* qk = q + k * ldq;
  fk_chain(
      P, [&](int j) { return (double)__ldg(qk + j); },
      [&](int m, double x, double y, double z) {
        pos[(int64_t)m * ldpos + k] =
            make_float4(__double2float_rn(x), __double2float_rn(y), __double2float_rn(z), 0.0f);
      });
}

cudaError_t launch_fk(const FkParams& P, const float* q, int64_t n, int64_t ldq, float4* pos, int64_t ldpos,
                      cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + kFkThreads - 1) / kFkThreads;
  fk_kernel<<<(unsigned)blocks, kFkThreads, 0, st>>>(P, q, n, ldq, pos, ldpos);
  g_launches.fetch_add(1);
  return cudaGetLastError();
}

}  // namespace fastron
