// Probe: (1) MUFU.EX2 / MUFU.RCP error vs exact, (2) does F2F.F64.F32 contend with MUFU?
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void ex2_err(const float* x, float* y, float* r, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { float v; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(v) : "f"(-x[i])); y[i] = v;
               float w; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(1.0f + x[i])); r[i] = w; }
}
template <int CVT>
__global__ void __launch_bounds__(256) mix(float seed, int iters, float* out) {
  float v[8]; double acc[4] = {0, 0, 0, 0};
  for (int c = 0; c < 8; ++c) v[c] = seed * (threadIdx.x + c) * 1e-6f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
    if (CVT == 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(v[c])); acc[c] += d; }
    }
    if (CVT == 2) {
#pragma unroll
      for (int c = 0; c < 4; ++c) { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(v[c]));
        asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[c]) : "d"(d), "d"(1.0000001)); }
    }
  }
  float s = 0; for (int c = 0; c < 8; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)(acc[0] + acc[1] + acc[2] + acc[3]);
}
int main() {
  const int n = 1 << 24;
  float *x, *y, *r; cudaMallocManaged(&x, n * 4); cudaMallocManaged(&y, n * 4); cudaMallocManaged(&r, n * 4);
  for (int i = 0; i < n; ++i) x[i] = 40.0f * (float)i / n;
  ex2_err<<<n / 256, 256>>>(x, y, r, n); cudaDeviceSynchronize();
  double mx = 0, mean = 0, mxr = 0, meanr = 0; int cnt = 0;
  for (int i = 0; i < n; ++i) {
    double ref = exp2(-(double)x[i]);
    if (ref < 1e-30) continue;
    double e = ((double)y[i] - ref) / ref; mx = fmax(mx, fabs(e)); mean += e;
    double rr = 1.0 / (1.0 + (double)x[i]); double er = ((double)r[i] - rr) / rr; mxr = fmax(mxr, fabs(er)); meanr += er; ++cnt;
  }
  printf("{\"ex2_max_rel\": %.3e, \"ex2_mean_rel\": %.3e, \"rcp_max_rel\": %.3e, \"rcp_mean_rel\": %.3e, \"ulp\": %.3e", mx, mean / cnt, mxr, meanr / cnt, ldexp(1.0, -23));
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  const char* names[] = {"mufu_only", "mufu+cvt(4/8)", "mufu+cvt+dfma(4/8)"};
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a);
      if (k == 0) mix<0><<<148 * 8, 256>>>(1.0001f, 4096, out);
      if (k == 1) mix<1><<<148 * 8, 256>>>(1.0001f, 4096, out);
      if (k == 2) mix<2><<<148 * 8, 256>>>(1.0001f, 4096, out);
      cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf(", \"%s_ms\": %.3f, \"%s_mufu_per_clk_sm\": %.2f", names[k], ms, names[k], 148.0 * 8 * 256 * 4096 * 8 / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  printf("}\n");
  return 0;
}
