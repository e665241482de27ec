// Probe: inner loop of the scoring kernel fed from shared memory (LDS -> registers) vs
// from the kernel-parameter constant bank (LDCU -> uniform registers, FADD2 R, R, UR).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) { f2 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(f2 v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float hi(f2 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { f2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { f2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ex2n(float x) { float r; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-x)); return r; }
__device__ __forceinline__ double cvt(float x) { uint32_t b = __float_as_uint(x); return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29)); }

constexpr int NS = 300, NP = 4, QT = 4;
struct Chunk { f2 rec[NS][NP][3]; double alpha[NS]; };

template <bool FROM_PARAM>
__global__ void __launch_bounds__(128) k(const __grid_constant__ Chunk C, const f2* __restrict__ gsup, int reps, double* out) {
  __shared__ f2 srec[NS][NP][3];
  __shared__ double salpha[NS];
  if (!FROM_PARAM) {
    for (int i = threadIdx.x; i < NS * NP * 3; i += blockDim.x) (&srec[0][0][0])[i] = gsup[i];
    for (int i = threadIdx.x; i < NS; i += blockDim.x) salpha[i] = 0.001 * i;
    __syncthreads();
  }
  f2 ux[QT][NP], uy[QT][NP], uz[QT][NP];
  for (int j = 0; j < QT; ++j)
    for (int p = 0; p < NP; ++p) {
      float b = 0.001f * (threadIdx.x + 7 * j + p);
      ux[j][p] = pk(b, b + 0.1f); uy[j][p] = pk(b * 0.5f, b); uz[j][p] = pk(0.2f, b);
    }
  double f[QT] = {0, 0, 0, 0};
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int s = 0; s < NS; ++s) {
      f2 acc[QT];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        f2 vx, vy, vz;
        if (FROM_PARAM) { vx = C.rec[s][p][0]; vy = C.rec[s][p][1]; vz = C.rec[s][p][2]; }
        else { vx = srec[s][p][0]; vy = srec[s][p][1]; vz = srec[s][p][2]; }
        f2 dx[QT], dy[QT], dz[QT];
#pragma unroll
        for (int j = 0; j < QT; ++j) dx[j] = sub2(ux[j][p], vx);
#pragma unroll
        for (int j = 0; j < QT; ++j) dy[j] = sub2(uy[j][p], vy);
#pragma unroll
        for (int j = 0; j < QT; ++j) dz[j] = sub2(uz[j][p], vz);
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          f2 q = mul2(dx[j], dx[j]); q = fma2(dy[j], dy[j], q); q = fma2(dz[j], dz[j], q);
          f2 t = pk(ex2n(lo(q)), ex2n(hi(q)));
          acc[j] = p == 0 ? t : add2(acc[j], t);
        }
      }
      const double a = FROM_PARAM ? C.alpha[s] : salpha[s];
#pragma unroll
      for (int j = 0; j < QT; ++j) { f[j] = fma(a, cvt(lo(acc[j])), f[j]); f[j] = fma(a, cvt(hi(acc[j])), f[j]); }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = f[0] + f[1] + f[2] + f[3];
}

int main() {
  static Chunk C;
  for (int s = 0; s < NS; ++s) { for (int p = 0; p < NP; ++p) for (int c = 0; c < 3; ++c) { float v = 0.01f * (s % 17) + c; unsigned long long b; float vv[2] = {v, v + 0.05f}; memcpy(&b, vv, 8); C.rec[s][p][c] = b; } C.alpha[s] = 0.001 * s; }
  f2* g; cudaMalloc(&g, sizeof(C.rec)); cudaMemcpy(g, C.rec, sizeof(C.rec), cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 148 * 64 * 128 * 8);
  int reps = 20;
  for (int v = 0; v < 2; ++v) {
    for (int w = 0; w < 2; ++w) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      const int grid = 148 * 3 * 8;
      if (v == 0) k<false><<<grid, 128>>>(C, g, reps, out); else k<true><<<grid, 128>>>(C, g, reps, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double mufu = (double)grid * 128 * QT * NS * NP * 2 * reps;
      if (w) printf("%s: %.3f ms, MUFU frac of 148x16x1.965GHz = %.3f (err %s)\n", v ? "param/UR" : "smem", ms, mufu / (ms * 1e-3) / (148 * 16 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
