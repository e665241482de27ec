// Probe: throughput of the scoring inner loop variants (smem-fed supports, M = 8).
//   PACKED: f32x2 instructions vs scalar FP32; F64: per-support fp64 accumulation vs fp32
//   partial; QT: queries per thread. Prints the achieved fraction of the MUFU roofline.
#include <cstdio>
#include <cstdint>
#include <cstring>
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

constexpr int NS = 256, NP = 4;

template <bool PACKED, bool F64, int QT>
__global__ void __launch_bounds__(128) k(const float* __restrict__ gsup, int reps, double* out) {
  __shared__ __align__(16) float srec[NS][NP][8];
  __shared__ double salpha[NS];
  for (int i = threadIdx.x; i < NS * NP * 8; i += blockDim.x) (&srec[0][0][0])[i] = gsup[i];
  for (int i = threadIdx.x; i < NS; i += blockDim.x) salpha[i] = 0.001 * i;
  __syncthreads();
  float qx[QT][8], qy[QT][8], qz[QT][8];
  for (int j = 0; j < QT; ++j)
    for (int m = 0; m < 8; ++m) { float b = 0.001f * (threadIdx.x + 7 * j + m); qx[j][m] = b; qy[j][m] = 0.5f * b; qz[j][m] = 0.2f + b; }
  double f[QT];
  float fp[QT];
  for (int j = 0; j < QT; ++j) { f[j] = 0; fp[j] = 0; }
  for (int r = 0; r < reps; ++r) {
#pragma unroll 2
    for (int s = 0; s < NS; ++s) {
      float ev[QT], od[QT];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float4 xy = *reinterpret_cast<const float4*>(&srec[s][p][0]);
        const float2 zz = *reinterpret_cast<const float2*>(&srec[s][p][4]);
#pragma unroll
        for (int j = 0; j < QT; ++j) {
          float t0, t1;
          if (PACKED) {
            f2 dx = sub2(pk(qx[j][2 * p], qx[j][2 * p + 1]), pk(xy.x, xy.y));
            f2 dy = sub2(pk(qy[j][2 * p], qy[j][2 * p + 1]), pk(xy.z, xy.w));
            f2 dz = sub2(pk(qz[j][2 * p], qz[j][2 * p + 1]), pk(zz.x, zz.y));
            f2 q = mul2(dx, dx); q = fma2(dy, dy, q); q = fma2(dz, dz, q);
            t0 = ex2n(lo(q)); t1 = ex2n(hi(q));
            if (p == 0) { ev[j] = t0; od[j] = t1; }
            else { f2 a = add2(pk(ev[j], od[j]), pk(t0, t1)); ev[j] = lo(a); od[j] = hi(a); }
          } else {
            float dx0 = qx[j][2 * p] - xy.x, dy0 = qy[j][2 * p] - xy.z, dz0 = qz[j][2 * p] - zz.x;
            float dx1 = qx[j][2 * p + 1] - xy.y, dy1 = qy[j][2 * p + 1] - xy.w, dz1 = qz[j][2 * p + 1] - zz.y;
            float q0 = dx0 * dx0; q0 = fmaf(dy0, dy0, q0); q0 = fmaf(dz0, dz0, q0);
            float q1 = dx1 * dx1; q1 = fmaf(dy1, dy1, q1); q1 = fmaf(dz1, dz1, q1);
            t0 = ex2n(q0); t1 = ex2n(q1);
            if (p == 0) { ev[j] = t0; od[j] = t1; } else { ev[j] += t0; od[j] += t1; }
          }
        }
      }
      const double a = salpha[s];
#pragma unroll
      for (int j = 0; j < QT; ++j) {
        if (F64) { f[j] = fma(a, cvt(ev[j]), f[j]); f[j] = fma(a, cvt(od[j]), f[j]); }
        else fp[j] = fmaf((float)0.001f, ev[j] + od[j], fp[j]);
      }
    }
  }
  double o = 0; for (int j = 0; j < QT; ++j) o += f[j] + fp[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = o;
}

template <bool PACKED, bool F64, int QT>
void run(const char* name, const float* g, double* out) {
  int reps = 24 / QT * 4;
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<PACKED, F64, QT>, 128, 0);
  cudaFuncAttributes at; cudaFuncGetAttributes(&at, k<PACKED, F64, QT>);
  const int grid = 148 * occ * 6;
  for (int w = 0; w < 2; ++w) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<PACKED, F64, QT><<<grid, 128>>>(g, reps, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double mufu = (double)grid * 128 * QT * NS * 8 * reps;
    if (w) printf("%-28s regs %3d occ %d  %.3f ms  MUFU frac %.3f\n", name, at.numRegs, occ, ms, mufu / (ms * 1e-3) / (148 * 16 * 1.965e9));
  }
}

int main() {
  static float h[NS * NP * 8];
  for (int i = 0; i < NS * NP * 8; ++i) h[i] = 0.001f * (i % 97);
  float* g; cudaMalloc(&g, sizeof(h)); cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, (size_t)148 * 32 * 6 * 128 * 8);
  run<true, true, 4>("packed f64acc QT=4", g, out);
  run<false, true, 4>("scalar f64acc QT=4", g, out);
  run<true, false, 4>("packed f32acc QT=4", g, out);
  run<false, false, 4>("scalar f32acc QT=4", g, out);
  run<true, true, 2>("packed f64acc QT=2", g, out);
  run<false, true, 2>("scalar f64acc QT=2", g, out);
  run<true, true, 8>("packed f64acc QT=8", g, out);
  run<false, true, 8>("scalar f64acc QT=8", g, out);
  run<true, true, 6>("packed f64acc QT=6", g, out);
  run<true, true, 3>("packed f64acc QT=3", g, out);
  return 0;
}
