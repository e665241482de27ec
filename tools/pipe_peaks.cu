// Microbenchmark: per-SM throughput of the pipes the FK-kernel scoring path uses
// (MUFU.EX2, MUFU.RCP, FFMA, FFMA2/FADD2, DADD/DFMA) and the fused term sequence.
// Prints ops/clk/SM using clock64 + globaltimer (so the SM clock is measured, not assumed).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_1910_06451_b200/csrc/fastron_device.cuh"

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint64_t gtimer(){ uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;}
__device__ __forceinline__ void upk(unsigned long long v, float& a, float& b){ asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }

struct Rec { unsigned long long clk0, clk1, t0, t1; };

#define CHAINS 8
template <int OP>
__global__ void __launch_bounds__(256) bench(float seed, int iters, float* out, Rec* rec) {
  float v[CHAINS]; unsigned long long p[CHAINS]; double dv[CHAINS];
  for (int c = 0; c < CHAINS; ++c) { v[c] = seed * (threadIdx.x + c + 1) * 1e-7f; p[c] = pk(v[c], v[c] + 1e-7f); dv[c] = v[c]; }
  __syncthreads();
  unsigned long long c0 = clock64(); uint64_t t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
      if (OP == 1) {  // rcp(rcp(x)) folds away (round 1 measured an impossible 2,120/clk): perturb
        asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(v[c]) : "f"(seed));
      }
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[c]) : "f"(seed), "f"(v[(c+1)%CHAINS]));
      if (OP == 3) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(p[(c+3)%CHAINS]), "l"(p[(c+1)%CHAINS]));
      if (OP == 4) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(p[(c+1)%CHAINS]));
      if (OP == 5) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(dv[c]) : "d"(dv[(c+1)%CHAINS]));
      if (OP == 6) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dv[c]) : "d"(dv[(c+3)%CHAINS]), "d"(dv[(c+1)%CHAINS]));
      if (OP == 7) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(v[c]) : "f"(v[(c+1)%CHAINS]));
    }
  }
  unsigned long long c1 = clock64(); uint64_t t1 = gtimer();
  float s = 0.f; double ds = 0.0;
  for (int c = 0; c < CHAINS; ++c) { float a, b; upk(p[c], a, b); s += v[c] + a + b; ds += dv[c]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)ds;
  if (threadIdx.x == 0) rec[blockIdx.x] = Rec{c0, c1, t0, t1};
}

// The fused Gaussian term on an m-pair, as the scoring kernel issues it:
// 3 FADD2 + FMUL2 + 2 FFMA2 + 2 MUFU.EX2 + 1 FADD2 per 2 terms.
__global__ void __launch_bounds__(256) bench_term(float seed, int iters, float* out, Rec* rec) {
  unsigned long long ux[4], uy[4], uz[4], acc[4];
  for (int c = 0; c < 4; ++c) { float b = seed * (threadIdx.x + c); ux[c] = pk(b, b + 0.1f); uy[c] = pk(b * 0.5f, b); uz[c] = pk(b * 0.25f, b); acc[c] = 0ull; }
  unsigned long long vx = pk(0.1f, 0.2f), vy = pk(0.3f, 0.1f), vz = pk(0.2f, 0.4f);
  __syncthreads();
  unsigned long long c0 = clock64(); uint64_t t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      unsigned long long dx, dy, dz, s;
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(ux[c]), "l"(vx));
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(uy[c]), "l"(vy));
      asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(uz[c]), "l"(vz));
      asm volatile("mul.rn.f32x2 %0, %1, %1;" : "=l"(s) : "l"(dx));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(s) : "l"(dy));
      asm volatile("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(s) : "l"(dz));
      float a, b; upk(s, a, b);
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[c]) : "l"(pk(a, b)));
    }
    vx ^= 1ull; vy ^= 1ull;  // keep the loop from being hoisted
  }
  unsigned long long c1 = clock64(); uint64_t t1 = gtimer();
  float s = 0.f; for (int c = 0; c < 4; ++c) { float a, b; upk(acc[c], a, b); s += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = Rec{c0, c1, t0, t1};
}

// Same term with scalar FP32 ops: 3 FADD + FMUL + 2 FFMA + MUFU.EX2 + FADD per term.
__global__ void __launch_bounds__(256) bench_term_scalar(float seed, int iters, float* out, Rec* rec) {
  float ux[8], uy[8], uz[8], acc[8];
  for (int c = 0; c < 8; ++c) { float b = seed * (threadIdx.x + c); ux[c] = b; uy[c] = b * 0.5f; uz[c] = b * 0.25f; acc[c] = 0.f; }
  float vx = 0.1f, vy = 0.3f, vz = 0.2f;
  __syncthreads();
  unsigned long long c0 = clock64(); uint64_t t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float dx, dy, dz, s;
      asm volatile("sub.rn.f32 %0, %1, %2;" : "=f"(dx) : "f"(ux[c]), "f"(vx));
      asm volatile("sub.rn.f32 %0, %1, %2;" : "=f"(dy) : "f"(uy[c]), "f"(vy));
      asm volatile("sub.rn.f32 %0, %1, %2;" : "=f"(dz) : "f"(uz[c]), "f"(vz));
      asm volatile("mul.rn.f32 %0, %1, %1;" : "=f"(s) : "f"(dx));
      asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(s) : "f"(dy));
      asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(s) : "f"(dz));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(s));
      asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[c]) : "f"(s));
    }
    vx += 1e-9f; vy -= 1e-9f;
  }
  unsigned long long c1 = clock64(); uint64_t t1 = gtimer();
  float s = 0.f; for (int c = 0; c < 8; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec[blockIdx.x] = Rec{c0, c1, t0, t1};
}

// The product's term function (fastron_device.cuh accum_term) on 4 control-point pairs x
// QT = 3 queries per support, as the scoring kernel issues it; KIND 0 = Gaussian (7 packed
// FP32 ops + 2 MUFU per pair), 1 = RQ with the Newton step (11 + 2). The support operand
// changes every iteration (no hoisting); the accumulators are written out (no dead code).
template <int KIND>
__global__ void __launch_bounds__(128) bench_accum(float seed, int iters, float* out, Rec* rec) {
  fastron::f2 ux[3][4], uy[3][4], uz[3][4];
  for (int j = 0; j < 3; ++j)
    for (int p = 0; p < 4; ++p) {
      const float b = seed * (threadIdx.x + 7 * j + p) * 1e-3f;
      ux[j][p] = fastron::pk(b, b + 0.1f); uy[j][p] = fastron::pk(0.5f * b, b); uz[j][p] = fastron::pk(0.25f * b, 0.3f);
    }
  fastron::f2 vx = fastron::pk(0.1f, 0.2f), vy = fastron::pk(0.3f, 0.1f), vz = fastron::pk(0.2f, 0.4f);
  const fastron::f2 dv = fastron::pk(1e-6f, -1e-6f);
  double f[3] = {0.0, 0.0, 0.0};
  __syncthreads();
  unsigned long long c0 = clock64(); uint64_t t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
    fastron::f2 acc[3];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        fastron::accum_term<KIND>(acc[j], fastron::sub2(ux[j][p], vx), fastron::sub2(uy[j][p], vy), fastron::sub2(uz[j][p], vz), p == 0);
#pragma unroll
    for (int j = 0; j < 3; ++j) f[j] += (double)fastron::lo(acc[j]) + (double)fastron::hi(acc[j]);
    vx = fastron::add2(vx, dv); vy = fastron::add2(vy, dv); vz = fastron::add2(vz, dv);
  }
  unsigned long long c1 = clock64(); uint64_t t1 = gtimer();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(f[0] + f[1] + f[2]);
  if (threadIdx.x == 0) rec[blockIdx.x] = Rec{c0, c1, t0, t1};
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", prop.name, sms);
  const int blocks = sms * 4, threads = 256, iters = 4096;
  float* out; Rec* rec; CK(cudaMalloc(&out, blocks * threads * 4)); CK(cudaMalloc(&rec, blocks * sizeof(Rec)));
  Rec* h = new Rec[blocks];
  const char* names[] = {"mufu_ex2", "mufu_rcp", "ffma", "ffma2", "fadd2", "dadd", "dfma", "fadd", "term_pair",
                         "term_scalar", "accum_gaussian_terms", "accum_rq_newton_terms"};
  for (int op = 0; op < 12; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      switch (op) {
        case 0: bench<0><<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 1: bench<1><<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 2: bench<2><<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 3: bench<3><<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 4: bench<4><<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 5: bench<5><<<blocks, threads>>>(1.0001f, iters / 4, out, rec); break;
        case 6: bench<6><<<blocks, threads>>>(1.0001f, iters / 4, out, rec); break;
        case 7: bench<7><<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 8: bench_term<<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 9: bench_term_scalar<<<blocks, threads>>>(1.0001f, iters, out, rec); break;
        case 10: bench_accum<0><<<blocks, 128>>>(1.0001f, iters / 4, out, rec); break;
        case 11: bench_accum<1><<<blocks, 128>>>(1.0001f, iters / 4, out, rec); break;
      }
      CK(cudaGetLastError());
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      CK(cudaMemcpy(h, rec, blocks * sizeof(Rec), cudaMemcpyDeviceToHost));
      if (rep == 0) continue;
      double clk = 0, ns = 0;
      for (int b = 0; b < blocks; ++b) { clk += (double)(h[b].clk1 - h[b].clk0); ns += (double)(h[b].t1 - h[b].t0); }
      clk /= blocks; ns /= blocks;
      double mhz = clk / ns * 1e3;
      int it = (op == 5 || op == 6 || op >= 10) ? iters / 4 : iters;
      double ops_per_block = (double)threads * it * (op >= 8 ? 8 : CHAINS);  // op 8: 4 pairs x 2 MUFU terms
      if (op >= 10) ops_per_block = 128.0 * it * 24;  // 3 queries x 8 terms (one MUFU each) per iteration
      // blocks resident 4/SM (256 thr, low regs) -> per-SM ops per clock = 4 * ops_per_block / clk
      // per-SM rate from the event time and the measured clock (robust to residency)
      double per_sm_clk = (double)blocks * ops_per_block / (ms * 1e-3) / sms / (mhz * 1e6);
      double total_rate = (double)blocks * ops_per_block / (ms * 1e-3);
      printf(", \"%s\": {\"ops_per_clk_per_sm\": %.2f, \"sm_mhz\": %.0f, \"Gops\": %.1f, \"ms\": %.3f}", names[op], per_sm_clk, mhz, total_rate * 1e-9, ms);
    }
  }
  printf("}\n");
  return 0;
}
