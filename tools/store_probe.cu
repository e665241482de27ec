// Store-pattern probe for K3: write an n x n fp32 matrix with
//   P1 coalesced float4 rows (ideal), P2 the column-slot Gram pattern (128 consecutive floats
//   per row and column slot, plus 16-byte mirror segments of 4 rows for 32 columns per warp),
//   P3 only its mirror segments, P4 only its direct rows, P5 mirror segments of 8 rows (32 B),
//   with no arithmetic; prints GB/s of the n^2 * 4 bytes each pattern writes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_probe tools/store_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void p1(float4* K, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    K[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

// units as the Gram's: column block b (384 columns) x row tile (64 rows), upper triangle + diagonal
template <int MODE, int CH>
__global__ void __launch_bounds__(128) pg(float* K, int64_t n, int64_t nb) {
  // unit -> (b, t) over the triangle of 6-tile blocks: block b has 6 (b + 1) tiles
  int64_t u = blockIdx.x, b = 0;
  while (6 * (b + 1) <= u) { u -= 6 * (b + 1); ++b; }
  const int64_t j0 = b * 384, r0 = u * 64;
  const bool mirror = r0 < j0;
  const int tid = threadIdx.x;
  float v[CH][3];
  for (int c4 = 0; c4 < 64; c4 += CH) {
#pragma unroll
    for (int rr = 0; rr < CH; ++rr)
#pragma unroll
      for (int j = 0; j < 3; ++j) v[rr][j] = (float)(r0 + c4 + rr) + j;
    if (MODE & 1) {
#pragma unroll
      for (int rr = 0; rr < CH; ++rr)
#pragma unroll
        for (int j = 0; j < 3; ++j) K[(r0 + c4 + rr) * n + j0 + j * 128 + tid] = v[rr][j];
    }
    if ((MODE & 2) && mirror) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float* p = K + (j0 + j * 128 + tid) * n + r0 + c4;
#pragma unroll
        for (int q = 0; q < CH; q += 4) *reinterpret_cast<float4*>(p + q) = make_float4(v[q][j], v[q + 1][j], v[q + 2][j], v[q + 3][j]);
      }
    }
  }
}

int main() {
  const int64_t n = 19968;  // 52 blocks of 384
  const int64_t nb = n / 384;
  float* K;
  cudaMalloc(&K, n * n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int64_t units = 6 * nb * (nb + 1) / 2;
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-34s %8.3f ms  %7.1f GB/s (n^2 x 4 B)\n", name, ms, n * n * 4.0 / ms * 1e-6);
  };
  run("P1 coalesced float4 rows", [&] { p1<<<148 * 8, 256>>>((float4*)K, n * n / 4); });
  run("P2 gram direct + mirror (4 rows)", [&] { pg<3, 4><<<units, 128>>>(K, n, nb); });
  run("P3 gram mirror only (4 rows)", [&] { pg<2, 4><<<units, 128>>>(K, n, nb); });
  run("P4 gram direct only", [&] { pg<1, 4><<<units, 128>>>(K, n, nb); });
  run("P5 gram direct + mirror (8 rows)", [&] { pg<3, 8><<<units, 128>>>(K, n, nb); });
  run("P6 gram direct + mirror (16 rows)", [&] { pg<3, 16><<<units, 128>>>(K, n, nb); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
