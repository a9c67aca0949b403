// Microbenchmark: does MUFU.EX2 overlap with FFMA / FFMA2 issue on one SM sub-partition?  Each loop
// iteration issues 16 independent MUFU.EX2 and NF independent FFMA (or FFMA2); prints clk per iteration
// per sub-partition for 1 / 2 / 4 warps per sub-partition.  max(128, NF) = full overlap, 128 + NF = none.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mufu_overlap mufu_overlap.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2603_08982_b200/csrc/tc_common.cuh"
using namespace svg::tc;

template <int NM, int NF, int PACKED>
__global__ void k(float* out, long long* clk, float seed, int reps) {
  float m[16], f[16];
  uint64_t g[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    m[i] = seed * (i + 1) + threadIdx.x * 1e-3f;
    f[i] = seed * (i + 3);
    g[i] = pack2(f[i], m[i]);
  }
  const float c0 = seed * 0.5f, c1 = seed * 0.25f;
  const uint64_t c2 = pack2(c0, c1), c3 = pack2(c1, c0);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (u < NM) m[u] = ex2(m[u]);
#pragma unroll
      for (int j = 0; j < NF / 16; ++j) {
        if (PACKED) g[(u + j) & 15] = ffma2(g[(u + j) & 15], c2, c3);
        else f[(u + j) & 15] = fmaf(f[(u + j) & 15], c0, c1);
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float a, b;
    unpack2(g[i], a, b);
    acc += m[i] + f[i] + a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[0] = t1 - t0;
}

template <int NM, int NF, int PACKED>
void run() {
  float* out; long long* clk;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&clk, 64);
  const int reps = 2000;
  printf("MUFU %2d + %s %3d:", NM, PACKED ? "FFMA2" : "FFMA ", NF);
  for (int w : {1, 2, 4}) {
    k<NM, NF, PACKED><<<1, 128 * w>>>(out, clk, 0.37f, reps);
    k<NM, NF, PACKED><<<1, 128 * w>>>(out, clk, 0.37f, reps);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("  w=%d: %6.1f clk/iter", w, (double)h / reps);
  }
  printf("\n");
  cudaFree(out); cudaFree(clk);
}

int main() {
  run<16, 0, 0>(); run<0, 64, 0>(); run<0, 128, 0>(); run<0, 64, 1>(); run<0, 128, 1>();
  run<16, 32, 0>(); run<16, 64, 0>(); run<16, 128, 0>(); run<16, 256, 0>();
  run<16, 32, 1>(); run<16, 64, 1>(); run<16, 128, 1>();
  return 0;
}
