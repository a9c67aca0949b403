// Microbenchmark: tcgen05.ld throughput (TMEM -> registers) per SM, for 4 / 8 / 16 warps and the
// 32x32b.x32 / .x16 / .x64 shapes.  One CTA, 512 TMEM columns; every warp reads its own lane quarter.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2603_08982_b200/csrc/tc_common.cuh"
using namespace svg::tc;

#define TMEM_LD64(taddr, r)                                                                        \
  asm volatile(                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "                                                    \
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "                    \
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "           \
      "%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "           \
      "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"    \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), \
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), \
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63]) \
      : "r"(taddr) : "memory")

template <int SHAPE>
__global__ void k(float* out, long long* clk, int reps) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(smem_u32(&slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + (((uint32_t)((warp & 3) * 32)) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const uint32_t col = (uint32_t)(((r + warp) * 64) & 511);
    if (SHAPE == 32) {
      uint32_t a[32], b[32];
      TMEM_LD32(tmem + (col & 448), a);
      TMEM_LD32(tmem + (col & 448) + 32, b);
      tc_wait_ld();
      acc += a[0] ^ b[31];
    } else {
      uint32_t a[64];
      TMEM_LD64(tmem + (col & 448), a);
      tc_wait_ld();
      acc += a[0] ^ a[63];
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = (float)acc;
  if (threadIdx.x == 0) clk[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 4096); cudaMalloc(&clk, 64);
  const int reps = 4000;
  for (int shape : {32, 64})
    for (int warps : {4, 8, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (shape == 32) k<32><<<1, warps * 32>>>(out, clk, reps); else k<64><<<1, warps * 32>>>(out, clk, reps);
      }
      cudaError_t e = cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)reps * warps * 32 * 64 * 4;  // 64 columns x 32 lanes x 4 B per warp per rep
      printf("shape x%d, %2d warps: %8lld clk, %6.1f B/clk/SM  (%s)\n", shape, warps, h, bytes / (double)h, cudaGetErrorString(e));
    }
  return 0;
}
