// Microbenchmark: tcgen05.mma issue-to-completion rate per SM for SS / TS operands and M = 64 / 128,
// N = 64 / 128 / 256 (kind::f16, K = 16 per instruction).  One CTA per SM, one elected thread issues
// REPS x 8 MMAs (8 k-steps over 128-wide operands in shared memory, garbage data) and waits for the
// commit; prints clk per MMA.  Answers: does M = 64 cost half of M = 128?  How far is SS QK^T at N = 64
// from its MMA floor (shared-memory operand bandwidth)?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu -lcuda
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2603_08982_b200/csrc/tc_common.cuh"
using namespace svg::tc;

__global__ void __launch_bounds__(128) k(long long* clk, int M, int N, int ts, int reps) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA = smem_u32(smem), sB = sA + 128 * 128 * 2, bar = sB + 256 * 128 * 2;
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 128 * 128 * 2 + 256 * 128 * 2 + 64);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(smem_u32(slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1 && elect_one()) {
    const uint32_t idesc = make_idesc(M, N, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t ad = make_desc(sA + (uint32_t)((kk >> 2) * (128 * 128) + (kk & 3) * 32), 16, 1024);
        const uint64_t bd = make_desc(sB + (uint32_t)((kk >> 2) * (256 * 128) + (kk & 3) * 32), 16, 1024);
        if (ts == 1) umma_ts(tmem, tmem + 256 + (uint32_t)(kk * 8), bd, idesc, kk > 0);
        else if (ts == 0) umma_ss(tmem, ad, bd, idesc, kk > 0);
        else {  // ts == 2: SS, two independent accumulations interleaved k-step by k-step (A and D differ)
          umma_ss(tmem, ad, bd, idesc, kk > 0);
          const uint64_t ad2 = make_desc(sA + 64 * 128 + (uint32_t)((kk >> 2) * (128 * 128) + (kk & 3) * 32), 16, 1024);
          umma_ss(tmem + 256, ad2, bd, idesc, kk > 0);
        }
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) clk[0] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* clk; cudaMalloc(&clk, 64);
  const size_t smem = 1024 + 128 * 128 * 2 + 256 * 128 * 2 + 256;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 2000;
  for (int ts = 0; ts < 3; ++ts)
    for (int M : {64, 128})
      for (int N : {32, 64, 128, 256}) {
        k<<<148, 128, smem>>>(clk, M, N, ts, reps);
        cudaError_t e = cudaDeviceSynchronize();
        long long h = 0; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
        printf("%s M=%3d N=%3d: %7.1f clk per MMA (floor 128*N/256 = %d)%s\n",
               ts == 0 ? "SS" : (ts == 1 ? "TS" : "SS two interleaved accumulators"), M, N,
               (double)h / (reps * (ts == 2 ? 16.0 : 8.0)), 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
