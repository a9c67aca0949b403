// Microbenchmark: issue rate (clk per warp instruction, per SM sub-partition) of the instructions the
// attention softmax uses: MUFU.EX2, F2FP pack (cvt.rn.bf16x2.f32), FFMA, FFMA2, FADD2, FMNMX3, LEA.
// One block of 4*W warps (W warps per sub-partition); independent chains so latency does not matter.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define REP 256
template <int OP>
__global__ void k(float* out, long long* clk, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * 0.01f + threadIdx.x * 1e-4f;
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) u[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < REP; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(1.0001f), "f"(0.5f));
      if (OP == 3) {
        unsigned long long p, q = 0x3f8000003f800000ull, c = 0x3f0000003f000000ull;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p) : "l"(q), "l"(c));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a[i]), "=f"(a[(i + 1) & 7]) : "l"(p));
      }
      if (OP == 4) asm volatile("max.f32 %0, %0, %1;\n\tmax.f32 %0, %0, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      if (OP == 5) asm volatile("shl.b32 %0, %0, 23;\n\tadd.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
      if (OP == 6) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(0.5f));
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps_per_smsp) {
  float* out; long long* clk;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&clk, 1024);
  int threads = 128 * warps_per_smsp;
  k<OP><<<1, threads>>>(out, clk, 0.3f);
  k<OP><<<1, threads>>>(out, clk, 0.3f);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (REP * 8.0 * warps_per_smsp);
  printf("%-28s warps/SMSP=%d  %.2f clk per warp-instruction (per sub-partition)\n", name, warps_per_smsp, per);
  cudaFree(out); cudaFree(clk);
}

int main() {
  for (int w : {1, 2, 4}) {
    run<0>("MUFU.EX2", w);
    run<1>("F2FP.BF16.PACK_AB", w);
    run<2>("FFMA", w);
    run<3>("FFMA2 (+pack/unpack movs)", w);
    run<4>("FMNMX x2 (or FMNMX3)", w);
    run<5>("SHL+IADD (LEA)", w);
    run<6>("FADD", w);
  }
  return 0;
}
