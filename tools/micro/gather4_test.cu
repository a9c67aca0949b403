// Microtest: TMA tile::gather4 into SWIZZLE_128B shared memory; which boxDim[1] does it want?
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap tm, const int* rows, uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(base + 8192);
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(base), sbar = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x < 16) {   // 16 lanes x 4 rows = 64 rows x 128 B = 8 KB
    int g = threadIdx.x;
    if (g == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(8192));
    __syncwarp(0xffff);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(sb + g * 512), "l"(&tm), "r"(64), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]),
        "r"(rows[4 * g + 3]), "r"(sbar) : "memory");
  }
  // wait
  asm volatile("{ .reg .pred p; L: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @p bra D; bra L; D: }" ::"r"(sbar) : "memory");
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = ((uint16_t*)base)[i];
}

int main() {
  const int R = 1000, C = 128;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 7 + c);  // pattern
  uint16_t* d; cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  std::vector<int> rows(64); for (int i = 0; i < 64; ++i) rows[i] = (i * 37 + 11) % R;
  int* drows; cudaMalloc(&drows, 256); cudaMemcpy(drows, rows.data(), 256, cudaMemcpyHostToDevice);
  uint16_t* dout; cudaMalloc(&dout, 8192);
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  printf("entry %p qr %d\n", fn, (int)qr);
  for (int boxrows : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {C, R}; cuuint64_t strides[1] = {C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxrows}; cuuint32_t es[2] = {1, 1};
    CUresult rc = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("boxrows %d encode rc %d\n", boxrows, (int)rc);
    cudaMemset(dout, 0xff, 8192);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    k<<<1, 128, 16384>>>(tm, drows, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  launch: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) { cudaGetLastError(); continue; }
    std::vector<uint16_t> o(4096); cudaMemcpy(o.data(), dout, 8192, cudaMemcpyDeviceToHost);
    // expected: row slot s (0..63), chunk c (0..7) at byte s*128 + ((c ^ (s&7))<<4); columns 64..127
    int bad = 0;
    for (int s = 0; s < 64; ++s) for (int c = 0; c < 8; ++c) for (int e2 = 0; e2 < 8; ++e2) {
      uint16_t want = (uint16_t)(rows[s] * 7 + 64 + c * 8 + e2);
      uint16_t got = o[(s * 128 + ((c ^ (s & 7)) << 4)) / 2 + e2];
      if (want != got) { if (bad < 4) printf("  mismatch s=%d c=%d e=%d want %u got %u\n", s, c, e2, want, got); ++bad; }
    }
    printf("  boxrows %d: %d mismatches of 4096\n", boxrows, bad);
  }
  return 0;
}
