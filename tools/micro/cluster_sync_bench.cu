// How expensive is cluster.sync() for 8 CTAs x 512 threads on B200?  (seeding kernel design input)
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;
template <int NC>
__global__ void __cluster_dims__(NC, 1, 1) __launch_bounds__(512, 1) k(int iters, long long* out, int mode) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ int s_x[8];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 1 && threadIdx.x < NC) *cl.map_shared_rank(&s_x[cl.block_rank()], threadIdx.x) = i;
    if (mode == 2) __syncthreads(); else cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}
int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int mode = 0; mode < 3; ++mode) {
    k<8><<<40 * 8, 512>>>(2000, d, mode); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster 8, grid 320, mode %d (0=sync,1=dsmem+sync,2=__syncthreads): %lld cycles/iter  (%s)\n", mode, h, cudaGetErrorString(cudaGetLastError()));
    k<4><<<40 * 4, 512>>>(2000, d, mode); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster 4, grid 160, mode %d: %lld cycles/iter\n", mode, h);
    k<2><<<40 * 2, 512>>>(2000, d, mode); cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster 2, grid 80, mode %d: %lld cycles/iter\n", mode, h);
  }
  return 0;
}
