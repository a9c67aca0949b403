// Batched Lloyd k-means + stable cluster-contiguous permutation (subsystem 1).
//
// Reference semantics: /root/reference/pkg/src/routedattn/clustering.py
//   _sq_dists  :55-62   d2 = max(|x|^2 - 2 x.c + |c|^2, 0)
//   _lloyd     :104-141 argmin (ties -> lowest index), bincount, empty-cluster repair,
//                       convergence test BEFORE the centroid update, member-mean update
//   kmeans     :193-198 final centroids = member means, permutation = stable argsort, offsets
//
// Two launches per Lloyd iteration, all `bh` instances batched: the distance contraction
// (kmeans_tc.cu, or assign_fp32_kernel below in fp32 check mode) and lloyd_step_kernel
// (lloyd_step.cu: sizes, repair, convergence, permutation, means, next iteration's bounds).
// Instances that have converged set done[h] and cost nothing afterwards.  No floating-point atomics
// anywhere: counts use integer atomics, means/inertia use fixed-order reductions, so results are
// deterministic run to run.
#include <cooperative_groups.h>

#include "common.cuh"

namespace svg {

// ------------------------------------------------------------------------------------------------
// assignment, fp32 CUDA-core version: one thread per token, token row in registers, centroid tiles
// broadcast from shared memory.  (The tcgen05 version lives in kmeans_tc.cu.)
// ------------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128)
    assign_fp32_kernel(const bf16* __restrict__ x, const float* __restrict__ cent,
                       const float* __restrict__ cnorm, int n, int c, int32_t* __restrict__ assign,
                       float* __restrict__ own_d2, const int32_t* __restrict__ done) {
  const int h = blockIdx.y;
  if (done[h]) return;
  constexpr int TC = 32;
  __shared__ float4 sc[TC][D / 4];
  __shared__ float scn[TC];
  const int tid = threadIdx.x;
  const int t = blockIdx.x * 128 + tid;
  const int tt = min(t, n - 1);

  float xr[D];
  {
    const uint4* xp = reinterpret_cast<const uint4*>(x + ((size_t)h * n + tt) * D);
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      uint4 u = __ldg(xp + i);
      unpack8(u, xr + 8 * i);
    }
  }
  float xn = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) xn = fmaf(xr[k], xr[k], xn);

  float best = INFINITY;
  int bi = 0;
  const float* ch = cent + (size_t)h * c * D;
  for (int c0 = 0; c0 < c; c0 += TC) {
    __syncthreads();
    for (int i = tid; i < TC * (D / 4); i += 128) {
      int r = i / (D / 4), q = i % (D / 4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c0 + r < c) v = __ldg(reinterpret_cast<const float4*>(ch + (size_t)(c0 + r) * D) + q);
      sc[r][q] = v;
    }
    if (tid < TC) scn[tid] = (c0 + tid < c) ? cnorm[(size_t)h * c + c0 + tid] : 0.f;
    __syncthreads();
    const int lim = min(TC, c - c0);
    for (int r = 0; r < lim; r += 4) {
      float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
      for (int q = 0; q < D / 4; ++q) {
        float4 a0 = sc[r][q], a1 = sc[r + 1][q], a2 = sc[r + 2][q], a3 = sc[r + 3][q];
        d0 = fmaf(xr[4 * q], a0.x, d0); d0 = fmaf(xr[4 * q + 1], a0.y, d0);
        d0 = fmaf(xr[4 * q + 2], a0.z, d0); d0 = fmaf(xr[4 * q + 3], a0.w, d0);
        d1 = fmaf(xr[4 * q], a1.x, d1); d1 = fmaf(xr[4 * q + 1], a1.y, d1);
        d1 = fmaf(xr[4 * q + 2], a1.z, d1); d1 = fmaf(xr[4 * q + 3], a1.w, d1);
        d2 = fmaf(xr[4 * q], a2.x, d2); d2 = fmaf(xr[4 * q + 1], a2.y, d2);
        d2 = fmaf(xr[4 * q + 2], a2.z, d2); d2 = fmaf(xr[4 * q + 3], a2.w, d2);
        d3 = fmaf(xr[4 * q], a3.x, d3); d3 = fmaf(xr[4 * q + 1], a3.y, d3);
        d3 = fmaf(xr[4 * q + 2], a3.z, d3); d3 = fmaf(xr[4 * q + 3], a3.w, d3);
      }
      float dd[4] = {d0, d1, d2, d3};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (r + u < lim) {
          // same association as the reference: (|x|^2 - 2 x.c) + |c|^2, clipped at zero
          float v = fmaxf((xn - 2.0f * dd[u]) + scn[r + u], 0.f);
          if (v < best) {  // strict: ties keep the lowest cluster index
            best = v;
            bi = c0 + r + u;
          }
        }
      }
    }
  }
  if (t < n) {
    assign[(size_t)h * n + t] = bi;
    own_d2[(size_t)h * n + t] = best;
  }
}

// ------------------------------------------------------------------------------------------------
// member means in ascending row order, float64 accumulation, one rounding to f32.
// perm == nullptr means `x` is already cluster-contiguous (segment_means).
// ------------------------------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void cluster_mean_one(const bf16* __restrict__ x, const int32_t* __restrict__ perm,
                                                 int n, int c, int h, int j, const int32_t* __restrict__ sizes,
                                                 const int32_t* __restrict__ offsets, float* __restrict__ means,
                                                 float* __restrict__ norms, const uint8_t* __restrict__ dirty,
                                                 float* __restrict__ move) {
  if (dirty && !dirty[(size_t)h * c + j]) {  // same members in the same order: the mean is unchanged
    if (threadIdx.x == 0) move[(size_t)h * c + j] = 0.f;
    return;
  }
  constexpr int EPL = D / 32;
  __shared__ double part[4][D];
  __shared__ float s_c[D];
  __shared__ float s_dc[D];  // new - old per component (for the centre movement)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nj = sizes[(size_t)h * c + j], o = offsets[(size_t)h * c + j];
  double acc[EPL];
#pragma unroll
  for (int u = 0; u < EPL; ++u) acc[u] = 0.0;
  // rows are taken 32 at a time: warp w owns rows 8w..8w+7 of each group and issues its 8 row
  // loads back to back (independent), then accumulates them in ascending order
  for (int base = 0; base < nj; base += 32) {
    int pidx = 0;
    if (base + lane < nj) pidx = perm ? perm[(size_t)h * n + o + base + lane] : (o + base + lane);
    uint2 buf[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = warp * 8 + q;
      const int row = __shfl_sync(0xffffffffu, pidx, r);
      buf[q] = make_uint2(0u, 0u);
      if (base + r < nj) {
        const bf16* p = x + ((size_t)h * n + row) * D + lane * EPL;
        if (EPL == 4) buf[q] = __ldg(reinterpret_cast<const uint2*>(p));
        else buf[q].x = __ldg(reinterpret_cast<const uint32_t*>(p));
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc[0] += (double)__uint_as_float(buf[q].x << 16);
      acc[1] += (double)__uint_as_float(buf[q].x & 0xffff0000u);
      if constexpr (EPL == 4) {
        acc[2] += (double)__uint_as_float(buf[q].y << 16);
        acc[3] += (double)__uint_as_float(buf[q].y & 0xffff0000u);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < EPL; ++u) part[warp][lane * EPL + u] = acc[u];
  __syncthreads();
  if (tid < D) {
    float* out = means + ((size_t)h * c + j) * D;
    float m;
    const float old = out[tid];
    if (nj > 0) {
      double s = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
      m = (float)(s / (double)nj);
      out[tid] = m;
    } else {
      m = old;
    }
    s_c[tid] = m;
    s_dc[tid] = m - old;
  }
  __syncthreads();
  if (warp == 0) {
    float s = 0.f, mv = 0.f;
    for (int k = lane; k < D; k += 32) {
      s = fmaf(s_c[k], s_c[k], s);
      mv = fmaf(s_dc[k], s_dc[k], mv);
    }
    s = warp_sum(s);
    mv = warp_sum(mv);
    if (lane == 0) {
      if (norms) norms[(size_t)h * c + j] = s;
      if (move) move[(size_t)h * c + j] = sqrtf(mv);
    }
  }
}

// grid = (min(c, kMeanBlocks), bh): a block walks clusters blockIdx.x, blockIdx.x + gridDim.x, ...
// (instances that have converged cost one block-exit per block, not one per cluster)
constexpr int kMeanBlocks = 160;
template <int D>
__global__ void __launch_bounds__(128)
    cluster_mean_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ perm, int n, int c,
                        const int32_t* __restrict__ sizes, const int32_t* __restrict__ offsets,
                        float* __restrict__ means, float* __restrict__ norms,
                        const int32_t* __restrict__ done, const uint8_t* __restrict__ dirty,
                        float* __restrict__ move) {
  const int h = blockIdx.y;
  if (done && done[h]) return;
  for (int j = blockIdx.x; j < c; j += gridDim.x) {
    cluster_mean_one<D>(x, perm, n, c, h, j, sizes, offsets, means, norms, dirty, move);
    __syncthreads();  // shared partials are reused by the next cluster
  }
}

// ------------------------------------------------------------------------------------------------
// Inertia of the LAST distance evaluation (clustering.py:126, 189) when tokens were skipped: exact
// fp32 squared distances of every token to its centre, summed in float64 in a fixed order.  Runs
// only for instances that finished in this iteration (converged now, or the iteration cap), before
// the centroid update overwrites the centres the evaluation used.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ bool finishing_now(int h, int iter, int last, const int32_t* done,
                                              const int32_t* iters_run) {
  if (iters_run[h] != iter + 1) return false;  // converged in an earlier iteration
  return done[h] || last;
}

__global__ void __launch_bounds__(256)
    exact_inertia_kernel(const bf16* __restrict__ x_all, const float* __restrict__ cent_all,
                         const int32_t* __restrict__ assign_all, int n, int c, int d, int nchunks, int iter,
                         int last, double* __restrict__ chunk_inertia, const int32_t* __restrict__ done,
                         const int32_t* __restrict__ iters_run) {
  const int h = blockIdx.y;
  if (!finishing_now(h, iter, last, done, iters_run)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bf16* x = x_all + (size_t)h * n * d;
  const float* cent = cent_all + (size_t)h * c * d;
  const int32_t* assign = assign_all + (size_t)h * n;
  const int lo = blockIdx.x * kSortChunk, hi = min(n, lo + kSortChunk);
  __shared__ double s_part[8];
  double dsum = 0.0;
  for (int t = lo + warp; t < hi; t += 8) {
    const float* cr = cent + (size_t)assign[t] * d;
    float acc = 0.f;
    for (int k = lane * 2; k < d; k += 64) {
      const uint32_t xb = __ldg(reinterpret_cast<const uint32_t*>(x + (size_t)t * d + k));
      const float2 cc = *reinterpret_cast<const float2*>(cr + k);
      const float d0 = __uint_as_float(xb << 16) - cc.x, d1 = __uint_as_float(xb & 0xffff0000u) - cc.y;
      acc = fmaf(d0, d0, acc);
      acc = fmaf(d1, d1, acc);
    }
    dsum += (double)warp_sum(acc);
  }
  if (lane == 0) s_part[warp] = dsum;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += s_part[w];
    chunk_inertia[(size_t)h * nchunks + blockIdx.x] = s;
  }
}

// every != 0: every instance that ran this iteration (the stored own distances are current)
__global__ void inertia_sum_kernel(int bh, int nchunks, int iter, int last, int every,
                                   const double* __restrict__ chunk_inertia,
                                   double* __restrict__ inertia, const int32_t* __restrict__ done,
                                   const int32_t* __restrict__ iters_run) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= bh) return;
  if (every ? iters_run[h] != iter + 1 : !finishing_now(h, iter, last, done, iters_run)) return;
  double s = 0.0;
  for (int chn = 0; chn < nchunks; ++chn) s += chunk_inertia[(size_t)h * nchunks + chn];
  inertia[h] = s;
}

// ------------------------------------------------------------------------------------------------
// row gather (permute_rows): 16-byte chunks
// ------------------------------------------------------------------------------------------------
__global__ void gather_rows_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ perm,
                                   int n, int chunks_per_row, uint4* __restrict__ out) {
  const int h = blockIdx.y;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * chunks_per_row) return;
  const int row = (int)(idx / chunks_per_row), ch = (int)(idx % chunks_per_row);
  const int src = perm[(size_t)h * n + row];
  out[((size_t)h * n + row) * chunks_per_row + ch] =
      __ldg(x + ((size_t)h * n + src) * chunks_per_row + ch);
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
int launch_token_norms(int bh, int n, int d, const bf16* x, float* xnorm, cudaStream_t st);
int launch_kmeans_assign_tc(int bh, int n, int d, int c, int iter, const bf16* x, KmeansScratch& sc,
                            int32_t* assign, cudaStream_t st);

bool KmeansScratch::carve(Carver& cv, int bh, int n, int c, int d) {
  const int nchunks = ceil_div(n, kSortChunk);
  prev_assign = cv.take<int32_t>((size_t)bh * n);
  own_d2 = cv.take<float>((size_t)bh * n);
  cnorm = cv.take<float>((size_t)bh * c);
  chunk_inertia = cv.take<double>((size_t)bh * nchunks);
  done = cv.take<int32_t>(bh);
  const int cpad = ceil_div(c, 128) * 128;
  pieces = cv.take<bf16>((size_t)bh * 2 * cpad * d);  // kPieces = 2 (kmeans_tc.cu)
  cnorm_pad = cv.take<float>((size_t)bh * cpad);
  xnorm = cv.take<float>((size_t)bh * n);
  ub = cv.take<float>((size_t)bh * n);
  lb = cv.take<float>((size_t)bh * n);
  active = cv.take<int32_t>((size_t)bh * n);
  nactive = cv.take<int32_t>(bh);
  move = cv.take<float>((size_t)bh * c);
  dirty = cv.take<uint8_t>((size_t)bh * c);
  iters_run = cv.take<int32_t>(bh);
  resid_nz = cv.take<int32_t>(bh);
  dmin = cv.take<float>((size_t)bh * c);
  return cv.ok;
}

// Sum of the own distances the assignment stored (non-skipping modes), per counting-sort chunk in
// a fixed order; feeds inertia_sum_kernel.
__global__ void __launch_bounds__(256)
    own_inertia_kernel(const float* __restrict__ own, int n, int nchunks, int iter, double* __restrict__ chunk_inertia,
                       const int32_t* __restrict__ iters_run) {
  const int h = blockIdx.y;
  if (iters_run[h] != iter + 1) return;  // converged in an earlier iteration
  __shared__ double s_part[8];
  const int tid = threadIdx.x;
  const int lo = blockIdx.x * kSortChunk, hi = min(n, lo + kSortChunk);
  double dsum = 0.0;
  for (int t = lo + tid; t < hi; t += 256) dsum += (double)own[(size_t)h * n + t];
  dsum = warp_sum(dsum);
  if ((tid & 31) == 0) s_part[tid >> 5] = dsum;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += s_part[w];
    chunk_inertia[(size_t)h * nchunks + blockIdx.x] = s;
  }
}

// Lloyd loop: per iteration ONE assignment launch (tcgen05, or the fp32 check kernel) and ONE
// lloyd_step_kernel launch (everything else, see lloyd_step.cu).  Instances that have converged set
// done[h]; once all have, both kernels exit in their prologue.
int launch_kmeans(int exec_mode, int bh, int n, int d, int c, const bf16* x, const float* init,
                  int max_iters, int32_t* assign, int32_t* perm, int32_t* sizes, int32_t* offsets,
                  float* centroids, int32_t* iters, double* inertia, KmeansScratch& sc,
                  cudaStream_t st) {
  const int nchunks = ceil_div(n, kSortChunk);
  SVG_CUDA_OK(cudaMemcpyAsync(centroids, init, (size_t)bh * c * d * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
  const bool full_eval = (exec_mode & SVGEAR_KMEANS_FULL_EVAL) != 0;
  const bool use_tc = (exec_mode & 0xff) == SVGEAR_EXEC_BF16_TENSOR;
  const bool bounded = use_tc && !full_eval;  // skip tokens whose bounds prove they cannot move
  if (use_tc) {
    int rc = launch_token_norms(bh, n, d, x, sc.xnorm, st);
    if (rc) return rc;
  }
  LloydStepArgs a;
  a.x = x; a.n = n; a.c = c; a.cpad = ceil_div(c, 128) * 128;
  a.iter = -1; a.max_iters = max_iters;
  a.use_tc = use_tc; a.bounded = bounded; a.bounded_state = use_tc; a.phases = 3;
  a.wsort = 0; a.scratch_bytes = 0;
  a.assign = assign; a.prev = sc.prev_assign; a.perm = perm; a.sizes = sizes; a.offsets = offsets; a.iters = iters;
  a.cent = centroids; a.cnorm = sc.cnorm; a.own = sc.own_d2; a.ub = sc.ub; a.lb = sc.lb; a.move = sc.move;
  a.dmin = sc.dmin; a.cnorm_pad = sc.cnorm_pad; a.xnorm = sc.xnorm; a.dirty = sc.dirty; a.pieces = sc.pieces;
  a.active = sc.active; a.nactive = sc.nactive; a.resid_nz = sc.resid_nz; a.done = sc.done; a.iters_run = sc.iters_run;
  int rc = launch_lloyd_step(a, bh, d, st);
  if (rc) return rc;
  for (int it = 0; it < max_iters; ++it) {
    if (use_tc) {
      rc = launch_kmeans_assign_tc(bh, n, d, c, it, x, sc, assign, st);
      if (rc) return rc;
    } else {
      dim3 ga(ceil_div(n, 128), bh);
      if (d == 128)
        assign_fp32_kernel<128><<<ga, 128, 0, st>>>(x, centroids, sc.cnorm, n, c, assign, sc.own_d2, sc.done);
      else
        assign_fp32_kernel<64><<<ga, 128, 0, st>>>(x, centroids, sc.cnorm, n, c, assign, sc.own_d2, sc.done);
      SVG_LAUNCH_OK();
    }
    a.iter = it;
    if (!inertia) {
      a.phases = 3;
      rc = launch_lloyd_step(a, bh, d, st);
      if (rc) return rc;
      continue;
    }
    // inertia of the LAST distance evaluation (clustering.py:126, 189), wanted by the staged API only:
    // it needs the centres the evaluation used, so it sits between the two halves of the step
    a.phases = 1;
    rc = launch_lloyd_step(a, bh, d, st);
    if (rc) return rc;
    const int last = it == max_iters - 1;
    if (bounded) {  // own distances of skipped tokens are stale: recompute the sum exactly
      exact_inertia_kernel<<<dim3(nchunks, bh), 256, 0, st>>>(x, centroids, assign, n, c, d, nchunks, it, last,
                                                             sc.chunk_inertia, sc.done, sc.iters_run);
      SVG_LAUNCH_OK();
      inertia_sum_kernel<<<ceil_div(bh, 128), 128, 0, st>>>(bh, nchunks, it, last, 0, sc.chunk_inertia, inertia, sc.done, sc.iters_run);
    } else {
      own_inertia_kernel<<<dim3(nchunks, bh), 256, 0, st>>>(sc.own_d2, n, nchunks, it, sc.chunk_inertia, sc.iters_run);
      SVG_LAUNCH_OK();
      inertia_sum_kernel<<<ceil_div(bh, 128), 128, 0, st>>>(bh, nchunks, it, last, 1, sc.chunk_inertia, inertia, sc.done, sc.iters_run);
    }
    SVG_LAUNCH_OK();
    a.phases = 2;
    rc = launch_lloyd_step(a, bh, d, st);
    if (rc) return rc;
  }
  return SVGEAR_OK;
}

int launch_gather_rows(int bh, int n, int d, const bf16* x, const int32_t* perm, bf16* out,
                       cudaStream_t st) {
  const int cpr = d / 8;
  const long long total = (long long)n * cpr;
  gather_rows_kernel<<<dim3((unsigned)((total + 255) / 256), bh), 256, 0, st>>>(
      reinterpret_cast<const uint4*>(x), perm, n, cpr, reinterpret_cast<uint4*>(out));
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

int launch_segment_means(int bh, int n, int d, int c, const bf16* xp, const int32_t* sizes,
                         const int32_t* offsets, float* means, float* norms, cudaStream_t st) {
  if (d == 128)
    cluster_mean_kernel<128><<<dim3(min(c, kMeanBlocks), bh), 128, 0, st>>>(xp, nullptr, n, c, sizes, offsets, means,
                                                         norms, nullptr, nullptr, nullptr);
  else
    cluster_mean_kernel<64><<<dim3(min(c, kMeanBlocks), bh), 128, 0, st>>>(xp, nullptr, n, c, sizes, offsets, means,
                                                        norms, nullptr, nullptr, nullptr);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
