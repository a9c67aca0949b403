// Batched Lloyd k-means + stable cluster-contiguous permutation (subsystem 1).
//
// Reference semantics: /root/reference/pkg/src/routedattn/clustering.py
//   _sq_dists  :55-62   d2 = max(|x|^2 - 2 x.c + |c|^2, 0)
//   _lloyd     :104-141 argmin (ties -> lowest index), bincount, empty-cluster repair,
//                       convergence test BEFORE the centroid update, member-mean update
//   kmeans     :193-198 final centroids = member means, permutation = stable argsort, offsets
//
// One launch sequence per Lloyd iteration, all `bh` instances batched in grid.y; instances that
// have converged set done[h] and every later kernel returns immediately for them.  No
// floating-point atomics anywhere: counts use integer atomics, means/inertia use fixed-order
// reductions, so results are deterministic run to run.
#include <cooperative_groups.h>

#include "common.cuh"

namespace svg {

// ------------------------------------------------------------------------------------------------
// centroid squared norms
// ------------------------------------------------------------------------------------------------
__global__ void centroid_norm_kernel(const float* __restrict__ cent, int d, int total,
                                     float* __restrict__ cnorm) {
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= total) return;
  const float* p = cent + (size_t)row * d;
  float s = 0.f;
  for (int k = lane; k < d; k += 32) s = fmaf(p[k], p[k], s);
  s = warp_sum(s);
  if (lane == 0) cnorm[row] = s;
}

// ------------------------------------------------------------------------------------------------
// assignment, fp32 CUDA-core version: one thread per token, token row in registers, centroid tiles
// broadcast from shared memory.  (The tcgen05 version lives in kmeans_tc.cu.)
// ------------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128)
    assign_fp32_kernel(const bf16* __restrict__ x, const float* __restrict__ cent,
                       const float* __restrict__ cnorm, int n, int c, int32_t* __restrict__ assign,
                       float* __restrict__ own_d2, int32_t* __restrict__ sizes,
                       int32_t* __restrict__ changed, const int32_t* __restrict__ done) {
  const int h = blockIdx.y;
  if (done[h]) return;
  constexpr int TC = 32;
  __shared__ float4 sc[TC][D / 4];
  __shared__ float scn[TC];
  const int tid = threadIdx.x;
  const int t = blockIdx.x * 128 + tid;
  const int tt = min(t, n - 1);

  if (blockIdx.x == 0) {  // reset the per-iteration counters of this instance
    for (int j = tid; j < c; j += 128) sizes[(size_t)h * c + j] = 0;
    if (tid == 0) changed[h] = 0;
  }

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
// cluster sizes (integer atomics -> deterministic)
// ------------------------------------------------------------------------------------------------
// The last block of an instance to finish (ticket counter) also records whether any cluster is
// empty, so that the repair helpers can return after reading one flag.
__global__ void sizes_hist_kernel(const int32_t* __restrict__ assign, int n, int c,
                                  int32_t* __restrict__ sizes, int32_t* __restrict__ ticket,
                                  int32_t* __restrict__ has_empty, const int32_t* __restrict__ done) {
  const int h = blockIdx.y;
  if (done[h]) return;
  extern __shared__ int32_t hist[];
  for (int j = threadIdx.x; j < c; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  const int per_block = ceil_div(n, gridDim.x);
  const int lo = blockIdx.x * per_block, hi = min(n, lo + per_block);
  for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) atomicAdd(&hist[assign[(size_t)h * n + t]], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x)
    if (hist[j]) atomicAdd(&sizes[(size_t)h * c + j], hist[j]);
  __threadfence();
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ticket[h], 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  int empty = 0;
  for (int j = threadIdx.x; j < c; j += blockDim.x) empty |= (__ldcg(&sizes[(size_t)h * c + j]) == 0);
  empty = __syncthreads_or(empty);
  if (threadIdx.x == 0) {
    has_empty[h] = empty;
    ticket[h] = 0;
  }
}

// ------------------------------------------------------------------------------------------------
// empty-cluster repair (clustering.py:116-124): for each empty cluster in ascending order move the
// token with the largest own distance (first maximum) among clusters of size >= 2.
// ------------------------------------------------------------------------------------------------
// The own distances the tensor-core assignment stores are |x|^2 - 2x.c + |c|^2 in fp32 (cancellation
// noise ~1e-5 |x|^2) and, with bound-based skipping, stale for skipped tokens.  The repair rule
// ranks tokens by own distance (clustering.py:118), so an instance that actually has an empty
// cluster (rare) first gets all of them recomputed exactly — fp32 sum of squared differences against
// the current centres — by this grid-wide kernel; other instances return after scanning their sizes.
__global__ void __launch_bounds__(256)
    own_refresh_kernel(int n, int c, int d, const bf16* __restrict__ x_all, const float* __restrict__ cent_all,
                       const int32_t* __restrict__ assign_all, const int32_t* __restrict__ has_empty,
                       float* __restrict__ own_all, const int32_t* __restrict__ done) {
  const int h = blockIdx.y;
  if (done[h] || !has_empty[h]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bf16* x = x_all + (size_t)h * n * d;
  const float* cent = cent_all + (size_t)h * c * d;
  const int32_t* assign = assign_all + (size_t)h * n;
  float* own = own_all + (size_t)h * n;
  constexpr int kSpan = 1024;  // tokens per block step
  for (int lo = blockIdx.x * kSpan; lo < n; lo += gridDim.x * kSpan) {
  const int hi = min(n, lo + kSpan);
  for (int t0 = lo + warp * 4; t0 < hi; t0 += 32) {  // 4 independent rows per warp step
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = min(t0 + u, hi - 1);
      const float* cr = cent + (size_t)assign[t] * d;
      for (int k = lane * 2; k < d; k += 64) {
        const uint32_t xb = __ldg(reinterpret_cast<const uint32_t*>(x + (size_t)t * d + k));
        const float2 cc = *reinterpret_cast<const float2*>(cr + k);
        const float d0 = __uint_as_float(xb << 16) - cc.x, d1 = __uint_as_float(xb & 0xffff0000u) - cc.y;
        acc[u] = fmaf(d0, d0, acc[u]);
        acc[u] = fmaf(d1, d1, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float v = warp_sum(acc[u]);
      if (lane == 0 && t0 + u < hi) own[t0 + u] = v;
    }
  }
  }
}

__global__ void __launch_bounds__(1024)
    repair_kernel(int n, int c, int32_t* __restrict__ assign_all,
                  float* __restrict__ own_all, int32_t* __restrict__ sizes_all, float* __restrict__ ub_all,
                  float* __restrict__ lb_all, uint8_t* __restrict__ dirty_all,
                  const int32_t* __restrict__ done) {
  const int h = blockIdx.x;
  if (done[h]) return;
  int32_t* assign = assign_all + (size_t)h * n;
  float* own = own_all + (size_t)h * n;
  int32_t* sizes = sizes_all + (size_t)h * c;
  constexpr int kMaxList = 1024;
  __shared__ float s_val[32];
  __shared__ int s_idx[32];
  __shared__ int s_wcount[32];
  __shared__ int s_empty[kMaxList];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  while (true) {
    // ascending list of the (first kMaxList) empty clusters; a repaired cluster never becomes
    // empty again because donors only come from clusters with >= 2 members
    int carry = 0;
    for (int base = 0; base < c; base += 1024) {
      const int j = base + tid;
      const bool flag = j < c && sizes[j] == 0;
      const unsigned bal = __ballot_sync(0xffffffffu, flag);
      __syncthreads();
      if (lane == 0) s_wcount[warp] = __popc(bal);
      __syncthreads();
      int woff = 0, tot = 0;
      for (int w = 0; w < 32; ++w) {
        const int cw = s_wcount[w];
        if (w < warp) woff += cw;
        tot += cw;
      }
      const int pos = carry + woff + __popc(bal & ((1u << lane) - 1u));
      if (flag && pos < kMaxList) s_empty[pos] = j;
      carry += tot;
    }
    __syncthreads();
    const int ne = min(carry, kMaxList);
    if (ne == 0) return;
    for (int ei = 0; ei < ne; ++ei) {
      const int e = s_empty[ei];
      __syncthreads();
      float bv = -1.f;
      int bx = 0x7fffffff;
      for (int t = tid; t < n; t += blockDim.x) {
        if (sizes[assign[t]] >= 2) {
          float v = own[t];
          if (v > bv) { bv = v; bx = t; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int ox = __shfl_xor_sync(0xffffffffu, bx, o);
        if (ov > bv || (ov == bv && ox < bx)) { bv = ov; bx = ox; }
      }
      if (lane == 0) { s_val[warp] = bv; s_idx[warp] = bx; }
      __syncthreads();
      if (warp == 0) {
        bv = s_val[lane];
        bx = s_idx[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          int ox = __shfl_xor_sync(0xffffffffu, bx, o);
          if (ov > bv || (ov == bv && ox < bx)) { bv = ov; bx = ox; }
        }
        if (lane == 0 && bx != 0x7fffffff) {
          const int from = assign[bx];
          sizes[from] -= 1;
          sizes[e] += 1;
          assign[bx] = e;
          own[bx] = 0.f;
          if (dirty_all) {  // both memberships changed; the moved token is re-evaluated next time
            dirty_all[(size_t)h * c + from] = 1;
            dirty_all[(size_t)h * c + e] = 1;
            ub_all[(size_t)h * n + bx] = 0.f;
            lb_all[(size_t)h * n + bx] = 0.f;
          }
        }
      }
    }
    __syncthreads();
    if (carry <= kMaxList) return;
  }
}

// ------------------------------------------------------------------------------------------------
// per-chunk histogram + convergence compare + inertia partials
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    chunk_hist_kernel(const int32_t* __restrict__ assign, int32_t* __restrict__ prev,
                      const float* __restrict__ own, int n, int c, int nchunks, int iter,
                      int32_t* __restrict__ chunk_counts, double* __restrict__ chunk_inertia,
                      int32_t* __restrict__ changed, const int32_t* __restrict__ done) {
  const int h = blockIdx.y;
  if (done[h]) return;
  extern __shared__ int32_t hist[];
  __shared__ double s_part[8];
  const int tid = threadIdx.x;
  for (int j = tid; j < c; j += 256) hist[j] = 0;
  __syncthreads();
  const int lo = blockIdx.x * kSortChunk, hi = min(n, lo + kSortChunk);
  int diff = 0;
  double dsum = 0.0;
  for (int t = lo + tid; t < hi; t += 256) {
    size_t g = (size_t)h * n + t;
    int a = assign[g];
    atomicAdd(&hist[a], 1);
    if (iter > 0) diff |= (prev[g] != a);
    prev[g] = a;
    dsum += (double)own[g];
  }
  diff = __syncthreads_or(diff);
  if (tid == 0 && diff) atomicOr(&changed[h], 1);
  int32_t* out = chunk_counts + ((size_t)h * nchunks + blockIdx.x) * c;
  for (int j = tid; j < c; j += 256) out[j] = hist[j];
  dsum = warp_sum(dsum);
  if ((tid & 31) == 0) s_part[tid >> 5] = dsum;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += s_part[w];
    chunk_inertia[(size_t)h * nchunks + blockIdx.x] = s;
  }
}

// ------------------------------------------------------------------------------------------------
// offsets (exclusive scan of sizes), per-chunk scatter bases, inertia, convergence decision
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
    scan_kernel(int n, int c, int nchunks, int iter, const int32_t* __restrict__ sizes_all,
                int32_t* __restrict__ offsets_all, int32_t* __restrict__ chunk_counts,
                const double* __restrict__ chunk_inertia, double* __restrict__ inertia,
                int32_t* __restrict__ iters, int32_t* __restrict__ iters_run,
                int32_t* __restrict__ nactive, int32_t* __restrict__ resid_nz,
                const int32_t* __restrict__ changed, int32_t* __restrict__ done) {
  const int h = blockIdx.x;
  if (done[h]) return;
  const int32_t* sizes = sizes_all + (size_t)h * c;
  int32_t* offsets = offsets_all + (size_t)h * c;
  __shared__ int s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int PER = kMaxClusters / 1024;  // 4 consecutive clusters per thread
  int v[PER], tot = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    int j = tid * PER + u;
    v[u] = j < c ? sizes[j] : 0;
    tot += v[u];
  }
  int inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_warp[lane] = wi - w;  // exclusive warp base
  }
  __syncthreads();
  int run = s_warp[warp] + inc - tot;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    int j = tid * PER + u;
    if (j < c) {
      offsets[j] = run;
      int base = run;
      int32_t* col = chunk_counts + (size_t)h * nchunks * c + j;
      for (int ch0 = 0; ch0 < nchunks; ch0 += 8) {
        int cnt[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cnt[q] = ch0 + q < nchunks ? col[(size_t)(ch0 + q) * c] : 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (ch0 + q < nchunks) col[(size_t)(ch0 + q) * c] = base;
          base += cnt[q];
        }
      }
    }
    run += v[u];
  }
  if (tid == 0) {
    double s = 0.0;
    for (int chn = 0; chn < nchunks; ++chn) s += chunk_inertia[(size_t)h * nchunks + chn];
    if (inertia) inertia[h] = s;
    if (iters) iters[h] = iter + 1;
    iters_run[h] = iter + 1;
    nactive[h] = 0;  // the next iteration's filter appends to an empty list
    resid_nz[h] = 0;
    if (iter > 0 && !changed[h]) done[h] = 1;  // assignments unchanged -> converged
  }
}

// ------------------------------------------------------------------------------------------------
// stable scatter: perm[base[cluster] + rank among earlier same-cluster tokens] = token
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    scatter_perm_kernel(const int32_t* __restrict__ assign, int n, int c, int nchunks,
                        const int32_t* __restrict__ chunk_base, int32_t* __restrict__ perm,
                        const int32_t* __restrict__ done) {
  const int h = blockIdx.y;
  if (done[h]) return;
  extern __shared__ int32_t cnt[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int32_t* base_in = chunk_base + ((size_t)h * nchunks + blockIdx.x) * c;
  for (int j = tid; j < c; j += 256) cnt[j] = base_in[j];
  __syncthreads();
  for (int r = 0; r < kSortChunk / 256; ++r) {
    const int t = blockIdx.x * kSortChunk + r * 256 + tid;
    const bool valid = t < n;
    const int a = valid ? assign[(size_t)h * n + t] : (0x7fffff00 | lane);
    const unsigned m = __match_any_sync(0xffffffffu, a);
    const int leader = __ffs(m) - 1;
    const int rank = __popc(m & ((1u << lane) - 1u));
    int base = 0;
    for (int w = 0; w < 8; ++w) {
      if (warp == w && valid && lane == leader) {
        base = cnt[a];
        cnt[a] = base + __popc(m);
      }
      __syncthreads();
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) perm[(size_t)h * n + base + rank] = t;
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

__global__ void inertia_sum_kernel(int bh, int nchunks, int iter, int last, const double* __restrict__ chunk_inertia,
                                   double* __restrict__ inertia, const int32_t* __restrict__ done,
                                   const int32_t* __restrict__ iters_run) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= bh) return;
  if (!finishing_now(h, iter, last, done, iters_run)) return;
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
int launch_kmeans_assign_tc(int bh, int n, int d, int c, int iter, bool full_eval, const bf16* x,
                            const float* cent, const float* cnorm, KmeansScratch& sc, int32_t* assign,
                            int32_t* sizes, cudaStream_t st);

bool KmeansScratch::carve(Carver& cv, int bh, int n, int c, int d) {
  const int nchunks = ceil_div(n, kSortChunk);
  prev_assign = cv.take<int32_t>((size_t)bh * n);
  own_d2 = cv.take<float>((size_t)bh * n);
  cnorm = cv.take<float>((size_t)bh * c);
  chunk_counts = cv.take<int32_t>((size_t)bh * nchunks * c);
  chunk_inertia = cv.take<double>((size_t)bh * nchunks);
  done = cv.take<int32_t>(bh);
  changed = cv.take<int32_t>(bh);
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
  ticket = cv.take<int32_t>(bh);
  has_empty = cv.take<int32_t>(bh);
  resid_nz = cv.take<int32_t>(bh);
  dmin = cv.take<float>((size_t)bh * c);
  movers = cv.take<float2>(bh);
  return cv.ok;
}

int launch_kmeans(int exec_mode, int bh, int n, int d, int c, const bf16* x, const float* init,
                  int max_iters, int32_t* assign, int32_t* perm, int32_t* sizes, int32_t* offsets,
                  float* centroids, int32_t* iters, double* inertia, KmeansScratch& sc,
                  cudaStream_t st) {
  const int nchunks = ceil_div(n, kSortChunk);
  SVG_CUDA_OK(cudaMemcpyAsync(centroids, init, (size_t)bh * c * d * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
  SVG_CUDA_OK(cudaMemsetAsync(sc.done, 0, (size_t)bh * 4, st));
  SVG_CUDA_OK(cudaMemsetAsync(sc.changed, 0, (size_t)bh * 4, st));
  SVG_CUDA_OK(cudaMemsetAsync(sc.ticket, 0, (size_t)bh * 4, st));
  SVG_CUDA_OK(cudaMemsetAsync(sc.resid_nz, 0, (size_t)bh * 4, st));
  centroid_norm_kernel<<<ceil_div(bh * c, 8), 256, 0, st>>>(centroids, d, bh * c, sc.cnorm);
  SVG_LAUNCH_OK();
  const bool full_eval = (exec_mode & SVGEAR_KMEANS_FULL_EVAL) != 0;
  const bool use_tc = (exec_mode & 0xff) == SVGEAR_EXEC_BF16_TENSOR;
  const bool bounded = use_tc && !full_eval;  // skip tokens whose bounds prove they cannot move
  if (use_tc) {
    int rc = launch_token_norms(bh, n, d, x, sc.xnorm, st);
    if (rc) return rc;
    SVG_CUDA_OK(cudaMemsetAsync(sc.nactive, 0, (size_t)bh * 4, st));
    SVG_CUDA_OK(cudaMemsetAsync(sc.move, 0, (size_t)bh * c * 4, st));
  }
  const size_t hist_smem = (size_t)c * sizeof(int32_t);
  const int hist_blocks = max(1, min(64, ceil_div(n, 4096)));
  for (int it = 0; it < max_iters; ++it) {
    dim3 ga(ceil_div(n, 128), bh);
    if (use_tc) {
      int rc = launch_kmeans_assign_tc(bh, n, d, c, it, full_eval, x, centroids, sc.cnorm, sc, assign, sizes, st);
      if (rc) return rc;
    } else if (d == 128)
      assign_fp32_kernel<128><<<ga, 128, 0, st>>>(x, centroids, sc.cnorm, n, c, assign, sc.own_d2,
                                                  sizes, sc.changed, sc.done);
    else
      assign_fp32_kernel<64><<<ga, 128, 0, st>>>(x, centroids, sc.cnorm, n, c, assign, sc.own_d2,
                                                 sizes, sc.changed, sc.done);
    SVG_LAUNCH_OK();
    sizes_hist_kernel<<<dim3(hist_blocks, bh), 256, hist_smem, st>>>(assign, n, c, sizes, sc.ticket,
                                                                     sc.has_empty, sc.done);
    SVG_LAUNCH_OK();
    if (use_tc) {  // exact own distances for the donor choice (the tensor-core ones are rounded / stale)
      own_refresh_kernel<<<dim3(min(ceil_div(n, 1024), 64), bh), 256, 0, st>>>(n, c, d, x, centroids, assign, sc.has_empty,
                                                           sc.own_d2, sc.done);
      SVG_LAUNCH_OK();
    }
    repair_kernel<<<bh, 1024, 0, st>>>(n, c, assign, sc.own_d2, sizes, sc.ub, sc.lb,
                                       use_tc ? sc.dirty : nullptr, sc.done);
    SVG_LAUNCH_OK();
    chunk_hist_kernel<<<dim3(nchunks, bh), 256, hist_smem, st>>>(
        assign, sc.prev_assign, sc.own_d2, n, c, nchunks, it, sc.chunk_counts, sc.chunk_inertia,
        sc.changed, sc.done);
    SVG_LAUNCH_OK();
    scan_kernel<<<bh, 1024, 0, st>>>(n, c, nchunks, it, sizes, offsets, sc.chunk_counts,
                                     sc.chunk_inertia, inertia, iters, sc.iters_run, sc.nactive,
                                     sc.resid_nz, sc.changed, sc.done);
    SVG_LAUNCH_OK();
    if (bounded && inertia) {  // own distances of skipped tokens are stale: recompute the sum exactly
      const int last = it == max_iters - 1;
      exact_inertia_kernel<<<dim3(nchunks, bh), 256, 0, st>>>(x, centroids, assign, n, c, d, nchunks, it, last,
                                                             sc.chunk_inertia, sc.done, sc.iters_run);
      SVG_LAUNCH_OK();
      inertia_sum_kernel<<<ceil_div(bh, 128), 128, 0, st>>>(bh, nchunks, it, last, sc.chunk_inertia, inertia, sc.done, sc.iters_run);
      SVG_LAUNCH_OK();
    }
    scatter_perm_kernel<<<dim3(nchunks, bh), 256, hist_smem, st>>>(assign, n, c, nchunks,
                                                                   sc.chunk_counts, perm, sc.done);
    SVG_LAUNCH_OK();
    const uint8_t* dirty = bounded ? sc.dirty : nullptr;
    if (d == 128)
      cluster_mean_kernel<128><<<dim3(min(c, kMeanBlocks), bh), 128, 0, st>>>(x, perm, n, c, sizes, offsets, centroids,
                                                           sc.cnorm, sc.done, dirty, sc.move);
    else
      cluster_mean_kernel<64><<<dim3(min(c, kMeanBlocks), bh), 128, 0, st>>>(x, perm, n, c, sizes, offsets, centroids,
                                                          sc.cnorm, sc.done, dirty, sc.move);
    SVG_LAUNCH_OK();
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

// ------------------------------------------------------------------------------------------------
// Device-side seeding: k-means++ (D^2 sampling, clustering.py:65-84) run on a strided SUBSAMPLE of
// m = min(n, oversample*c) tokens with a counter-based hash RNG.  It is NOT the reference's draw
// (that needs numpy's generator over all n tokens, host side); it is the start used when the
// caller supplies no centres and asks for a device-side start.  One CTA per instance; the
// running min-distance array lives in shared memory; deterministic.
// ------------------------------------------------------------------------------------------------
namespace svg {

__device__ __forceinline__ uint32_t hash_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t x = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du;
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}

// A thread-block CLUSTER of 8 CTAs serves one instance: every thread keeps ONE subsample token in
// registers for the whole run; per step each CTA reloads the newest centre (256 B), updates its
// min-distances, block-scans them, and the 8 partial sums are exchanged through distributed shared
// memory (2 cluster barriers per step).
constexpr int kSeedCtas = 8;
constexpr int kSeedBatch = 4;      // centres drawn per round
constexpr int kSeedThreads = 512;  // one subsample token per thread, held in registers

template <int D>
__global__ void __cluster_dims__(kSeedCtas, 1, 1) __launch_bounds__(kSeedThreads, 3)
    seed_pp_kernel(const bf16* __restrict__ x, int n, int c, int m, uint32_t seed, float* __restrict__ cent) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int h = blockIdx.x / kSeedCtas;
  __shared__ __align__(16) __nv_bfloat162 s_c2[kSeedBatch][D / 2];  // newest centres (bf16 tokens)
  __shared__ float s_warp[32];
  __shared__ float s_part[kSeedCtas];     // partial sums of all CTAs (written through DSMEM)
  __shared__ int s_pick[kSeedBatch];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bf16* xh = x + (size_t)h * n * D;
  float* ch = cent + (size_t)h * c * D;
  auto sample_row = [&](int s) -> size_t { return (size_t)(((long long)s * n) / m); };
  const int per = (m + kSeedCtas - 1) / kSeedCtas;  // samples per CTA, <= kSeedThreads
  const int s_mine = rank * per + tid;
  const bool have = tid < per && s_mine < m;
  // the token of this thread is re-read from L2 every round (all centres of a round share the
  // read); keeping it in registers would cost 64 registers and limit residency to one CTA per SM
  const uint4* my_row = reinterpret_cast<const uint4*>(xh + sample_row(have ? s_mine : 0) * D);
  float mind = have ? INFINITY : 0.f;
  // Centres are drawn in rounds of up to kSeedBatch (one while fewer than 128 remain): the draws of
  // a round share one D^2 distribution, which amortises the two cluster barriers per round.
  int picks[kSeedBatch];
  picks[0] = (int)(hash_u32(seed, (uint32_t)h, 0u) % (uint32_t)m);
  int cnt = 1, npicked = 0;
  while (true) {
    if (tid < cnt * D) {
      const int i = tid / D, k = tid % D;
      const bf16 b = xh[sample_row(picks[i]) * D + k];
      reinterpret_cast<bf16*>(&s_c2[i][0])[k] = b;
      if (rank == 0) ch[(size_t)(npicked + i) * D + k] = __bfloat162float(b);
    }
    __syncthreads();
    npicked += cnt;
    if (npicked >= c) break;
    if (have) {
      // squared distances to the round's centres.  Tokens and centres are bf16, so the differences
      // and 16-element partial sums are formed with packed bf16x2 math (HSUB2/HFMA2.BF16: one
      // instruction per two elements) and flushed to fp32 every 16 elements; the ~1 % noise only
      // perturbs sampling weights.
      float d2[kSeedBatch];
      __nv_bfloat162 a2[kSeedBatch];
#pragma unroll
      for (int i = 0; i < kSeedBatch; ++i) { d2[i] = 0.f; a2[i] = __floats2bfloat162_rn(0.f, 0.f); }
#pragma unroll 2
      for (int q = 0; q < D / 8; ++q) {
        const uint4 u = __ldg(my_row + q);
        const __nv_bfloat162 x0 = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
        const __nv_bfloat162 x1 = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
        const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&u.z);
        const __nv_bfloat162 x3 = *reinterpret_cast<const __nv_bfloat162*>(&u.w);
#pragma unroll
        for (int i = 0; i < kSeedBatch; ++i) {
          if (i < cnt) {
            const uint4 cu = *reinterpret_cast<const uint4*>(&s_c2[i][4 * q]);
            __nv_bfloat162 df = __hsub2(x0, *reinterpret_cast<const __nv_bfloat162*>(&cu.x));
            a2[i] = __hfma2(df, df, a2[i]);
            df = __hsub2(x1, *reinterpret_cast<const __nv_bfloat162*>(&cu.y));
            a2[i] = __hfma2(df, df, a2[i]);
            df = __hsub2(x2, *reinterpret_cast<const __nv_bfloat162*>(&cu.z));
            a2[i] = __hfma2(df, df, a2[i]);
            df = __hsub2(x3, *reinterpret_cast<const __nv_bfloat162*>(&cu.w));
            a2[i] = __hfma2(df, df, a2[i]);
            if (q & 1) {
              const float2 f = __bfloat1622float2(a2[i]);
              d2[i] += f.x + f.y;
              a2[i] = __floats2bfloat162_rn(0.f, 0.f);
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kSeedBatch; ++i)
        if (i < cnt) mind = fminf(mind, d2[i]);
    }
    // block scan of the per-thread values (fixed order, fp32: this only steers the sampling)
    float inc = mind;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      float w = lane < kSeedThreads / 32 ? s_warp[lane] : 0.f, wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
      const float tot = __shfl_sync(0xffffffffu, wi, 31);
      if (lane < kSeedCtas) *cluster.map_shared_rank(&s_part[rank], lane) = tot;  // publish to CTA `lane`
      if (lane < kSeedBatch) s_pick[lane] = -1;
    }
    cluster.sync();
    float total = 0.f, before = 0.f;
#pragma unroll
    for (int r = 0; r < kSeedCtas; ++r) {
      if (r == rank) before = total;
      total += s_part[r];
    }
    const int left = c - npicked;
    const int next = left >= 128 ? kSeedBatch : 1;
    if (total > 0.f && have && mind > 0.f) {
      const float lo = before + s_warp[warp] + inc - mind;
      for (int i = 0; i < next; ++i) {
        const float u = ((float)(hash_u32(seed, (uint32_t)h, (uint32_t)(npicked + i) + 1u) >> 8) + 0.5f) *
                        (1.0f / 16777216.0f);
        const float target = u * total;
        // intervals are built from the same partial sums on every CTA; a target on a rounding
        // boundary can be claimed by two adjacent threads: keep the larger index
        if (target >= lo && target < lo + mind) {
#pragma unroll
          for (int r = 0; r < kSeedCtas; ++r) atomicMax(cluster.map_shared_rank(&s_pick[i], r), s_mine);
        }
      }
    }
    cluster.sync();
    for (int i = 0; i < next; ++i) {
      int pk = s_pick[i];
      if (pk < 0) pk = (int)(hash_u32(seed, (uint32_t)h, (uint32_t)(npicked + i) + 77777u) % (uint32_t)m);
      for (int j = 0; j < i; ++j)
        if (picks[j] == pk) pk = (pk + 1 + i) % m;  // two draws of a round hit the same token
      picks[i] = pk;
    }
    cnt = next;
  }
  cluster.sync();  // no CTA may exit while peers can still write its shared memory
}

int launch_seed_pp(int bh, int n, int d, int c, const bf16* x, int oversample, uint32_t seed, float* cent,
                   cudaStream_t st) {
  long long mm = (long long)oversample * c;
  if (mm > n) mm = n;
  if (mm > kSeedThreads * kSeedCtas) mm = kSeedThreads * kSeedCtas;  // subsample capacity
  const int m = (int)mm;
  if (m < c) return SVGEAR_EUNSUPPORTED;  // more clusters than the subsample can hold
  if (d == 128)
    seed_pp_kernel<128><<<bh * kSeedCtas, kSeedThreads, 0, st>>>(x, n, c, m, seed, cent);
  else
    seed_pp_kernel<64><<<bh * kSeedCtas, kSeedThreads, 0, st>>>(x, n, c, m, seed, cent);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg

// ------------------------------------------------------------------------------------------------
// Seeding from a precomputed Gram matrix of the subsample (G = Xs Xs^T, bf16, a plain library GEMM
// done by the caller): d^2(s, c) = G[s][s] + G[c][c] - 2 G[c][s], so a round only reads the Gram
// rows of its new centres (8 KB each) instead of every subsample token.  One CTA per instance,
// 4 subsample tokens per thread, no cluster needed.  Same D^2 rounds as seed_pp_kernel.
// ------------------------------------------------------------------------------------------------
namespace svg {

constexpr int kGramPer = 4;  // samples per thread (m <= 4096)
constexpr int kGramBatch = 8;  // centres drawn per round while many remain (graded down towards the end)

__global__ void __launch_bounds__(1024)
    seed_gram_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gram, int n, int d, int c, int m,
                     uint32_t seed, int first, float* __restrict__ cent) {
  const int h = blockIdx.x;
  __shared__ float s_warp[32];
  __shared__ float s_total;
  __shared__ int s_pick[kGramBatch];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bf16* xh = x + (size_t)h * n * d;
  const bf16* gh = gram + (size_t)h * m * m;
  float* ch = cent + (size_t)h * c * d;
  auto sample_row = [&](int s) -> size_t { return (size_t)(((long long)s * n) / m); };
  const int s0 = tid * kGramPer;
  float nrm[kGramPer], mind[kGramPer];
#pragma unroll
  for (int e = 0; e < kGramPer; ++e) {
    const int s = s0 + e;
    nrm[e] = s < m ? __bfloat162float(gh[(size_t)s * m + s]) : 0.f;
    mind[e] = s < m ? INFINITY : 0.f;
  }
  int picks[kGramBatch];
  picks[0] = (int)(hash_u32(seed, (uint32_t)(first + h), 0u) % (uint32_t)m);
  int cnt = 1, npicked = 0;
  while (true) {
    for (int e = tid; e < cnt * d; e += 1024) {
      const int i = e / d, k = e % d;
      ch[(size_t)(npicked + i) * d + k] = __bfloat162float(xh[sample_row(picks[i]) * d + k]);
    }
    npicked += cnt;
    if (npicked >= c) break;
    for (int i = 0; i < cnt; ++i) {
      const int pc = picks[i];
      const float nc = __bfloat162float(gh[(size_t)pc * m + pc]);
      const bf16* grow = gh + (size_t)pc * m;
      float g[kGramPer];
      if (s0 + kGramPer <= m && (m & 3) == 0) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(grow + s0));
        g[0] = __uint_as_float(u.x << 16); g[1] = __uint_as_float(u.x & 0xffff0000u);
        g[2] = __uint_as_float(u.y << 16); g[3] = __uint_as_float(u.y & 0xffff0000u);
      } else {
#pragma unroll
        for (int e = 0; e < kGramPer; ++e) g[e] = s0 + e < m ? __bfloat162float(grow[s0 + e]) : 0.f;
      }
#pragma unroll
      for (int e = 0; e < kGramPer; ++e) {
        const float d2 = (s0 + e == pc) ? 0.f : fmaxf(nrm[e] + nc - 2.f * g[e], 0.f);
        if (s0 + e < m) mind[e] = fminf(mind[e], d2);
      }
    }
    float mine = 0.f;
#pragma unroll
    for (int e = 0; e < kGramPer; ++e) mine += mind[e];
    float inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    __syncthreads();  // previous round's readers of s_warp / s_pick are done
    if (lane == 31) s_warp[warp] = inc;
    if (tid < kGramBatch) s_pick[tid] = -1;
    __syncthreads();
    if (warp == 0) {
      float w = s_warp[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
      if (lane == 31) s_total = wi;
    }
    __syncthreads();
    const float total = s_total;
    const int left = c - npicked;
    // the draws of a round share one D^2 distribution; the later a centre is drawn the more the
    // distribution it is drawn from matters, so the batch shrinks towards the end
    const int next = left >= 256 ? kGramBatch : (left >= 128 ? 4 : (left >= 32 ? 2 : 1));
    if (total > 0.f && mine > 0.f) {
      const float lo = s_warp[warp] + inc - mine;
      for (int i = 0; i < next; ++i) {
        const float u = ((float)(hash_u32(seed, (uint32_t)(first + h), (uint32_t)(npicked + i) + 1u) >> 8) + 0.5f) *
                        (1.0f / 16777216.0f);
        const float target = u * total;
        if (target >= lo && target < lo + mine) {
          float run = lo;
          int chosen = -1;
#pragma unroll
          for (int e = 0; e < kGramPer; ++e) {
            run += mind[e];
            if (chosen < 0 && target < run && mind[e] > 0.f) chosen = s0 + e;
          }
          if (chosen < 0) {  // rounding: fall back to this thread's largest entry
            float best = -1.f;
#pragma unroll
            for (int e = 0; e < kGramPer; ++e)
              if (mind[e] > best) { best = mind[e]; chosen = s0 + e; }
          }
          atomicMax(&s_pick[i], chosen);
        }
      }
    }
    __syncthreads();
    for (int i = 0; i < next; ++i) {
      int pk = s_pick[i];
      if (pk < 0 || pk >= m) pk = (int)(hash_u32(seed, (uint32_t)(first + h), (uint32_t)(npicked + i) + 77777u) % (uint32_t)m);
      for (int j = 0; j < i; ++j)
        if (picks[j] == pk) pk = (pk + 1 + i) % m;
      picks[i] = pk;
    }
    cnt = next;
  }
}

int launch_seed_gram(int bh, int n, int d, int c, int m, const bf16* x, const bf16* gram, uint32_t seed,
                     float* cent, cudaStream_t st, int first_instance) {
  if (m > 1024 * kGramPer || m < c) return SVGEAR_ESHAPE;
  seed_gram_kernel<<<bh, 1024, 0, st>>>(x, gram, n, d, c, m, seed, first_instance, cent);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
