// The reference's k-means++ draw, on the device, bit for bit.
//
// Reference: clustering._kmeans_pp_init (/root/reference/pkg/src/routedattn/clustering.py:65-84) driven by
// numpy's Generator(PCG64) seeded from SeedSequence(entropy=side_seed, spawn_key=(restart,))
// (clustering.py:178-180):
//     idx_0 = rng.integers(n);  d2 = ((x - x[idx_0])**2).sum(axis=1)
//     for c in 1..k-1:  total = d2.sum()
//                       idx_c = rng.choice(n, p=d2/total)  if total > 0  else  lowest unused index
//                       d2 = minimum(d2, ((x - x[idx_c])**2).sum(axis=1))
// To return the SAME centres as numpy, every floating-point operation is done in float64 in numpy's
// order (no fused multiply-adds: explicit __d*_rn intrinsics):
//   * row sums and d2.sum(): numpy's pairwise summation (8 interleaved accumulators on blocks of
//     <= 128 elements, combined ((0+1)+(2+3))+((4+5)+(6+7)); longer arrays split recursively at
//     n/2 rounded down to a multiple of 8);
//   * choice(p=): cdf = cumsum(p) SEQUENTIALLY, cdf /= cdf[-1], index = searchsorted(cdf, u, "right")
//     with u = (next_uint64 >> 11) * 2^-53;
//   * integers(n): Lemire's bounded 32-bit draw on PCG64's buffered 32-bit output.
// The PCG64 state of every instance comes from the host (SeedSequence hashing is a few integer
// operations in numpy); everything after that runs here.  One thread-block cluster per instance:
// all CTAs update the distances of their token range, CTA 0 draws.  The sequential cumsum is one
// dependent float64 add per token per round (staged through shared memory; ≈0.3 ms per round at
// 75,600 tokens) — this is the parity path (seed-faithful centres at any scale without a host stage), not the production
// seeding (seed.cu).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace svg {

namespace {

constexpr int kRefThreads = 512;
constexpr int kRefMaxCl = 8;
constexpr int kCdfChunk = 4096;  // float64 values per staging buffer of the sequential cumsum (a multiple of 8)

struct Pcg64 {
  unsigned __int128 state, inc;
  int has32;
  uint32_t u32;
  __device__ uint64_t next64() {
    const unsigned __int128 mult = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ uint32_t next32() {  // numpy's pcg64_next32: the high half of an output is kept for the next call
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __device__ uint32_t bounded(uint32_t n) {  // Generator.integers(n), n <= 2^32: buffered_bounded_lemire_uint32
    const uint32_t rng = n - 1u;
    if (rng == 0u) return 0u;
    const uint64_t excl = (uint64_t)rng + 1u;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  __device__ double uniform() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

// numpy's pairwise sum of a[0..n), n <= 128 (one leaf of the recursion)
// (the values were written by other CTAs of the cluster in this launch: L2 loads)
__device__ __forceinline__ double leaf_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, __ldcg(a + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = __ldcg(a + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __ldcg(a + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, __ldcg(a + i));
  return res;
}

// squared distance of one bf16 row to the centre row (float64 in shared memory): the D products in
// numpy's pairwise order for D in {64, 128} (a single leaf)
template <int D>
__device__ __forceinline__ double row_d2(const bf16* __restrict__ xr, const double* __restrict__ cen) {
  double r[8];
  const uint4* p = reinterpret_cast<const uint4*>(xr);
#pragma unroll
  for (int blk = 0; blk < D / 8; ++blk) {
    const uint4 u = __ldg(p + blk);
    float f[8];
    unpack8(u, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double df = __dsub_rn((double)f[j], cen[blk * 8 + j]);
      const double sq = __dmul_rn(df, df);
      r[j] = blk == 0 ? sq : __dadd_rn(r[j], sq);
    }
  }
  return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                   __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
}

template <int D>
__global__ void __launch_bounds__(kRefThreads, 1)
    seed_reference_kernel(const bf16* __restrict__ x, int n, int c, const uint64_t* __restrict__ pcg_states,
                          float* __restrict__ cent, int32_t* __restrict__ picks_out, double* __restrict__ ws_d2,
                          double* __restrict__ ws_cdf, double* __restrict__ ws_leaf, uint8_t* __restrict__ ws_chosen,
                          int32_t* __restrict__ ws_pick, int32_t* __restrict__ ws_leaftab, int nleaf_cap) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  const int h = (int)blockIdx.x / CL;
  const int tid = threadIdx.x;
  const bf16* xh = x + (size_t)h * n * D;
  double* d2 = ws_d2 + (size_t)h * n;
  double* cdf = ws_cdf + (size_t)h * n;
  double* leaf = ws_leaf + (size_t)h * nleaf_cap;
  uint8_t* chosen = ws_chosen + (size_t)h * n;
  int32_t* pick_slot = ws_pick + h;
  float* ch = cent + (size_t)h * c * D;
  extern __shared__ __align__(16) double s_chunk[];  // [2][kCdfChunk]: staging of the sequential cumsum
  __shared__ double s_cen[D];
  __shared__ int s_idx, s_nleaf;
  __shared__ double s_total;
  __shared__ int s_min[kRefThreads / 32];
  const int per = (n + CL - 1) / CL;
  const int lo = min(n, rank * per), hi = min(n, lo + per);

  Pcg64 g;  // only thread 0 of CTA 0 draws
  if (rank == 0 && tid == 0) {
    const uint64_t* st = pcg_states + (size_t)h * 4;
    g.state = ((unsigned __int128)st[0] << 64) | st[1];
    g.inc = ((unsigned __int128)st[2] << 64) | st[3];
    g.has32 = 0;
    g.u32 = 0;
    *pick_slot = (int)g.bounded((uint32_t)n);
  }
  for (int t = lo + tid; t < hi; t += kRefThreads) chosen[t] = 0;
  // leaves of numpy's pairwise recursion over [0, n) (n is fixed: one table per instance, built once):
  // longer arrays split at n/2 rounded down to a multiple of 8, leaves hold <= 128 elements
  int32_t* leaftab = ws_leaftab + (size_t)h * 2 * nleaf_cap;
  if (rank == 0 && tid == 0) {
    int stack_lo[40], stack_n[40], sp = 1, nl = 0;
    stack_lo[0] = 0; stack_n[0] = n;
    while (sp > 0) {
      --sp;
      const int l0 = stack_lo[sp], ln = stack_n[sp];
      if (ln <= 128) {
        leaftab[2 * nl] = l0; leaftab[2 * nl + 1] = ln; ++nl;
      } else {
        int n2 = ln / 2;
        n2 -= n2 % 8;
        stack_lo[sp] = l0 + n2; stack_n[sp] = ln - n2; ++sp;  // right child below the left one
        stack_lo[sp] = l0; stack_n[sp] = n2; ++sp;
      }
    }
    s_nleaf = nl;
  }
  __threadfence();
  cluster.sync();

  for (int round = 0; round < c; ++round) {
    const int idx = __ldcg(pick_slot);
    // the new centre: float64 copy for the distances, float32 row of the output
    if (tid < D) {
      const float v = __bfloat162float(xh[(size_t)idx * D + tid]);
      s_cen[tid] = (double)v;
      if (rank == 0) ch[(size_t)round * D + tid] = v;
    }
    if (rank == 0 && tid == 0) {
      chosen[idx] = 1;
      if (picks_out) picks_out[(size_t)h * c + round] = idx;
    }
    __syncthreads();
    if (round + 1 == c) break;
    // d2 = minimum(d2, |x - centre|^2)
    for (int t = lo + tid; t < hi; t += kRefThreads) {
      const double v = row_d2<D>(xh + (size_t)t * D, s_cen);
      d2[t] = round == 0 ? v : fmin(__ldcg(d2 + t), v);
    }
    __threadfence();
    cluster.sync();
    if (rank == 0) {
      // total = d2.sum(): leaves of numpy's recursion in parallel, then the same combine order
      const int nleaf = s_nleaf;
      for (int i = tid; i < nleaf; i += kRefThreads) leaf[i] = leaf_sum(d2 + leaftab[2 * i], leaftab[2 * i + 1]);
      __syncthreads();
      if (tid == 0) {
        // combine: post-order evaluation with a value stack (node = left + right)
        int stack_lo[40], stack_n[40], stack_state[40], sp = 0, next_leaf = 0;
        double val[40];
        int vp = 0;
        stack_lo[0] = 0; stack_n[0] = n; stack_state[0] = 0; sp = 1;
        while (sp > 0) {
          const int l0 = stack_lo[sp - 1], ln = stack_n[sp - 1];
          if (ln <= 128) {
            val[vp++] = leaf[next_leaf++];
            --sp;
          } else if (stack_state[sp - 1] == 0) {
            stack_state[sp - 1] = 1;
            int n2 = ln / 2;
            n2 -= n2 % 8;
            stack_lo[sp] = l0 + n2; stack_n[sp] = ln - n2; stack_state[sp] = 0; ++sp;  // right (evaluated second)
            stack_lo[sp] = l0; stack_n[sp] = n2; stack_state[sp] = 0; ++sp;            // left (evaluated first)
          } else {
            const double b = val[--vp], a = val[--vp];
            val[vp++] = __dadd_rn(a, b);
            --sp;
          }
        }
        s_total = val[0];
      }
      __syncthreads();
      const double total = s_total;
      if (total > 0.0) {
        // p = d2 / total, cdf = cumsum(p) SEQUENTIALLY (one dependent add per token, thread 0), staged
        // through shared memory in chunks: while thread 0 runs the chain over chunk k, the other threads
        // write chunk k-1 back and bring chunk k+1 in (the same thread stores and reloads a slot)
        const int nchunks = (n + kCdfChunk - 1) / kCdfChunk;
        for (int i = tid; i < min(kCdfChunk, n); i += kRefThreads) s_chunk[i] = __ddiv_rn(__ldcg(d2 + i), total);
        __syncthreads();
        double s = 0.0;
        for (int kch = 0; kch < nchunks; ++kch) {
          double* cur = s_chunk + (kch & 1) * kCdfChunk;
          double* oth = s_chunk + ((kch + 1) & 1) * kCdfChunk;
          const int c0 = kch * kCdfChunk, len = min(kCdfChunk, n - c0);
          if (tid == 0) {
            // the adds are the dependent chain: batches of 8 through registers (loads of a batch are
            // independent), scalar tail
            int i = 0;
            for (; i + 8 <= len; i += 8) {
              double v[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) v[j] = cur[i + j];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                s = __dadd_rn(s, v[j]);
                v[j] = s;
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) cur[i + j] = v[j];
            }
            for (; i < len; ++i) {
              s = __dadd_rn(s, cur[i]);
              cur[i] = s;
            }
          } else {
            const int p0 = c0 - kCdfChunk, plen = kch > 0 ? kCdfChunk : 0;
            const int n0 = c0 + kCdfChunk, nlen = max(0, min(kCdfChunk, n - n0));
            for (int i = tid - 1; i < max(plen, nlen); i += kRefThreads - 1) {
              if (i < plen) cdf[p0 + i] = oth[i];
              if (i < nlen) oth[i] = __ddiv_rn(__ldcg(d2 + n0 + i), total);
            }
          }
          __syncthreads();
        }
        {
          const int kl = nchunks - 1, c0 = kl * kCdfChunk, len = n - c0;
          const double* cur = s_chunk + (kl & 1) * kCdfChunk;
          for (int i = tid; i < len; i += kRefThreads) cdf[c0 + i] = cur[i];
        }
        __syncthreads();
        if (tid == 0) {
          const double last = s;
          const double u = g.uniform();
          // searchsorted(cdf / last, u, side="right"): first index whose normalised value exceeds u
          int a = 0, b = n;
          while (a < b) {
            const int mid = (a + b) >> 1;
            if (__ddiv_rn(cdf[mid], last) <= u) a = mid + 1; else b = mid;
          }
          s_idx = a;
        }
      } else {
        // every token coincides with a chosen centre: the lowest unused index (clustering.py:78-81)
        int best = 0x7fffffff;
        for (int t = tid; t < n; t += kRefThreads)
          if (!__ldcg(chosen + t)) { best = t; break; }
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if ((tid & 31) == 0) s_min[tid >> 5] = best;
        __syncthreads();
        if (tid == 0) {
          for (int w = 1; w < kRefThreads / 32; ++w) best = min(best, s_min[w]);
          s_idx = best;
        }
      }
      __syncthreads();
      if (tid == 0) *pick_slot = s_idx;
      __threadfence();
    }
    cluster.sync();
  }
}

}  // namespace

size_t seed_reference_ws_bytes(int bh, int n) {
  const size_t nleaf_cap = (size_t)n / 32 + 64;
  return align_up((size_t)bh * n * 8, 256) * 2 + align_up((size_t)bh * nleaf_cap * 8, 256) * 2 +
         align_up((size_t)bh * n, 256) + align_up((size_t)bh * 4, 256) + 1024;
}

int launch_seed_reference(int bh, int n, int d, int c, const bf16* x, const uint64_t* pcg_states, float* cent,
                          int32_t* picks, void* ws, size_t ws_bytes, cudaStream_t st) {
  Carver cv(ws, ws_bytes);
  const int nleaf_cap = n / 32 + 64;
  double* w_d2 = cv.take<double>((size_t)bh * n);
  double* w_cdf = cv.take<double>((size_t)bh * n);
  double* w_leaf = cv.take<double>((size_t)bh * nleaf_cap);
  uint8_t* w_chosen = cv.take<uint8_t>((size_t)bh * n);
  int32_t* w_pick = cv.take<int32_t>(bh);
  int32_t* w_leaftab = cv.take<int32_t>((size_t)bh * 2 * nleaf_cap);
  if (!cv.ok) return SVGEAR_EWORKSPACE;
  const size_t smem = (size_t)2 * kCdfChunk * sizeof(double);
  SVG_CUDA_OK(cudaFuncSetAttribute(seed_reference_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SVG_CUDA_OK(cudaFuncSetAttribute(seed_reference_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int cl = 1;
  while (cl < kRefMaxCl && n / (cl * 2) >= 2048) cl *= 2;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(bh * cl));
  lc.blockDim = dim3(kRefThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (d == 128)
    SVG_CUDA_OK(cudaLaunchKernelEx(&lc, seed_reference_kernel<128>, x, n, c, pcg_states, cent, picks, w_d2, w_cdf, w_leaf,
                                   w_chosen, w_pick, w_leaftab, nleaf_cap));
  else
    SVG_CUDA_OK(cudaLaunchKernelEx(&lc, seed_reference_kernel<64>, x, n, c, pcg_states, cent, picks, w_d2, w_cdf, w_leaf,
                                   w_chosen, w_pick, w_leaftab, nleaf_cap));
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
