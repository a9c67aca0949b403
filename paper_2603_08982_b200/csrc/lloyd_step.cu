// One launch per Lloyd iteration for everything that is not the distance contraction.
//
// Reference step: clustering._lloyd (clustering.py:104-141) after the argmin —
//   bincount (:115), empty-cluster repair (:116-124), convergence test (:130-131), member means
//   (:133-135) — plus kmeans' stable argsort / offsets (:197-198), and the bookkeeping the
//   tensor-core assignment of the NEXT iteration needs (split-bf16 centre pieces, Hamerly bound
//   update, active-token list).
//
// One thread-block CLUSTER serves one instance (hardware co-scheduled, so the phases are separated
// by cluster barriers and nothing can deadlock against other kernels).  CTA r owns the contiguous
// token range r; every warp of it owns a contiguous sub-range, which makes the counting sort stable
// without any cross-warp ordering:
//   A1  per-warp histograms of the assignments (+ "did anything change" against the previous ones)
//   A2  cluster sizes = sum of the CTA histograms through distributed shared memory
//   A3  (rare) empty clusters: exact own distances, donor search across the cluster, redo A1-A2
//   A4  converged?  -> done[h], the instance costs nothing from here on
//   A5  stable permutation: offsets + earlier CTAs + earlier warps + rank inside the warp step
//   B1  member means of the clusters whose membership changed (fixed order, f64), centre movement
//   B2  next iteration: centre pieces, big movers, bound update + active list
// No floating-point atomics; every result is bit-identical to the unfused kernels it replaces.
#include <cooperative_groups.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace svg {

namespace {

constexpr int kStepThreads = 512;
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kMaxCl = 16;
constexpr int kTeams = kStepThreads / 128;  // 128-thread teams of the mean phase
constexpr int kMaxMovers = 64;
constexpr int kPieces = 2;

struct Cand {
  float val;
  int idx;
  int from;
  int pad;
};

__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, 128;" ::"r"(team + 1) : "memory");
}

// exclusive scan of v[0..c) into out[0..c), c <= kMaxClusters, whole block
__device__ void block_exclusive_scan(const int32_t* v, int32_t* out, int c, int32_t* s_warp) {
  constexpr int PER = kMaxClusters / kStepThreads;  // 8 consecutive entries per thread
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int loc[PER], tot = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = tid * PER + u;
    loc[u] = j < c ? v[j] : 0;
    tot += loc[u];
  }
  int inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < kStepWarps ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kStepWarps) s_warp[lane] = wi - w;
  }
  __syncthreads();
  int run = s_warp[warp] + inc - tot;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = tid * PER + u;
    if (j < c) out[j] = run;
    run += loc[u];
  }
  __syncthreads();
}

// exact fp32 squared distance of token row `xr` to centre row `cr`: lanes split the row, fixed tree
__device__ __forceinline__ float own_dist_row(const bf16* xr, const float* cr, int d, int lane) {
  float acc = 0.f;
  for (int k = lane * 2; k < d; k += 64) {
    const uint32_t xb = __ldg(reinterpret_cast<const uint32_t*>(xr + k));
    const float2 cc = *reinterpret_cast<const float2*>(cr + k);
    const float d0 = __uint_as_float(xb << 16) - cc.x, d1 = __uint_as_float(xb & 0xffff0000u) - cc.y;
    acc = fmaf(d0, d0, acc);
    acc = fmaf(d1, d1, acc);
  }
  return warp_sum(acc);
}

// Member mean of cluster j by one 128-thread team: rows in ascending order, 32 at a time, warp w of
// the team owns rows 8w..8w+7 of each group (f64 chains), partials combined (0+1)+(2+3).  Two groups
// of row loads are kept in flight; the order of the additions is unchanged.
template <int D>
__device__ __forceinline__ void team_mean(const bf16* __restrict__ xh, const int32_t* __restrict__ permh, int j,
                                          int nj, int o, float* __restrict__ cent_row, float* norm_out,
                                          float* move_out, double* part, float* s_c, float* s_dc, int team,
                                          int ttid) {
  constexpr int EPL = D / 32;
  const int lane = ttid & 31, warp = ttid >> 5;
  double acc[EPL];
#pragma unroll
  for (int u = 0; u < EPL; ++u) acc[u] = 0.0;
  int nx0 = 0, nx1 = 0;
  if (lane < nj) nx0 = __ldcg(permh + o + lane);
  if (32 + lane < nj) nx1 = __ldcg(permh + o + 32 + lane);
  for (int base = 0; base < nj; base += 64) {
    const int pidx0 = nx0, pidx1 = nx1;
    if (base + 64 + lane < nj) nx0 = __ldcg(permh + o + base + 64 + lane);  // next batch's rows
    if (base + 96 + lane < nj) nx1 = __ldcg(permh + o + base + 96 + lane);
    uint2 buf[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int r = warp * 8 + (q & 7);
      const int row = __shfl_sync(0xffffffffu, q < 8 ? pidx0 : pidx1, r);
      buf[q] = make_uint2(0u, 0u);
      if (base + (q < 8 ? 0 : 32) + r < nj) {
        const bf16* p = xh + (size_t)row * D + lane * EPL;
        if (EPL == 4) buf[q] = __ldg(reinterpret_cast<const uint2*>(p));
        else buf[q].x = __ldg(reinterpret_cast<const uint32_t*>(p));
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      acc[0] += (double)__uint_as_float(buf[q].x << 16);
      acc[1] += (double)__uint_as_float(buf[q].x & 0xffff0000u);
      if constexpr (EPL == 4) {
        acc[2] += (double)__uint_as_float(buf[q].y << 16);
        acc[3] += (double)__uint_as_float(buf[q].y & 0xffff0000u);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < EPL; ++u) part[warp * D + lane * EPL + u] = acc[u];
  team_sync(team);
  if (ttid < D) {
    float m;
    const float old = cent_row[ttid];
    if (nj > 0) {
      const double s = (part[ttid] + part[D + ttid]) + (part[2 * D + ttid] + part[3 * D + ttid]);
      m = (float)(s / (double)nj);
      cent_row[ttid] = m;
    } else {
      m = old;
    }
    s_c[ttid] = m;
    s_dc[ttid] = m - old;
  }
  team_sync(team);
  if (warp == 0) {
    float s = 0.f, mv = 0.f;
    for (int k = lane; k < D; k += 32) {
      s = fmaf(s_c[k], s_c[k], s);
      mv = fmaf(s_dc[k], s_dc[k], mv);
    }
    s = warp_sum(s);
    mv = warp_sum(mv);
    if (lane == 0) {
      *norm_out = s;
      *move_out = sqrtf(mv);
    }
  }
  team_sync(team);  // part / s_c are reused by the team's next cluster
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(kStepThreads, 2) lloyd_step_kernel(const LloydStepArgs A) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int h = (int)blockIdx.x / CL;
  const int n = A.n, c = A.c, it = A.iter;
  const bool pre0 = it < 0;
  if (!pre0 && A.done[h]) return;  // done[h] is only written behind a cluster barrier of an earlier phase

  extern __shared__ __align__(16) uint8_t smem_raw[];
  // [scratch: per-warp histograms | refined-token bits | team mean scratch | mover centres]
  // [s_cta c] [s_sizes c] [s_off c] [s_list c]
  int32_t* hist = reinterpret_cast<int32_t*>(smem_raw);
  int32_t* s_cta = reinterpret_cast<int32_t*>(smem_raw + A.scratch_bytes);
  int32_t* s_sizes = s_cta + c;
  int32_t* s_off = s_sizes + c;
  int32_t* s_list = s_off + c;
  __shared__ int32_t s_warp[32];
  __shared__ float s_redf[3][kStepWarps];
  __shared__ int s_redi[kStepWarps];
  __shared__ Cand s_cand[2][kMaxCl];
  __shared__ float s_T[2][kMaxCl];
  __shared__ int s_diff, s_count;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bf16* xh = A.x + (size_t)h * n * D;
  int32_t* assign = A.assign + (size_t)h * n;
  float* cent = A.cent + (size_t)h * c * D;
  const float* cnorm = A.cnorm + (size_t)h * c;
  // token range of this CTA and sub-range of this warp (multiples of 32 so that warp steps stay aligned)
  const int per = ceil_div(ceil_div(n, CL), 32) * 32;
  const int lo = min(n, rank * per), hi = min(n, lo + per);
  const int wsort = A.wsort;
  const int wper = ceil_div(ceil_div(hi - lo, wsort), 32) * 32;
  const int wlo = min(hi, lo + warp * wper), whi = warp < wsort ? min(hi, wlo + wper) : wlo;
  constexpr int kBatch = 8;  // warp steps whose loads are issued together (the passes are latency bound)

  bool finished = false;  // converged in this launch (cluster-uniform)
  int nlist = 0;          // clusters whose centre was recomputed in B1 (list in s_list)
  if (pre0) {
    // ---------------------------------------------------------------- before the first iteration
    if (rank == 0) {
      if (tid == 0) {
        A.done[h] = 0;
        A.iters_run[h] = 0;
        A.nactive[h] = 0;
        A.resid_nz[h] = 0;
        if (A.iters) A.iters[h] = 0;
      }
      for (int j = tid; j < c; j += kStepThreads) A.move[(size_t)h * c + j] = 0.f;
    }
    for (int j = rank * kStepWarps + warp; j < c; j += CL * kStepWarps) {  // |c|^2 of the start centres
      const float* p = cent + (size_t)j * D;
      float s = 0.f;
      for (int k = lane; k < D; k += 32) s = fmaf(p[k], p[k], s);
      s = warp_sum(s);
      if (lane == 0) A.cnorm[(size_t)h * c + j] = s;
    }
  } else if (A.phases & 1) {
    // ---------------------------------------------------------------- A1/A2: histograms, sizes
    int32_t* prev = A.prev + (size_t)h * n;
    bool repaired = false;
    int changed = 0;
    while (true) {
      for (int i = tid; i < wsort * c; i += kStepThreads) hist[i] = 0;
      __syncthreads();
      int diff = 0;
      for (int b0 = wlo; b0 < whi; b0 += 32 * kBatch) {
        int a[kBatch], p[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int t = b0 + u * 32 + lane;
          a[u] = t < whi ? assign[t] : -1;
          p[u] = (t < whi && it > 0) ? prev[t] : a[u];
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          if (a[u] >= 0) atomicAdd(&hist[warp * c + a[u]], 1);
          diff |= (p[u] != a[u]);
        }
      }
      diff = __syncthreads_or(diff);
      for (int j = tid; j < c; j += kStepThreads) {
        int s = 0;
        for (int w = 0; w < wsort; ++w) s += hist[w * c + j];
        s_cta[j] = s;
      }
      if (tid == 0) s_diff = diff;
      cluster.sync();
      int empty = 0;
      for (int j = tid; j < c; j += kStepThreads) {
        int tot = 0, before = 0;
#pragma unroll 4
        for (int r = 0; r < CL; ++r) {
          const int v = *cluster.map_shared_rank(&s_cta[j], r);
          if (r < rank) before += v;
          tot += v;
        }
        s_sizes[j] = tot;
        s_off[j] = before;  // members in earlier CTAs (turned into scatter bases below)
        empty |= (tot == 0);
      }
      int ch = 0;
      if (tid < CL) ch = *cluster.map_shared_rank(&s_diff, tid);
      changed = __syncthreads_or(ch);
      empty = __syncthreads_or(empty);
      if (!empty || repaired) break;
      // -------------------------------------------------------------- A3: empty-cluster repair
      // (clustering.py:116-124) empty clusters in ascending order; donor = token with the largest
      // own distance (first maximum) among clusters that still have >= 2 members.  The own distances
      // the tensor-core assignment stored are rounded, and stale for skipped tokens, so donors are
      // ranked by EXACT distances (fp32 sum of squared differences against the current centres) —
      // computed only for tokens that can still be the maximum: every token has an upper bound
      // (ub^2 + margin) and, if it was evaluated against its current centre, a lower bound
      // (own - margin); a token is refined iff its upper bound reaches the best lower bound.
      float* own = A.own + (size_t)h * n;
      const float* ubh = A.ub + (size_t)h * n;
      const float* xnorm = A.xnorm + (size_t)h * n;
      uint32_t* refined = reinterpret_cast<uint32_t*>(smem_raw);  // one bit per token of this CTA
      int32_t* cand = A.active + (size_t)h * n + lo;              // scratch: the active list is dead here
      const bool prune = A.use_tc != 0;
      for (int i = tid; i < ceil_div(per, 32); i += kStepThreads) refined[i] = prune ? 0u : 0xffffffffu;
      float cn = 0.f;
      for (int j = tid; j < c; j += kStepThreads) cn = fmaxf(cn, cnorm[j]);
      cn = warp_max(cn);
      if (lane == 0) s_redf[2][warp] = cn;
      if (tid == 0) s_count = 0;
      __syncthreads();
      cn = s_redf[2][0];
      for (int w = 1; w < kStepWarps; ++w) cn = fmaxf(cn, s_redf[2][w]);
      if (warp == 0) {  // ascending list of the empty clusters (identical on every CTA)
        int cnt = 0;
        for (int base = 0; base < c; base += 32) {
          const int j = base + lane;
          const bool f = j < c && s_sizes[j] == 0;
          const unsigned bal = __ballot_sync(0xffffffffu, f);
          if (f) s_list[cnt + __popc(bal & ((1u << lane) - 1u))] = j;
          cnt += __popc(bal);
        }
        if (lane == 0) s_count = cnt;
      }
      __syncthreads();
      const int ne = s_count;
      for (int ei = 0; ei < ne; ++ei) {
        const int e = s_list[ei];
        if (prune) {
          // best lower bound over the eligible tokens of the whole instance
          float tl = -1.f;
          for (int t = lo + tid; t < hi; t += kStepThreads) {
            if (s_sizes[assign[t]] >= 2) {
              const float o = own[t];
              float lbv;
              if (refined[(t - lo) >> 5] >> ((t - lo) & 31) & 1u) lbv = o;
              else lbv = sqrtf(o) == ubh[t] ? o - (xnorm[t] + cn) * (1.0f / 4096.0f) : 0.f;
              tl = fmaxf(tl, lbv);
            }
          }
          tl = warp_max(tl);
          __syncthreads();
          if (lane == 0) s_redf[0][warp] = tl;
          if (tid == 0) s_count = 0;
          __syncthreads();
          if (warp == 0) {
            tl = lane < kStepWarps ? s_redf[0][lane] : -1.f;
            tl = warp_max(tl);
            if (lane < CL) *cluster.map_shared_rank(&s_T[ei & 1][rank], lane) = tl;
          }
          cluster.sync();
          float T = s_T[ei & 1][0];
          for (int r = 1; r < CL; ++r) T = fmaxf(T, s_T[ei & 1][r]);
          // refine every eligible token whose upper bound reaches T
          for (int t = lo + tid; t < hi; t += kStepThreads) {
            if (s_sizes[assign[t]] >= 2 && !(refined[(t - lo) >> 5] >> ((t - lo) & 31) & 1u)) {
              const float u = ubh[t];
              const float hib = u * u * (1.0f + 1.0f / 1024.0f) + (xnorm[t] + cn) * (1.0f / 4096.0f);
              if (hib >= T) cand[atomicAdd(&s_count, 1)] = t;
            }
          }
          __syncthreads();
          const int ncand = s_count;
          for (int i0 = warp * 4; i0 < ncand; i0 += kStepWarps * 4) {
            float v[4];
            int tt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              tt[u] = cand[min(i0 + u, ncand - 1)];
              v[u] = own_dist_row(xh + (size_t)tt[u] * D, cent + (size_t)assign[tt[u]] * D, D, lane);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (lane == 0 && i0 + u < ncand) {
                own[tt[u]] = v[u];
                atomicOr(&refined[(tt[u] - lo) >> 5], 1u << ((tt[u] - lo) & 31));
              }
          }
          __syncthreads();
        }
        float bv = -1.f;
        int bx = 0x7fffffff;
        for (int t = lo + tid; t < hi; t += kStepThreads) {
          if (s_sizes[assign[t]] >= 2 && (refined[(t - lo) >> 5] >> ((t - lo) & 31) & 1u)) {
            const float v = own[t];
            if (v > bv) { bv = v; bx = t; }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int ox = __shfl_xor_sync(0xffffffffu, bx, o);
          if (ov > bv || (ov == bv && ox < bx)) { bv = ov; bx = ox; }
        }
        if (lane == 0) { s_redf[0][warp] = bv; s_redi[warp] = bx; }
        __syncthreads();
        if (warp == 0) {
          bv = lane < kStepWarps ? s_redf[0][lane] : -1.f;
          bx = lane < kStepWarps ? s_redi[lane] : 0x7fffffff;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int ox = __shfl_xor_sync(0xffffffffu, bx, o);
            if (ov > bv || (ov == bv && ox < bx)) { bv = ov; bx = ox; }
          }
          Cand cd;
          cd.val = bv; cd.idx = bx; cd.from = bx != 0x7fffffff ? assign[bx] : -1; cd.pad = 0;
          if (lane < CL) *cluster.map_shared_rank(&s_cand[ei & 1][rank], lane) = cd;
        }
        cluster.sync();
        if (tid == 0) {
          Cand best = s_cand[ei & 1][0];
          for (int r = 1; r < CL; ++r) {
            const Cand o = s_cand[ei & 1][r];
            if (o.val > best.val || (o.val == best.val && o.idx < best.idx)) best = o;
          }
          if (best.idx != 0x7fffffff) {
            s_sizes[best.from] -= 1;
            s_sizes[e] += 1;
            if (best.idx >= lo && best.idx < hi) {  // the owner of the token applies the move
              assign[best.idx] = e;
              own[best.idx] = 0.f;
              if (A.bounded_state) {  // both memberships changed; the moved token is re-evaluated next time
                A.dirty[(size_t)h * c + best.from] = 1;
                A.dirty[(size_t)h * c + e] = 1;
                A.ub[(size_t)h * n + best.idx] = 0.f;
                A.lb[(size_t)h * n + best.idx] = 0.f;
              }
            }
          }
        }
        __syncthreads();
      }
      repaired = true;
      cluster.sync();  // nobody still reads the old CTA histograms; redo them from the repaired assignments
    }
    // ---------------------------------------------------------------- A4: decision, sizes, offsets
    finished = it > 0 && !changed;
    // scatter bases: offsets[j] + members in earlier CTAs (+ earlier warps below)
    for (int j = tid; j < c; j += kStepThreads) s_list[j] = s_off[j];
    __syncthreads();
    block_exclusive_scan(s_sizes, s_off, c, s_warp);
    if (rank == 0) {
      for (int j = tid; j < c; j += kStepThreads) {
        A.sizes[(size_t)h * c + j] = s_sizes[j];
        A.offsets[(size_t)h * c + j] = s_off[j];
      }
      if (tid == 0) {
        if (A.iters) A.iters[h] = it + 1;
        A.iters_run[h] = it + 1;
        A.nactive[h] = 0;  // the next iteration's filter appends to an empty list
        if (finished) A.done[h] = 1;  // assignments unchanged -> converged
      }
    }
    if (!finished) {
      // -------------------------------------------------------------- A5: stable permutation
      for (int j = tid; j < c; j += kStepThreads) {
        int run = s_off[j] + s_list[j];
        for (int w = 0; w < wsort; ++w) {
          const int cnt = hist[w * c + j];
          hist[w * c + j] = run;
          run += cnt;
        }
      }
      __syncthreads();
      int32_t* perm = A.perm + (size_t)h * n;
      int32_t* wh = hist + warp * c;
      for (int b0 = wlo; b0 < whi; b0 += 32 * kBatch) {
        int a[kBatch], pos[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int t = b0 + u * 32 + lane;
          a[u] = t < whi ? assign[t] : (0x7fffff00 | lane);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const bool valid = b0 + u * 32 + lane < whi;
          const unsigned m = __match_any_sync(0xffffffffu, a[u]);
          const int leader = __ffs(m) - 1;
          int base = 0;
          if (valid && lane == leader) {
            base = wh[a[u]];
            wh[a[u]] = base + __popc(m);
          }
          __syncwarp();
          pos[u] = __shfl_sync(0xffffffffu, base, leader) + __popc(m & ((1u << lane) - 1u));
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int t = b0 + u * 32 + lane;
          if (t < whi) {
            perm[pos[u]] = t;
            prev[t] = a[u];
          }
        }
      }
    }
  } else {
    // phase B alone (the caller ran the inertia kernels in between): reload what A left in memory
    for (int j = tid; j < c; j += kStepThreads) {
      s_sizes[j] = A.sizes[(size_t)h * c + j];
      s_off[j] = A.offsets[(size_t)h * c + j];
    }
  }
  if (finished || (!pre0 && !(A.phases & 2))) {
    cluster.sync();  // peers may still be reading this CTA's shared memory
    return;
  }
  __threadfence();
  cluster.sync();  // the permutation (all CTAs) is complete and visible; no remote shared-memory access below

  if (!pre0) {
    // ------------------------------------------------------------------ B1: member means
    if (tid == 0) s_count = 0;
    __syncthreads();
    const uint8_t* dirty = A.bounded ? A.dirty + (size_t)h * c : nullptr;
    // flags first (one L2 round trip for all of them; s_cta is dead: peers read it before the barrier above)
    for (int j = tid; j < c; j += kStepThreads) s_cta[j] = !dirty || __ldcg(dirty + j);
    __syncthreads();
    if (warp == 0) {
      int cnt = 0;
      for (int base = 0; base < c; base += 32) {
        const int j = base + lane;
        const bool f = j < c && s_cta[j];
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (f) s_list[cnt + __popc(bal & ((1u << lane) - 1u))] = j;
        else if (j < c && rank == 0) A.move[(size_t)h * c + j] = 0.f;  // same members in the same order
        cnt += __popc(bal);
      }
      if (lane == 0) s_count = cnt;
    }
    __syncthreads();
    nlist = s_count;
    const int team = tid >> 7, ttid = tid & 127;
    double* part = reinterpret_cast<double*>(smem_raw) + (size_t)team * (4 * D);
    float* s_c = reinterpret_cast<float*>(smem_raw + (size_t)kTeams * 4 * D * sizeof(double)) + (size_t)team * 2 * D;
    float* s_dc = s_c + D;
    const int32_t* permh = A.perm + (size_t)h * n;
    for (int i = rank * kTeams + team; i < nlist; i += CL * kTeams) {
      const int j = s_list[i];
      team_mean<D>(xh, permh, j, s_sizes[j], s_off[j], cent + (size_t)j * D, A.cnorm + (size_t)h * c + j,
                   A.move + (size_t)h * c + j, part, s_c, s_dc, team, ttid);
    }
    if (it + 1 >= A.max_iters || !A.use_tc) return;
    __threadfence();
    cluster.sync();  // centres, norms and movements of every cluster are complete and visible
  } else {
    if (!A.use_tc) return;
    __threadfence();
    cluster.sync();
  }

  // -------------------------------------------------------------------- B2: next iteration's inputs
  const bool all_active = !A.bounded || pre0;
  {  // fp32 centres -> kPieces bf16 pieces [piece][cpad][D] + padded norms (inf beyond c); only the
     // centres that were recomputed (all of them, and the padding rows, before the first iteration)
    const int cpad = A.cpad;
    int nz = 0;
    bf16* pieces = A.pieces + (size_t)h * kPieces * cpad * D;
    const int total = pre0 ? cpad * D : nlist * D;
    for (int i = rank * kStepThreads + tid; i < total; i += CL * kStepThreads) {
      const int j = pre0 ? i / D : s_list[i / D];
      const int idx = j * D + i % D;
      float v = j < c ? __ldcg(cent + idx) : 0.f;
#pragma unroll
      for (int p = 0; p < kPieces; ++p) {
        const bf16 b = __float2bfloat16_rn(v);
        pieces[(size_t)p * cpad * D + idx] = b;
        v -= __bfloat162float(b);
        if (p == 0) nz |= (v != 0.f);
      }
      if (i % D == 0) A.cnorm_pad[(size_t)h * cpad + j] = j < c ? __ldcg(cnorm + j) : INFINITY;
    }
    // centres that are exactly bf16 (start centres picked from the tokens) need only the first piece;
    // the flag is sticky: a zero second piece contributes exact zeros
    if (__syncthreads_or(nz) && tid == 0) atomicOr(&A.resid_nz[h], 1);
  }
  uint8_t* dirty_w = A.dirty + (size_t)h * c;
  if (rank == 0 && A.bounded_state)
    for (int j = tid; j < c; j += kStepThreads) dirty_w[j] = all_active ? 1 : 0;
  int32_t* active = A.active + (size_t)h * n;
  if (all_active) {
    for (int t = lo + tid; t < hi; t += kStepThreads) active[t] = t;
    if (rank == 0 && tid == 0) A.nactive[h] = n;
    return;
  }
  // Hamerly bound update.  A few centres that moved far (typically clusters refilled by the repair)
  // would void every token's lower bound through the global max-movement term; the big movers
  // L = {j : move[j] > max_move / 4} (|L| <= kMaxMovers) are bounded through the inter-centre
  // distance instead: dist(x, c_e) >= dist(c_a, c_e) - ub(x) >= dmin[a] - ub(x).
  const float* mv = A.move + (size_t)h * c;
  float m1 = 0.f, m2 = 0.f, cn = 0.f;
  int a1 = -1;
  for (int j = tid; j < c; j += kStepThreads) {
    const float v = __ldcg(mv + j);
    if (v > m1) { m2 = m1; m1 = v; a1 = j; } else if (v > m2) m2 = v;
    cn = fmaxf(cn, __ldcg(cnorm + j));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om1 = __shfl_xor_sync(0xffffffffu, m1, o), om2 = __shfl_xor_sync(0xffffffffu, m2, o);
    const int oa1 = __shfl_xor_sync(0xffffffffu, a1, o);
    if (om1 > m1) { m2 = fmaxf(m1, om2); m1 = om1; a1 = oa1; } else m2 = fmaxf(m2, om1);
    cn = fmaxf(cn, __shfl_xor_sync(0xffffffffu, cn, o));
  }
  if (lane == 0) { s_redf[0][warp] = m1; s_redf[1][warp] = m2; s_redf[2][warp] = cn; s_redi[warp] = a1; }
  if (tid == 0) s_count = 0;
  __syncthreads();
  m1 = s_redf[0][0]; m2 = s_redf[1][0]; cn = s_redf[2][0]; a1 = s_redi[0];
  for (int w = 1; w < kStepWarps; ++w) {
    if (s_redf[0][w] > m1) { m2 = fmaxf(m1, s_redf[1][w]); m1 = s_redf[0][w]; a1 = s_redi[w]; } else m2 = fmaxf(m2, s_redf[0][w]);
    cn = fmaxf(cn, s_redf[2][w]);
  }
  // big movers (thresholds on the un-inflated movements, as the bounds below inflate them)
  const float thr = m1 * 0.25f;
  float rest = 0.f;
  for (int j = tid; j < c; j += kStepThreads) {
    const float v = __ldcg(mv + j);
    if (v > thr && m1 > 0.f) {
      const int pos = atomicAdd(&s_count, 1);
      if (pos < kMaxMovers) s_list[pos] = j;
    } else {
      rest = fmaxf(rest, v);
    }
  }
  rest = warp_max(rest);
  __syncthreads();
  if (lane == 0) s_redf[0][warp] = rest;
  __syncthreads();
  rest = s_redf[0][0];
  for (int w = 1; w < kStepWarps; ++w) rest = fmaxf(rest, s_redf[0][w]);
  const int nl = s_count;
  const bool movers = !(nl == 0 || nl > kMaxMovers || c <= nl);
  float* dmin = A.dmin + (size_t)h * c;
  if (movers) {
    float* s_mc = reinterpret_cast<float*>(smem_raw);  // [nl][D] centres of the big movers
    for (int i = tid; i < nl * D; i += kStepThreads) s_mc[i] = __ldcg(cent + (size_t)s_list[i / D] * D + i % D);
    __syncthreads();
    // 8 lanes per cluster (D/8 consecutive elements each), 4 clusters per warp
    constexpr int epl = D / 8;
    const int sub = lane & 7;
    for (int a0 = (rank * kStepWarps + warp) * 4; a0 < c; a0 += CL * kStepWarps * 4) {
      const int a = a0 + (lane >> 3);
      const int aa = min(a, c - 1);
      float ca[epl];
#pragma unroll
      for (int k = 0; k < epl; ++k) ca[k] = __ldcg(cent + (size_t)aa * D + sub * epl + k);
      float best = INFINITY;
      for (int q = 0; q < nl; ++q) {
        const float* mc = s_mc + q * D + sub * epl;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < epl; ++k) {
          const float df = ca[k] - mc[k];
          acc = fmaf(df, df, acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        if (s_list[q] != aa) best = fminf(best, acc);
      }
      if (a < c && sub == 0) dmin[a] = sqrtf(best) * (1.0f - 1.0f / 65536.0f);
    }
    __threadfence();
    cluster.sync();  // every CTA's share of dmin is visible
  }
  // movements are rounded fp32 norms: inflate them slightly so the bounds stay bounds
  constexpr float kInfl = 1.0f + 1.0f / 65536.0f;
  m1 *= kInfl; m2 *= kInfl;
  const float mrest = rest * kInfl;
  const float* xnorm = A.xnorm + (size_t)h * n;
  float* ub = A.ub + (size_t)h * n;
  float* lb = A.lb + (size_t)h * n;
  constexpr int kFB = 4;  // warp steps per batch of the filter
  for (int b0 = lo + warp * (32 * kFB); b0 < hi; b0 += kStepWarps * 32 * kFB) {
    int a[kFB];
    float u[kFB], l[kFB], xn[kFB], mva[kFB], dm[kFB];
#pragma unroll
    for (int s = 0; s < kFB; ++s) {
      const int t = min(b0 + s * 32 + lane, hi - 1);
      a[s] = assign[t];
      u[s] = ub[t];
      l[s] = lb[t];
      xn[s] = xnorm[t];
    }
#pragma unroll
    for (int s = 0; s < kFB; ++s) {
      mva[s] = __ldcg(mv + a[s]);
      dm[s] = movers ? __ldcg(dmin + a[s]) : 0.f;
    }
    unsigned bal[kFB];
    int cnt = 0;
#pragma unroll
    for (int s = 0; s < kFB; ++s) {
      const int t = b0 + s * 32 + lane;
      bool act = false;
      if (t < hi) {
        const float uu = u[s] + mva[s] * kInfl;
        const float ll = movers ? fminf(l[s] - mrest, dm[s] - uu) : l[s] - (a[s] == a1 ? m2 : m1);
        ub[t] = uu;
        lb[t] = ll;
        // squared-space margin: the evaluated distances carry an absolute error of a few
        // 2^-17 (|x|^2 + |c|^2) (2-piece bf16 split + fp32 accumulation); 2^-12 covers it 30x
        const float marg = (xn[s] + cn) * (1.0f / 4096.0f);
        act = !(ll > 0.f && uu * uu * kInfl + marg < ll * ll * (2.0f - kInfl));
      }
      bal[s] = __ballot_sync(0xffffffffu, act);
      cnt += __popc(bal[s]);
    }
    if (cnt) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&A.nactive[h], cnt);
      base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
      for (int s = 0; s < kFB; ++s) {
        if (bal[s] >> lane & 1u) active[base + __popc(bal[s] & ((1u << lane) - 1u))] = b0 + s * 32 + lane;
        base += __popc(bal[s]);
      }
    }
  }
}


// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
namespace {

// Cluster size (<= 16, >= ~1024 tokens per CTA): the largest for which all instances of the call fit
// in about one CTA per SM.  The token passes are latency bound, so more CTAs per instance help, but
// the query side, the key side and a second head group run the same kernel concurrently on other
// streams: a launch that claims every CTA slot serialises them (measured: 45.9 ms/layer with
// bh*cl = 280, 43.8 ms with 140).  The occupancy query (it knows the GPC structure) confirms that
// the clusters are co-resident; cached per (cl, smem bucket).
template <int D>
int pick_cluster_size(int bh, int n, size_t smem, int max_cl) {
  static std::mutex mu;
  static int cache[kMaxCl + 1][32];
  static bool init = false;
  std::lock_guard<std::mutex> lk(mu);
  if (!init) {
    for (auto& row : cache)
      for (int& v : row) v = -1;
    init = true;
  }
  static const int forced = [] {
    const char* e = getenv("SVGEAR_LLOYD_CLUSTER");
    return e ? atoi(e) : 0;
  }();
  if (forced >= 1 && forced <= max_cl) return forced;
  const int bucket = (int)(smem / 8192) < 31 ? (int)(smem / 8192) : 31;
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      num_sms = 148;
  }
  int top = n / 1024;
  if (top > max_cl) top = max_cl;
  if (top > (num_sms + 12) / bh) top = (num_sms + 12) / bh;
  for (int cl = top; cl > 1; --cl) {
    int& occ = cache[cl][bucket];
    if (occ < 0) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3((unsigned)cl);
      q.blockDim = dim3(kStepThreads);
      q.dynamicSmemBytes = (size_t)(bucket + 1) * 8192;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, lloyd_step_kernel<D>, &q) != cudaSuccess) {
        (void)cudaGetLastError();
        nclusters = 0;
      }
      occ = nclusters;
    }
    if (occ >= bh) return cl;
  }
  return 1;
}

template <int D>
int launch_step_t(const LloydStepArgs& args, int bh, cudaStream_t st) {
  static int max_smem = 0, max_cl = 8;
  auto kern = lloyd_step_kernel<D>;
  if (max_smem == 0) {
    int dev = 0, v = 0;
    SVG_CUDA_OK(cudaGetDevice(&dev));
    SVG_CUDA_OK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    v -= 2048;  // static shared memory of the kernel
    SVG_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) max_cl = kMaxCl;
    (void)cudaGetLastError();
    max_smem = v;
  }
  // scratch region: per-warp histograms, or the mean teams' partials, or the big movers' centres
  const int c = args.c;
  const size_t fixed = (size_t)4 * c * sizeof(int32_t);
  const size_t team_bytes = (size_t)kTeams * (4 * D * sizeof(double) + 2 * D * sizeof(float));
  const size_t mover_bytes = (size_t)kMaxMovers * D * sizeof(float);
  const size_t budget = 100 * 1024;  // two CTAs per SM stay possible
  int wsort = kStepWarps;
  while (wsort > 1 && (size_t)wsort * c * 4 + fixed > budget) --wsort;
  size_t scratch = (size_t)wsort * c * 4;
  if (scratch < team_bytes) scratch = team_bytes;
  if (scratch < mover_bytes) scratch = mover_bytes;
  scratch = align_up(scratch, 16);
  // ... or one bit per token of a CTA (repair); sized for the smallest cluster this launch may get
  size_t smem = scratch + fixed;
  if ((long long)smem > max_smem) return SVGEAR_ESHAPE;
  const int cl = pick_cluster_size<D>(bh, args.n, smem, max_cl);
  const size_t bits = align_up((size_t)ceil_div(ceil_div(args.n, cl), 32) * 4 + 128, 16);
  if (bits > scratch) {
    scratch = bits;
    smem = scratch + fixed;
    if ((long long)smem > max_smem) return SVGEAR_ESHAPE;
  }
  LloydStepArgs a = args;
  a.wsort = wsort;
  a.scratch_bytes = (int)scratch;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(bh * cl));
  lc.blockDim = dim3(kStepThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  SVG_CUDA_OK(cudaLaunchKernelEx(&lc, kern, a));
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}
}  // namespace

int launch_lloyd_step(const LloydStepArgs& args, int bh, int d, cudaStream_t st) {
  return d == 128 ? launch_step_t<128>(args, bh, st) : launch_step_t<64>(args, bh, st);
}

}  // namespace svg
