// Device-side k-means++ seeding (D^2 sampling, clustering.py:65-84) on a strided SUBSAMPLE of
// m = min(n, oversample*c, 4096) tokens with a counter-based hash RNG.  It is NOT the reference's
// draw (that needs numpy's generator over all n tokens, host side: the Python shim's parity
// switch); it is the start the operator uses when the caller supplies no centres.
//
// Two kernels per side:
//   gram_tc_kernel   G = Xs Xs^T (bf16, fp32 accumulation in TMEM) on the tensor cores: one CTA per
//                    128-row tile of Xs walks all 128-column tiles; rows gathered with cp.async
//                    into the SWIZZLE_128B UMMA layout, tcgen05.mma SS, double-buffered TMEM.
//   seed_gram_kernel the sequential D^2 rounds: d^2(s, c) = G[s][s] + G[c][c] - 2 G[c][s], so a
//                    round only reads the Gram rows of its new centres (8 KB each) instead of every
//                    subsample token.  One CTA per instance, 4 subsample tokens per thread; centres
//                    are drawn in rounds of 8/4/2/1 (graded by how many remain), the Gram rows of a
//                    round are loaded together.  Deterministic.
#include "tc_common.cuh"

namespace svg {

using namespace tc;

namespace {

constexpr int GT = 128;        // Gram tile (rows and columns)
constexpr int GTHREADS = 224;  // warps 0-3 epilogue, 4 and 6 producers, 5 MMA issuer

enum { GB_AFULL = 0, GB_BFULL = 1 /*[2]*/, GB_BEMPTY = 3 /*[2]*/, GB_ACCFULL = 5 /*[2]*/, GB_ACCEMPTY = 7 /*[2]*/ };

template <int D>
struct GSmem {
  static constexpr int kTile = GT * D * 2;
  static constexpr int kA = 0;
  static constexpr int kB = kTile;          // 2 stages
  static constexpr int kBars = 3 * kTile;
  static constexpr int kStage = kBars + 128;  // epilogue staging: 4 warps x 32 rows x (64 + 16) bytes
  static constexpr size_t bytes() { return 1024 + kStage + 4 * 32 * 80; }
};

__device__ __forceinline__ size_t sample_row(int s, int n, int m) { return (size_t)(((long long)s * n) / m); }

template <int D>
__global__ void __launch_bounds__(GTHREADS)
    gram_tc_kernel(const bf16* __restrict__ x, int n, int m, bf16* __restrict__ gram) {
  using L = GSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase + L::kA, sB = sbase + L::kB, bars = sbase + L::kBars;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBars + 96);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = blockIdx.y, i0 = blockIdx.x * GT;
  const int NT = (m + GT - 1) / GT;
  const bf16* xh = x + (size_t)h * n * D;
  auto bar = [&](int i) -> uint32_t { return bars + 8u * (uint32_t)i; };
  if (tid == 0) {
    mbar_init(bar(GB_AFULL), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(GB_BFULL + b), 1);
      mbar_init(bar(GB_BEMPTY + b), 1);
      mbar_init(bar(GB_ACCFULL + b), 1);
      mbar_init(bar(GB_ACCEMPTY + b), 128);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(smem_u32(tmem_slot), 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4 || warp == 6) {
    // ---- producers: gather 128 subsample rows per tile (16-byte chunks, swizzled).  Two warps take
    // alternate column tiles so that two gathers are in flight; warp 4 also brings the row tile.
    // Token row of sample s = floor(s*n/m): one 64-bit divide per lane per tile, then exact
    // fixed-stride stepping (a divide per gathered row dominated the first version of this kernel).
    constexpr int CPR = D / 8, RPI = 32 / CPR;
    const int sub = lane / CPR, chunk = lane % CPR;
    const long long step_num = (long long)RPI * n;
    const int step_q = (int)(step_num / m), step_r = (int)(step_num % m);
    const size_t last_row = sample_row(m - 1, n, m);
    auto load_tile = [&](uint32_t dst, int s0) {
      const long long num = (long long)(s0 + sub) * n;
      int row = (int)(num / m), rem = (int)(num % m);
#pragma unroll 4
      for (int r0 = 0; r0 < GT; r0 += RPI) {
        const int r = r0 + sub;
        const size_t src = s0 + r < m ? (size_t)row : last_row;
        cp_async16(dst + (uint32_t)((chunk >> 3) * (GT * 128)) + swz(r, chunk & 7), xh + src * D + chunk * 8);
        row += step_q;
        rem += step_r;
        if (rem >= m) { rem -= m; ++row; }
      }
      cp_async_commit();
      cp_async_wait_all();
      fence_proxy_async();
      __syncwarp();
    };
    if (warp == 4) {
      load_tile(sA, i0);
      if (lane == 0) mbar_arrive(bar(GB_AFULL));
    }
    for (int jt = warp == 4 ? 0 : 1; jt < NT; jt += 2) {
      const int st = jt & 1;
      if (jt >= 2) mbar_wait(bar(GB_BEMPTY + st), ((jt >> 1) - 1) & 1);
      load_tile(sB + (uint32_t)st * L::kTile, jt * GT);
      if (lane == 0) mbar_arrive(bar(GB_BFULL + st));
    }
  } else if (warp == 5) {
    // ---- MMA issuer -----------------------------------------------------------------------------
    if (elect_one()) {
      const uint32_t idesc = make_idesc(GT, GT, 0);
      mbar_wait(bar(GB_AFULL), 0);
      for (int jt = 0; jt < NT; ++jt) {
        const int st = jt & 1;
        mbar_wait(bar(GB_BFULL + st), (jt >> 1) & 1);
        if (jt >= 2) mbar_wait(bar(GB_ACCEMPTY + st), ((jt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t bb = sB + (uint32_t)st * L::kTile;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = make_desc(sA + (uint32_t)((kk >> 2) * (GT * 128) + (kk & 3) * 32), 16, 1024);
          const uint64_t bd = make_desc(bb + (uint32_t)((kk >> 2) * (GT * 128) + (kk & 3) * 32), 16, 1024);
          umma_ss(tmem + (uint32_t)(st * GT), ad, bd, idesc, kk > 0 ? 1u : 0u);
        }
        umma_commit(bar(GB_BEMPTY + st));
        umma_commit(bar(GB_ACCFULL + st));
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ---- epilogue: fp32 accumulators -> bf16 rows of G ------------------------------------------
    const int r = warp * 32 + lane, s = i0 + r;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    bf16* grow = gram + ((size_t)h * m + min(s, m - 1)) * m;
    const bool vec = (m & 7) == 0;
    uint8_t* stage = smem + L::kStage + warp * (32 * 80);
    for (int jt = 0; jt < NT; ++jt) {
      const int st = jt & 1;
      mbar_wait(bar(GB_ACCFULL + st), (jt >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < GT; cb += 32) {
        uint32_t a[32];
        TMEM_LD32(tmem + lane_base + (uint32_t)(st * GT + cb), a);
        tc_wait_ld();
        const int col0 = jt * GT + cb;
        if (vec) {
          // through shared memory so that a warp instruction writes 8 rows x 64 contiguous bytes (full
          // sectors); a thread writing 16 bytes of its own row filled half a sector per store
          uint8_t* mine = stage + lane * 80;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 o;
            o.x = pack_bf16x2(__uint_as_float(a[q * 8 + 0]), __uint_as_float(a[q * 8 + 1]));
            o.y = pack_bf16x2(__uint_as_float(a[q * 8 + 2]), __uint_as_float(a[q * 8 + 3]));
            o.z = pack_bf16x2(__uint_as_float(a[q * 8 + 4]), __uint_as_float(a[q * 8 + 5]));
            o.w = pack_bf16x2(__uint_as_float(a[q * 8 + 6]), __uint_as_float(a[q * 8 + 7]));
            *reinterpret_cast<uint4*>(mine + q * 16) = o;
          }
          __syncwarp();
#pragma unroll
          for (int rr = 0; rr < 32; rr += 8) {
            const int row = rr + (lane >> 2), q = lane & 3;
            const int srow = i0 + warp * 32 + row;
            if (srow < m && col0 + q * 8 < m)
              *reinterpret_cast<uint4*>(gram + ((size_t)h * m + srow) * m + col0 + q * 8) =
                  *reinterpret_cast<const uint4*>(stage + row * 80 + q * 16);
          }
          __syncwarp();
        } else if (s < m) {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (col0 + q < m) grow[col0 + q] = __float2bfloat16_rn(__uint_as_float(a[q]));
        }
      }
      tc_fence_before();
      mbar_arrive(bar(GB_ACCEMPTY + st));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

__device__ __forceinline__ uint32_t hash_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t x = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du;
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}

constexpr int kGramPer = 4;    // samples per thread (m <= 4096)
constexpr int kGramBatch = 8;  // centres drawn per round while many remain (graded down towards the end)
#ifndef SVG_SEED_T8
#define SVG_SEED_T8 256
#define SVG_SEED_T4 128
#define SVG_SEED_T2 32
#endif
constexpr int kSeedT8 = SVG_SEED_T8, kSeedT4 = SVG_SEED_T4, kSeedT2 = SVG_SEED_T2;  // centres left: 8 / 4 / 2 per round
// The last centres are drawn GREEDILY (greedy k-means++: several D^2 candidates per round, the one that
// lowers the potential most is kept).  Plain D^2 sampling spends many of its last draws inside clusters
// that already hold a centre (when u well-separated clusters are still uncovered, a draw lands in one of
// them with probability ~ u*R / (u*R + c), R = between / within squared distance), and every such draw
// leaves one cluster with two centres and one without - the configuration Lloyd's iteration resolves
// slowest - the larger the clusters, the slower (a split cluster of 250 tokens keeps a Wan2.2 query side
// iterating for 20 rounds).  A greedy round costs about two plain rounds, so their number follows the
// cluster size: the last min(c/2, (n/c)^2 / 512) centres (124 of 300 query-side, 11 of 1000 key-side
// centres at the Wan2.2 shape; key-side iteration counts do not react to more).  SVG_SEED_GREEDY (compile time) overrides the count, 0 = plain sampling throughout.
#ifndef SVG_SEED_GREEDY
#define SVG_SEED_GREEDY -1
#endif
// The draws of a batched round share one D^2 distribution, so two of them can land in the same
// uncovered cluster (probability ~ batch^2 / 2u per round).  A draw is dropped when an earlier draw of
// its round lies closer to it than half its distance to the nearest existing centre (one Gram entry per
// pair, read by one warp): had the round been sequential, the earlier draw would have covered it.
// Measured at the Wan2.2 shape: query-side Lloyd iterations 438 -> 398 in sum but 15 -> 19 at most, +0.4 ms
// of key-side seeding, layer time unchanged - off by default.
#ifndef SVG_SEED_FILTER
#define SVG_SEED_FILTER 0
#endif

__global__ void __launch_bounds__(1024)
    seed_gram_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gram, int n, int d, int c, int m,
                     uint32_t seed, int first, int greedy_left, float* __restrict__ cent) {
  const int h = blockIdx.x;
  __shared__ float s_warp[32];
  __shared__ float s_total;
  __shared__ int s_pick[kGramBatch];
  __shared__ float s_target[kGramBatch];
  __shared__ float s_red[32][kGramBatch + 1];  // greedy rounds: per-warp potential gains of the candidates
  __shared__ float s_gain[kGramBatch];
  __shared__ float s_pmind[kGramBatch];  // D^2 of the round's draws
  __shared__ int s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bf16* xh = x + (size_t)h * n * d;
  const bf16* gh = gram + (size_t)h * m * m;
  float* ch = cent + (size_t)h * c * d;
  const int s0 = tid * kGramPer;
  const bool vec = s0 + kGramPer <= m && (m & 3) == 0;
  __shared__ float s_diag[1024 * kGramPer];    // G[s][s] = |x_s|^2
  __shared__ int32_t s_rows[1024 * kGramPer];  // token row of sample s
  float nrm[kGramPer], mind[kGramPer];
#pragma unroll
  for (int e = 0; e < kGramPer; ++e) {
    const int s = s0 + e;
    nrm[e] = s < m ? __bfloat162float(gh[(size_t)s * m + s]) : 0.f;
    mind[e] = s < m ? INFINITY : 0.f;
    s_diag[s] = nrm[e];
    s_rows[s] = s < m ? (int32_t)sample_row(s, n, m) : 0;
  }
  __syncthreads();
  int picks[kGramBatch];
#pragma unroll
  for (int i = 0; i < kGramBatch; ++i) picks[i] = 0;
  picks[0] = (int)(hash_u32(seed, (uint32_t)(first + h), 0u) % (uint32_t)m);
  int cnt = 1, npicked = 0;
  while (true) {
    // all global loads of the round are issued before anything consumes them: the Gram rows of the
    // new centres (unless this is the last round), then the centre tokens themselves
    const bool more = npicked + cnt < c;
    uint2 gu[kGramBatch];
#pragma unroll
    for (int i = 0; i < kGramBatch; ++i)
      if (more && i < cnt && vec) gu[i] = __ldg(reinterpret_cast<const uint2*>(gh + (size_t)picks[i] * m + s0));
    for (int e = tid; e < cnt * d; e += 1024) {
      const int i = e / d, k = e % d;
      int pk = picks[0];
#pragma unroll
      for (int j = 1; j < kGramBatch; ++j) pk = i == j ? picks[j] : pk;
      ch[(size_t)(npicked + i) * d + k] = __bfloat162float(xh[(size_t)s_rows[pk] * d + k]);
    }
    npicked += cnt;
    if (!more) break;
#pragma unroll
    for (int i = 0; i < kGramBatch; ++i) {
      if (i < cnt) {
        const float nc = s_diag[picks[i]];
        float g[kGramPer];
        if (vec) {
          g[0] = __uint_as_float(gu[i].x << 16); g[1] = __uint_as_float(gu[i].x & 0xffff0000u);
          g[2] = __uint_as_float(gu[i].y << 16); g[3] = __uint_as_float(gu[i].y & 0xffff0000u);
        } else {  // ragged subsample sizes (small shapes only)
          const bf16* grow = gh + (size_t)picks[i] * m;
#pragma unroll
          for (int e = 0; e < kGramPer; ++e) g[e] = s0 + e < m ? __bfloat162float(grow[s0 + e]) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < kGramPer; ++e) {
          const float d2 = (s0 + e == picks[i]) ? 0.f : fmaxf(nrm[e] + nc - 2.f * g[e], 0.f);
          if (s0 + e < m) mind[e] = fminf(mind[e], d2);
        }
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
    __syncthreads();  // previous round's readers of s_warp / s_pick / s_target are done
    if (lane == 31) s_warp[warp] = inc;
    if (tid < kGramBatch) s_pick[tid] = -1;
    __syncthreads();
    const int left = c - npicked;
    // the draws of a round share one D^2 distribution; the later a centre is drawn the more the
    // distribution it is drawn from matters, so the batch shrinks towards the end
    const bool greedy = left <= greedy_left;  // kGramBatch candidates, one centre
    const int next = greedy ? kGramBatch : (left >= kSeedT8 ? kGramBatch : (left >= kSeedT4 ? 4 : (left >= kSeedT2 ? 2 : 1)));
    if (warp == 0) {
      float w = s_warp[lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[lane] = wi - w;
      const float total = __shfl_sync(0xffffffffu, wi, 31);
      if (lane == 31) s_total = total;
      // sampling targets of the round: once, not by every thread (the round is issue bound)
      if (lane < next) {
        const float u = ((float)(hash_u32(seed, (uint32_t)(first + h), (uint32_t)(npicked + lane) + 1u) >> 8) + 0.5f) *
                        (1.0f / 16777216.0f);
        s_target[lane] = u * total;
      }
    }
    __syncthreads();
    if (s_total > 0.f && mine > 0.f) {
      const float lo = s_warp[warp] + inc - mine;
      for (int i = 0; i < next; ++i) {
        const float target = s_target[i];
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
          float cm = mind[0];
#pragma unroll
          for (int e = 1; e < kGramPer; ++e) cm = chosen == s0 + e ? mind[e] : cm;
          s_pmind[i] = cm;  // a target lies in exactly one thread's interval
        }
      }
    }
    __syncthreads();
    if (tid == 0) {  // resolve the round's picks once (unclaimed targets, two draws on one token)
      int pk_prev[kGramBatch];
#pragma unroll
      for (int i = 0; i < kGramBatch; ++i) {
        if (i < next) {
          int pk = s_pick[i];
          if (pk < 0 || pk >= m) {
            pk = (int)(hash_u32(seed, (uint32_t)(first + h), (uint32_t)(npicked + i) + 77777u) % (uint32_t)m);
            s_pmind[i] = 0.f;  // fallback draws are never dropped
          }
#pragma unroll
          for (int j = 0; j < kGramBatch; ++j)
            if (j < i && pk_prev[j] == pk) { pk = (pk + 1 + i) % m; s_pmind[i] = 0.f; }
          pk_prev[i] = pk;
          s_pick[i] = pk;
        }
      }
    }
    __syncthreads();
    int kept = next;
    if (SVG_SEED_FILTER && !greedy && next > 1) {
      if (warp == 0) {
        // lane = pair (i < j) of the round's draws, i-major
        int pi = 0, pj = 1, rem = lane;
#pragma unroll
        for (int i = 0; i < kGramBatch - 1; ++i) {
          const int row = kGramBatch - 1 - i;
          if (rem >= 0 && rem < row) { pi = i; pj = i + 1 + rem; rem = -1; }
          else if (rem >= 0) rem -= row;
        }
        bool close = false;
        if (rem < 0 && pj < next) {
          const int a = s_pick[pi], b = s_pick[pj];
          const float dab = fmaxf(s_diag[a] + s_diag[b] - 2.f * __bfloat162float(gh[(size_t)a * m + b]), 0.f);
          close = dab < 0.5f * s_pmind[pj];
        }
        const unsigned bits = __ballot_sync(0xffffffffu, close);
        if (lane == 0) {
          unsigned keep = 1u;
          int w = 1;
          for (int j = 1; j < next; ++j) {
            bool drop = false;
            int idx = 0;
            for (int i = 0; i < kGramBatch - 1; ++i)
              for (int jj = i + 1; jj < kGramBatch; ++jj, ++idx)
                if (jj == j && (keep >> i & 1u) && (bits >> idx & 1u)) drop = true;
            if (!drop) {
              keep |= 1u << j;
              s_pick[w++] = s_pick[j];
            }
          }
          s_cnt = w;
        }
      }
      __syncthreads();
      kept = s_cnt;
    }
#pragma unroll
    for (int i = 0; i < kGramBatch; ++i)
      if (i < kept) picks[i] = s_pick[i];
    cnt = kept;
    if (greedy) {
      // potential gain of candidate i: sum over the samples of max(0, D^2 - d^2(sample, candidate)), in a
      // fixed summation order (thread-local, warp shuffle tree, 32 warps by one warp per candidate)
      float gain[kGramBatch];
#pragma unroll
      for (int i = 0; i < kGramBatch; ++i) {
        const float nc = s_diag[picks[i]];
        float g[kGramPer];
        if (vec) {
          const uint2 u = __ldg(reinterpret_cast<const uint2*>(gh + (size_t)picks[i] * m + s0));
          g[0] = __uint_as_float(u.x << 16); g[1] = __uint_as_float(u.x & 0xffff0000u);
          g[2] = __uint_as_float(u.y << 16); g[3] = __uint_as_float(u.y & 0xffff0000u);
        } else {
          const bf16* grow = gh + (size_t)picks[i] * m;
#pragma unroll
          for (int e = 0; e < kGramPer; ++e) g[e] = s0 + e < m ? __bfloat162float(grow[s0 + e]) : 0.f;
        }
        float acc = 0.f;
#pragma unroll
        for (int e = 0; e < kGramPer; ++e) {
          const float d2 = (s0 + e == picks[i]) ? 0.f : fmaxf(nrm[e] + nc - 2.f * g[e], 0.f);
          if (s0 + e < m) acc += fmaxf(mind[e] - d2, 0.f);
        }
        gain[i] = acc;
      }
#pragma unroll
      for (int i = 0; i < kGramBatch; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gain[i] += __shfl_xor_sync(0xffffffffu, gain[i], o);
        if (lane == 0) s_red[warp][i] = gain[i];
      }
      __syncthreads();
      if (warp < kGramBatch) {
        float v = s_red[lane][warp];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_gain[warp] = v;
      }
      __syncthreads();
      int best = 0;
      float bg = s_gain[0];
#pragma unroll
      for (int i = 1; i < kGramBatch; ++i)
        if (s_gain[i] > bg) { bg = s_gain[i]; best = i; }
      int pk = picks[0];
#pragma unroll
      for (int i = 1; i < kGramBatch; ++i) pk = best == i ? picks[i] : pk;
      picks[0] = pk;  // the next round loads its Gram row again (an L2 hit now)
      cnt = 1;
    }
  }
}

}  // namespace

int seed_subsample(int n, int c, int oversample) {
  long long m = (long long)oversample * c;
  if (m > n) m = n;
  if (m > 1024 * kGramPer) m = 1024 * kGramPer;
  return (int)m;
}

// k-means++ start centres of `bh` instances -> cent [bh][c][d] f32; gram_ws holds bh*m*m bf16
int launch_seed(int bh, int n, int d, int c, int oversample, const bf16* x, uint32_t seed, int first_instance,
                float* cent, bf16* gram_ws, cudaStream_t st) {
  const int m = seed_subsample(n, c, oversample);
  if (m < c) return SVGEAR_ESHAPE;  // more clusters than the subsample can hold
  const dim3 grid((unsigned)ceil_div(m, GT), (unsigned)bh);
  if (d == 128) {
    const size_t smem = GSmem<128>::bytes();
    SVG_CUDA_OK(cudaFuncSetAttribute(gram_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gram_tc_kernel<128><<<grid, GTHREADS, smem, st>>>(x, n, m, gram_ws);
  } else {
    const size_t smem = GSmem<64>::bytes();
    SVG_CUDA_OK(cudaFuncSetAttribute(gram_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gram_tc_kernel<64><<<grid, GTHREADS, smem, st>>>(x, n, m, gram_ws);
  }
  SVG_LAUNCH_OK();
  const long long per = n / c, quad = per * per / 512;  // greedy rounds grow with the square of the cluster size
  const int greedy_left = SVG_SEED_GREEDY >= 0 ? SVG_SEED_GREEDY : (int)(quad < c / 2 ? quad : c / 2);
  seed_gram_kernel<<<bh, 1024, 0, st>>>(x, gram_ws, n, d, c, m, seed, first_instance, greedy_left, cent);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
