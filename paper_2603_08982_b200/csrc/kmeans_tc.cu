// k-means assignment on the tensor cores (tcgen05 + TMEM), sm_100a.
//
// Reference step: clustering._sq_dists + argmin (clustering.py:55-62, 113):
//     d2[t,c] = max(|x_t|^2 - 2 x_t.c_c + |c_c|^2, 0),  assign[t] = first argmin_c d2[t,c].
// The x.c^T contraction is ~99.5 % of a Lloyd iteration.  Tokens are bf16 (exact); each fp32
// centroid is split into kPieces = 2 bf16 pieces c = c0 + c1 so that sum_p x.c_p reproduces
// the fp32 product to ~2^-17 relative with fp32 accumulation in TMEM — the pieces simply extend the
// K dimension of one GEMM (one piece when the centres are bf16-exact).  The epilogue (one thread per
// token) turns accumulator columns into distances and keeps the running (min, first index,
// runner-up), so the [n x C] distance matrix never exists in memory.
//
// Persistent kernel, work item = 256 ACTIVE tokens (two M=128 tiles, gathered through the active
// list) x all centroids, N tiles of 128.  Centroid-piece tiles (32 KB at d=128) stream through a
// 3-stage TMA ring; each piece tile is reused by both M tiles.  TMEM: 2 buffers x (2 M tiles x 128
// columns) = 512 columns, so the epilogue of N tile n overlaps the MMAs of N tile n+1.
//   warps 0-7 : epilogue (warp w -> M tile w/4, TMEM lanes 32*(w%4)..)
//   warp  8   : centroid-piece producer (TMA)      warp 9 : TMEM allocator + MMA issuer
//   warp 10   : token-tile producer (cp.async row gather)
#include "tc_common.cuh"

namespace svg {

using namespace tc;

namespace {
constexpr int kPieces = 2;
constexpr int KM = 256;     // tokens per work item (two M=128 tiles)
constexpr int KN = 128;     // centroids per N tile
constexpr int KSTAGES = 3;  // centroid-piece pipeline depth
constexpr int KTHREADS = 352;
constexpr int kMaxHeads = 256;  // instances per launch (larger batches are chunked)

enum {
  KB_AFULL = 0,                    // [2]
  KB_AEMPTY = 2,                   // [2]
  KB_BFULL = 4,                    // [KSTAGES]
  KB_BEMPTY = 4 + KSTAGES,         // [KSTAGES]
  KB_ACCFULL = 4 + 2 * KSTAGES,    // [2]
  KB_ACCEMPTY = 6 + 2 * KSTAGES    // [2]
};

template <int D>
struct KSmem {
  static constexpr int kABytes = KM * D * 2;
  static constexpr int kBBytes = KN * D * 2;
  static constexpr int kA = 0;                       // 2 buffers
  static constexpr int kB = kA + 2 * kABytes;        // KSTAGES stages
  static constexpr int kBars = kB + KSTAGES * kBBytes;
  static constexpr size_t bytes() { return 1024 + kBars + 256; }
};
}  // namespace

// |x|^2 per token (a per-token constant of the arg-min; it only enters own_d2 and the bounds).  One warp
// per row, lanes split the row (8-byte loads at d=128), fixed shuffle tree; 4 rows in flight per warp.
__global__ void __launch_bounds__(256)
    token_norm_kernel(const bf16* __restrict__ x, int d, long long total, float* __restrict__ xn) {
  const int lane = threadIdx.x & 31;
  const long long warp_id = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const long long nwarps = (long long)gridDim.x * (blockDim.x / 32);
  constexpr int R = 4;
  for (long long row0 = warp_id * R; row0 < total; row0 += nwarps * R) {
    float s[R];
    if (d == 128) {
      uint2 u[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long row = row0 + r < total ? row0 + r : total - 1;
        u[r] = __ldg(reinterpret_cast<const uint2*>(x + row * d) + lane);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float f0 = __uint_as_float(u[r].x << 16), f1 = __uint_as_float(u[r].x & 0xffff0000u);
        const float f2 = __uint_as_float(u[r].y << 16), f3 = __uint_as_float(u[r].y & 0xffff0000u);
        float a = 0.f;
        a = fmaf(f0, f0, a); a = fmaf(f1, f1, a); a = fmaf(f2, f2, a); a = fmaf(f3, f3, a);
        s[r] = a;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long row = row0 + r < total ? row0 + r : total - 1;
        float a = 0.f;
        for (int k = lane * 2; k < d; k += 64) {
          const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(x + row * d + k));
          const float f0 = __uint_as_float(u << 16), f1 = __uint_as_float(u & 0xffff0000u);
          a = fmaf(f0, f0, a); a = fmaf(f1, f1, a);
        }
        s[r] = a;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float v = warp_sum(s[r]);
      if (lane == 0 && row0 + r < total) xn[row0 + r] = v;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Exact bound-based skipping (Hamerly's bounds) — same assignments as plain Lloyd, fewer distances.
// Every token carries ub >= dist(x, c[assign]) and lb <= min_{j != assign} dist(x, c[j]); after a
// centroid update lloyd_step_kernel (lloyd_step.cu, phase B2) shifts them by the centre movements
// and compacts the tokens whose bounds overlap into the instance's `active` list.  This kernel
// re-evaluates exactly those tokens and refreshes both bounds.  Iteration 0 (and
// SVGEAR_KMEANS_FULL_EVAL) has every token active.
// ------------------------------------------------------------------------------------------------

// Persistent kernel: grid = #SMs; CTA b handles work items b, b+grid, ... where an item is a
// 256-token tile of a not-yet-converged instance.  Token tiles are double buffered (the next item's
// tile loads while the current one is multiplied), the centroid-piece ring and the two TMEM
// accumulator buffers run straight through item boundaries.
//   warps 0-7 : epilogue      warp 8 : centroid-piece producer      warp 9 : MMA issuer
//   warp 10   : token-tile producer
template <int D>
__global__ void __launch_bounds__(KTHREADS, 1)
    assign_tc_kernel(const __grid_constant__ CUtensorMap pieces_map, const bf16* __restrict__ x,
                     const float* __restrict__ cnorm_pad, const float* __restrict__ xnorm, int bh, int head0, int n,
                     int c, int cpad, int cpad16, int first_iter, int32_t* __restrict__ assign,
                     float* __restrict__ own_d2, float* __restrict__ ub, float* __restrict__ lb,
                     const int32_t* __restrict__ active, const int32_t* __restrict__ nactive,
                     uint8_t* __restrict__ dirty, const int32_t* __restrict__ resid_nz,
                     const int32_t* __restrict__ done) {
  using L = KSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int16_t s_heads[kMaxHeads];
  __shared__ int s_tstart[kMaxHeads + 1];  // first work item of each listed instance
  __shared__ int s_nactive;
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase + L::kA, sB = sbase + L::kB, bars = sbase + L::kBars;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBars + 192);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto bar = [&](int i) -> uint32_t { return bars + 8u * (uint32_t)i; };

  if (tid == 0) {
    int na = 0, items = 0;
    for (int h = 0; h < bh; ++h) {
      const int cnt = done[h] ? 0 : nactive[h];
      if (cnt > 0) {
        s_heads[na] = (int16_t)h;
        s_tstart[na++] = items;
        items += (cnt + KM - 1) / KM;
      }
    }
    s_tstart[na] = items;
    s_nactive = na;
  }
  __syncthreads();
  const int nlisted = s_nactive;
  const int total_items = s_tstart[nlisted];
  if ((int)blockIdx.x >= total_items) return;
  const int my_items = (total_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(KB_AFULL + b), 1);
      mbar_init(bar(KB_AEMPTY + b), 1);
      mbar_init(bar(KB_ACCFULL + b), 1);
      mbar_init(bar(KB_ACCEMPTY + b), 256);
    }
    for (int st = 0; st < KSTAGES; ++st) {
      mbar_init(bar(KB_BFULL + st), 1);
      mbar_init(bar(KB_BEMPTY + st), 1);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(smem_u32(tmem_slot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int NT = (cpad16 + KN - 1) / KN;  // N tiles; the last one may be narrower (multiple of 16)
  // work item -> (instance, 256-token tile of its active list): binary search in the item prefix
  auto locate = [&](int it, int& tile) -> int {
    const int item = (int)blockIdx.x + it * (int)gridDim.x;
    int lo = 0, hi = nlisted - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_tstart[mid] <= item) lo = mid; else hi = mid - 1;
    }
    tile = item - s_tstart[lo];
    return s_heads[lo];
  };

  if (warp == 8) {
    // =========================== centroid-piece producer (TMA, one elected thread) ==============
    // pieces are a plain [instance][piece][cpad][D] bf16 matrix: one 128-row x 64-column box per
    // slab lands in the canonical SWIZZLE_128B layout (the previous 2048 16-byte cp.async per unit
    // cost ~2000 clk of issue time per unit — twice the unit's MMA time)
    if (elect_one()) {
      int u = 0;  // running unit counter across items
      for (int it = 0; it < my_items; ++it) {
        int tile_unused;
        const int h = locate(it, tile_unused);
        const int np = resid_nz[h] ? kPieces : 1;  // pieces that are not identically zero
        const int U = NT * np;                      // pipeline units of this item
        for (int uu = 0; uu < U; ++uu, ++u) {
          const int st = u % KSTAGES;
          if (u >= KSTAGES) mbar_wait(bar(KB_BEMPTY + st), ((u / KSTAGES) - 1) & 1);
          const int nt = uu / np, p = uu % np;
          const uint32_t dst = sB + (uint32_t)st * L::kBBytes;
          const uint32_t fb = bar(KB_BFULL + st);
          mbar_expect_tx(fb, (uint32_t)L::kBBytes);
          const int row = ((head0 + h) * kPieces + p) * cpad + nt * KN;
#pragma unroll
          for (int sl = 0; sl < D / 64; ++sl) tma_box(dst + (uint32_t)(sl * (KN * 128)), &pieces_map, sl * 64, row, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 10) {
    // =========================== token-tile producer (A operand, double buffered) ===============
    constexpr int CPR = D / 8, RPI = 32 / CPR;
    const int sub = lane / CPR, chunk = lane % CPR;
    for (int it = 0; it < my_items; ++it) {
      const int b = it & 1;
      if (it >= 2) mbar_wait(bar(KB_AEMPTY + b), ((it >> 1) + 1) & 1);
      int tile;
      const int h = locate(it, tile);
      const int tok0 = tile * KM, na = nactive[h];
      const bf16* xsrc = x + (size_t)h * n * D;
      const int32_t* alist = active + (size_t)h * n;
      const uint32_t dst = sA + (uint32_t)b * L::kABytes;
#pragma unroll 4
      for (int r0 = 0; r0 < KM; r0 += RPI) {
        const int r = r0 + sub;  // row within the item: M tile r/128, row r%128
        const int row = __ldg(alist + min(tok0 + r, na - 1));
        const int mt = r >> 7, rr = r & 127;
        cp_async16(dst + (uint32_t)(mt * (128 * D * 2) + (chunk >> 3) * (128 * 128)) + swz(rr, chunk & 7),
                   xsrc + (size_t)row * D + chunk * 8);
      }
      cp_async_commit();
      cp_async_wait_all();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(KB_AFULL + b));
    }
  } else if (warp == 9) {
    // =========================== MMA issuer ======================================================
    if (elect_one()) {
      int u = 0, g = 0;  // running unit / N-tile counters
      for (int it = 0; it < my_items; ++it) {
        const int ab = it & 1;
        int tile_unused;
        const int np = resid_nz[locate(it, tile_unused)] ? kPieces : 1;
        mbar_wait(bar(KB_AFULL + ab), (it >> 1) & 1);
        const uint32_t abase = sA + (uint32_t)ab * L::kABytes;
        for (int nt = 0; nt < NT; ++nt, ++g) {
          const int buf = g & 1;
          const int nn = min(KN, cpad16 - nt * KN);
          const uint32_t idesc = make_idesc(128, nn, 0);
          if (g >= 2) mbar_wait(bar(KB_ACCEMPTY + buf), ((g >> 1) - 1) & 1);
          for (int p = 0; p < np; ++p, ++u) {
            const int st = u % KSTAGES;
            mbar_wait(bar(KB_BFULL + st), (u / KSTAGES) & 1);
            tc_fence_after();
            const uint32_t bb = sB + (uint32_t)st * L::kBBytes;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint64_t ad = make_desc(
                    abase + (uint32_t)(m * (128 * D * 2) + (kk >> 2) * (128 * 128) + (kk & 3) * 32), 16, 1024);
                const uint64_t bd = make_desc(bb + (uint32_t)((kk >> 2) * (KN * 128) + (kk & 3) * 32), 16, 1024);
                umma_ss(tmem + (uint32_t)(buf * 256 + m * 128), ad, bd, idesc, (p > 0 || kk > 0) ? 1u : 0u);
              }
            }
            umma_commit(bar(KB_BEMPTY + st));
          }
          umma_commit(bar(KB_ACCFULL + buf));
        }
        umma_commit(bar(KB_AEMPTY + ab));
      }
    }
    __syncwarp();
  } else {
    // =========================== epilogue: distances + running arg-min ===========================
    const int m = warp >> 2;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    int g = 0;
    for (int it = 0; it < my_items; ++it) {
      int tile;
      const int h = locate(it, tile);
      const int na = nactive[h];
      const int ti = tile * KM + m * 128 + (warp & 3) * 32 + lane;  // position in the active list
      const int t = __ldg(active + (size_t)h * n + min(ti, na - 1));
      const float xn = xnorm[(size_t)h * n + t];
      const float* cn = cnorm_pad + (size_t)h * cpad;
      // Two independent (min, first index, runner-up) chains over the even / odd columns halve the
      // serial compare-select dependency; they are merged once per token below.  |x|^2 is a
      // per-token constant of the arg-min, so the loop ranks w = |c|^2 - 2 x.c and the clip at zero
      // is applied once to the winner.  (The reference clips every entry, clustering.py:62; that
      // only matters when two DIFFERENT centroids are both within rounding of the token, and
      // identical centroids still tie exactly here.)
      float best0 = INFINITY, best1 = INFINITY, sec0 = INFINITY, sec1 = INFINITY;
      int bi0 = 0, bi1 = 1;
      auto rank32 = [&](const uint32_t(&a)[32], int cb) {
        // centre norms: 16-byte uniform loads (one LSU instruction per 4 columns; the per-column
        // scalar loads cost 14 % of the kernel)
        const float4* cn4 = reinterpret_cast<const float4*>(cn + cb);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 nv = __ldg(cn4 + j / 4);
          const float w0 = fmaf(-2.0f, __uint_as_float(a[j]), nv.x);
          const float w1 = fmaf(-2.0f, __uint_as_float(a[j + 1]), nv.y);
          const float w2 = fmaf(-2.0f, __uint_as_float(a[j + 2]), nv.z);
          const float w3 = fmaf(-2.0f, __uint_as_float(a[j + 3]), nv.w);
          sec0 = fminf(sec0, fmaxf(w0, best0));  // runner-up distance (lower bound for skipping)
          sec1 = fminf(sec1, fmaxf(w1, best1));
          // strict: ties keep the lowest cluster index (NaN from stale columns never wins)
          if (w0 < best0) { best0 = w0; bi0 = cb + j; }
          if (w1 < best1) { best1 = w1; bi1 = cb + j + 1; }
          sec0 = fminf(sec0, fmaxf(w2, best0));
          sec1 = fminf(sec1, fmaxf(w3, best1));
          if (w2 < best0) { best0 = w2; bi0 = cb + j + 2; }
          if (w3 < best1) { best1 = w3; bi1 = cb + j + 3; }
        }
      };
      for (int nt = 0; nt < NT; ++nt, ++g) {
        const int buf = g & 1;
        mbar_wait(bar(KB_ACCFULL + buf), (g >> 1) & 1);
        tc_fence_after();
        const uint32_t tcol = tmem + lane_base + (uint32_t)(buf * 256 + m * 128);
        const int nn = min(KN, cpad16 - nt * KN);
        const int cb = nt * KN;
        // 32-column chunks, the TMEM load of the next chunk in flight under the ranking of the
        // current one (a narrow last tile leaves stale columns: their norm is +inf)
        uint32_t a0[32], a1[32];
        TMEM_LD32(tcol, a0);
        tc_wait_ld();
        if (nn > 32) TMEM_LD32(tcol + 32, a1);
        rank32(a0, cb);
        if (nn > 32) {
          tc_wait_ld();
          if (nn > 64) TMEM_LD32(tcol + 64, a0);
          rank32(a1, cb + 32);
          if (nn > 64) {
            tc_wait_ld();
            if (nn > 96) TMEM_LD32(tcol + 96, a1);
            rank32(a0, cb + 64);
            if (nn > 96) {
              tc_wait_ld();
              rank32(a1, cb + 96);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(bar(KB_ACCEMPTY + buf));
      }
      // merge the chains: lower value wins, equal values keep the lower index
      const bool odd = best1 < best0 || (best1 == best0 && bi1 < bi0);
      const float best = odd ? best1 : best0;
      const int bi = odd ? bi1 : bi0;
      const float second = fminf(fminf(sec0, sec1), odd ? best0 : best1);
      if (ti < na) {
        const size_t gi = (size_t)h * n + t;
        const float d2 = fmaxf(xn + best, 0.f);
        if (!first_iter) {
          const int prev = assign[gi];
          if (prev != bi) {  // membership of both clusters changed: their means must be recomputed
            dirty[(size_t)h * c + prev] = 1;
            dirty[(size_t)h * c + bi] = 1;
          }
        }
        assign[gi] = bi;
        own_d2[gi] = d2;
        ub[gi] = sqrtf(d2);
        lb[gi] = sqrtf(fmaxf(xn + second, 0.f));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int launch_token_norms(int bh, int n, int d, const bf16* x, float* xnorm, cudaStream_t st) {
  const long long total = (long long)bh * n;
  token_norm_kernel<<<(unsigned)((total + 31) / 32 < 148 * 16 ? (total + 31) / 32 : 148 * 16), 256, 0, st>>>(x, d, total, xnorm);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

int launch_kmeans_assign_tc(int bh, int n, int d, int c, int iter, const bf16* x, KmeansScratch& sc,
                            int32_t* assign, cudaStream_t st) {
  const int cpad = ceil_div(c, KN) * KN;     // row stride of the piece arrays / norm array
  const int cpad16 = ceil_div(c, 16) * 16;   // columns actually multiplied
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    SVG_CUDA_OK(cudaGetDevice(&dev));
    SVG_CUDA_OK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  CUtensorMap pieces_map;
  if (!encode_rows_map(&pieces_map, sc.pieces, (uint64_t)bh * kPieces * cpad, d, KN)) return SVGEAR_ECUDA;
  for (int h0 = 0; h0 < bh; h0 += kMaxHeads) {
    const int nb = bh - h0 < kMaxHeads ? bh - h0 : kMaxHeads;
    const int items = nb * ceil_div(n, KM);  // upper bound; the kernel reads the real counts
    // SVGEAR_ASSIGN_GRID / SVGEAR_ASSIGN_GRID0: cap of the persistent grid after / in the first iteration
    // (experiment knob: a grid below the SM count lets the other side's kernels co-run)
    static const int cap_late = [] { const char* e = getenv("SVGEAR_ASSIGN_GRID"); return e ? atoi(e) : 0; }();
    static const int cap_first = [] { const char* e = getenv("SVGEAR_ASSIGN_GRID0"); return e ? atoi(e) : 0; }();
    const int cap = iter == 0 ? cap_first : cap_late;
    int grid = items < num_sms ? items : num_sms;
    if (cap > 0 && grid > cap) grid = cap;
    const bf16* xs = x + (size_t)h0 * n * d;
    const float* cs = sc.cnorm_pad + (size_t)h0 * cpad;
    const float* xns = sc.xnorm + (size_t)h0 * n;
    int32_t* as = assign + (size_t)h0 * n;
    float* os = sc.own_d2 + (size_t)h0 * n;
    float* us = sc.ub + (size_t)h0 * n;
    float* ls = sc.lb + (size_t)h0 * n;
    const int32_t* al = sc.active + (size_t)h0 * n;
    uint8_t* dt = sc.dirty + (size_t)h0 * c;
    if (d == 128) {
      const size_t smem = KSmem<128>::bytes();
      SVG_CUDA_OK(cudaFuncSetAttribute(assign_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      assign_tc_kernel<128><<<grid, KTHREADS, smem, st>>>(pieces_map, xs, cs, xns, nb, h0, n, c, cpad, cpad16, iter == 0, as, os,
                                                          us, ls, al, sc.nactive + h0, dt, sc.resid_nz + h0, sc.done + h0);
    } else {
      const size_t smem = KSmem<64>::bytes();
      SVG_CUDA_OK(cudaFuncSetAttribute(assign_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      assign_tc_kernel<64><<<grid, KTHREADS, smem, st>>>(pieces_map, xs, cs, xns, nb, h0, n, c, cpad, cpad16, iter == 0, as, os,
                                                         us, ls, al, sc.nactive + h0, dt, sc.resid_nz + h0, sc.done + h0);
    }
    SVG_LAUNCH_OK();
  }
  return SVGEAR_OK;
}

}  // namespace svg
