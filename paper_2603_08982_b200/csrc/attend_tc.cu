// Fused block-sparse FlashAttention for sm_100a (subsystem 3): tcgen05.mma with TMEM accumulators.
//
// Semantics: attention.exact_block_pass + compensation_pass of the reference
// (/root/reference/pkg/src/routedattn/attention.py:57-157) in ONE online softmax per query row:
//   * "exact" key tiles: the keys of every selected key cluster of the row's query cluster,
//     gathered (cluster ranges are contiguous in the permuted K/V) into dense 64-key tiles;
//   * "centroid" key tiles: all C_k centroids k̄_j with value v̄_j and logit bias ln|k_j|; columns
//     whose block is selected are masked to -inf (attention.py:130,146).
// The output row is normalised once and scattered back to original token order.
//
// Kernel structure: see the comment above attend_tc_kernel.
#include "tc_common.cuh"

namespace svg {

using namespace tc;

namespace {

constexpr int BM = 256;      // query rows per CTA: two M=128 halves that share every K/V tile
constexpr int BN = 64;       // keys per softmax chunk (one S buffer); a K/V tile holds G chunks
constexpr int threads_for(int halves, int tpr = 1) { return (4 * halves * tpr + 2 + halves) * 32; }  // softmax + 2 producers + issuers
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef SVG_POLY2
#define SVG_POLY2 0  // two-threads-per-row path: column pairs (of 4) whose exponential runs on the FMA pipe (0: 5.23, 1: 5.27, 2: 5.65 ms per 8 heads)
#endif
#ifndef SVG_ABL
#define SVG_ABL 0  // ablation bits for tools/attend_ablate.sh (timing only, results are garbage): 1 no softmax
#endif             // arithmetic, 2 never redo, 4 no QK^T MMAs, 8 no P.V MMAs, 16 no K/V loads, 32 one box per slab

template <int D, int NS, int HALVES, int G, int TPR = 1>
struct Smem {
  static constexpr int kQBytes = HALVES * 128 * D * 2;
  static constexpr int kTileBytes = G * BN * D * 2;
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;             // NS stages
  static constexpr int kV = kK + NS * kTileBytes;     // NS stages
  static constexpr int kBars = kV + NS * kTileBytes;  // mbarriers + tmem ptr + counters
  static constexpr int kXchg = kBars + 512;           // TPR = 2: [row][2] floats exchanged between the two threads of a row
  static constexpr int kLists = kXchg + (TPR == 2 ? HALVES * 128 * 2 * 4 : 0);
  static size_t bytes(int ckpad) { return 1024 + kLists + (size_t)(ckpad + 64) * 12; }
};

// mbarrier indices
template <int NS>
struct Bars {
  static constexpr int QFULL = 0;
  static constexpr int KFULL = 1;              // [NS]
  static constexpr int KEMPTY = KFULL + NS;    // [NS]
  static constexpr int VFULL = KEMPTY + NS;    // [NS]
  static constexpr int VEMPTY = VFULL + NS;    // [NS]
  static constexpr int SFULL = VEMPTY + NS;    // [half][buffer]
  static constexpr int PFULL = SFULL + 4;      // [half][buffer]
  static constexpr int ODONE = PFULL + 4;      // [half]  one phase per tile (O rescale inside the loop)
  static constexpr int OFINAL = ODONE + 2;     // [half]  single phase: every P.V of the CTA has landed
  static constexpr int COUNT = OFINAL + 2;
};

// Tensor maps of one launch (passed as a __grid_constant__ kernel parameter).  K and V (permuted,
// cluster-contiguous) are gathered as CONTIGUOUS ROW RUNS: a run is split into power-of-two row
// boxes, box height 2^i rows x 64 columns, SWIZZLE_128B — the hardware writes the canonical UMMA
// layout, a handful of bulk-tensor instructions replace 1024 16-byte cp.async gathers per tile.
struct TmaSet {
  CUtensorMap k[7];   // [bh*n_k][D] bf16, box {64 cols, 1<<i rows}
  CUtensorMap v[7];
  CUtensorMap kbar;   // [bh*ckpad][D] bf16, box {64, 64}
  CUtensorMap vbar;
  CUtensorMap q;      // [bh*n_q][D] bf16, box {64, 64}
};

}  // namespace

// One CTA = up to 256 consecutive rows of one query cluster (tile list built by build_tiles_kernel),
// one CTA per SM (512 TMEM columns).  Both 128-row halves see the same selected key clusters, so a
// K/V tile is gathered into shared memory once and multiplied twice — half the L2->smem traffic of
// one CTA per 128 rows, which is what bound the previous version.
//   warps 0-3 : softmax + epilogue of half 0 (thread == query row, TMEM lane == row)
//   warps 4-7 : same for half 1 (idle when the tile has <= 128 rows)
//   warp  8   : K producer — cp.async gathers into the canonical SWIZZLE_128B layout, NS-stage ring,
//               LAG tiles in flight
//   warp  9   : Q tile, then V producer
//   warps 10,11 : one elected tcgen05.mma issuer per half (warp 10 also allocates TMEM)
// TMEM columns: S[half][buf] at half*128 + buf*64 (64 fp32 columns; P (bf16) overwrites the first 32
// and is the A operand of P.V straight from TMEM), O[half] at 256 + half*D.  The softmax always works
// on 64-key CHUNKS, one per S buffer.  The running maximum is only raised when it grows by more than
// 2^8 (lazy rescale).
//   G = 1: a K/V tile is one chunk; QK^T (N = 64) of chunk u+1 runs under the softmax of chunk u (S
//          double buffered per half).  Each N = 64 MMA re-reads its 4 KB slice of Q for 2 KB of K:
//          192 B/clk of shared-memory operand traffic against 128 available, QK^T runs at 2/3 rate.
//   G = 2: a K/V tile is two chunks; ONE N = 128 QK^T per tile fills both S buffers (128 B/clk), issued
//          after the P.V of the previous tile's second chunk; the softmax of a half then alternates
//          with the other half's MMAs on the tensor pipe (the two halves ping-pong).
//   TPR = 2 (two threads per query row): 16 softmax warps, four per scheduler; the two warps of a row
//          group (same TMEM lane quarter, hence same scheduler) take 32 columns of a chunk each and agree
//          on the rare exact path with one named-barrier OR per chunk (see the softmax section).
template <int D, int NS, int HALVES, int G, int TPR>
__global__ void __launch_bounds__(threads_for(HALVES, TPR), 3 - HALVES)
    attend_tc_kernel(const __grid_constant__ TmaSet tm, int oob_row,
                     const float* __restrict__ lnw, const int32_t* __restrict__ q_perm,
                     const int32_t* __restrict__ k_sizes, const int32_t* __restrict__ k_offsets,
                     const uint8_t* __restrict__ mask, const int32_t* __restrict__ tile_list,
                     const int32_t* __restrict__ tile_count, int max_tiles, int n_q, int n_k, int c_q,
                     int c_k, int ckpad, float scale_log2e, bf16* __restrict__ out,
                     float* __restrict__ lse) {
  using L = Smem<D, NS, HALVES, G, TPR>;
  static_assert(TPR == 1 || HALVES == 2, "two threads per row: two halves");
  constexpr int TK = G * BN;  // keys per K/V tile
  constexpr int halves = HALVES;
  constexpr int kSoftWarps = 4 * HALVES * TPR, kWarpK = kSoftWarps, kWarpV = kSoftWarps + 1, kWarpMma = kSoftWarps + 2;
  constexpr int kTmemCols = 256 * HALVES, kOBase = 128 * HALVES;
  using B = Bars<NS>;
  const int h = blockIdx.y;
  // two-half tiles fill the tile list from the front, tiles of <= 128 rows from the back (build_tiles_kernel)
  if ((int)blockIdx.x >= tile_count[(HALVES == 2 ? 0 : gridDim.y) + h]) return;
  const int slot = HALVES == 2 ? (int)blockIdx.x : max_tiles - 1 - (int)blockIdx.x;
  const int32_t* te = tile_list + ((size_t)h * max_tiles + slot) * 4;
  const int qcl = te[0], row0 = te[1], nrows = te[2];

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase + L::kQ, sK = sbase + L::kK, sV = sbase + L::kV;
  const uint32_t bars = sbase + L::kBars;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBars + 384);
  int32_t* s_total = reinterpret_cast<int32_t*>(smem + L::kBars + 392);  // [0]=selected keys
  int32_t* s_pre = reinterpret_cast<int32_t*>(smem + L::kLists);          // [nsel+1] key prefix
  int32_t* s_row = s_pre + (ckpad + 64);                                    // [nsel] first row
  float* s_bias = reinterpret_cast<float*>(s_row + (ckpad + 64));          // [ckpad] log2 domain

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto bar = [&](int i) -> uint32_t { return bars + 8u * (uint32_t)i; };

  // ---- prologue: barriers, TMEM, per-cluster selection lists ------------------------------------
  if (tid == 0) {
    mbar_init(bar(B::QFULL), 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(bar(B::KFULL + s), 1);
      mbar_init(bar(B::KEMPTY + s), halves);  // one commit per MMA issuer (half)
      mbar_init(bar(B::VFULL + s), 1);
      mbar_init(bar(B::VEMPTY + s), halves);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(bar(B::SFULL + s), 1);
      mbar_init(bar(B::PFULL + s), 4 * TPR);  // one elected lane per softmax warp
    }
    mbar_init(bar(B::ODONE), 1);
    mbar_init(bar(B::ODONE + 1), 1);
    mbar_init(bar(B::OFINAL), 1);
    mbar_init(bar(B::OFINAL + 1), 1);
    fence_barrier_init();
  }
  if (warp == kWarpMma) tmem_alloc(smem_u32(tmem_slot), kTmemCols);
  const uint8_t* mrow = mask + ((size_t)h * c_q + qcl) * c_k;
  if (warp == 0) {
    // compact the selected key clusters of this query cluster: (first row, key-count prefix)
    int nsel = 0, total = 0;
    for (int j0 = 0; j0 < c_k; j0 += 32) {
      const int j = j0 + lane;
      const bool sel = j < c_k && mrow[j] != 0;
      const int sz = sel ? k_sizes[(size_t)h * c_k + j] : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      int inc = sz;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (sel) {
        const int pos = nsel + __popc(bal & ((1u << lane) - 1u));
        s_pre[pos] = total + inc - sz;
        s_row[pos] = k_offsets[(size_t)h * c_k + j];
      }
      nsel += __popc(bal);
      total += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      s_pre[nsel] = total;
      s_total[0] = total;
      s_total[1] = nsel;
    }
  } else if (warp >= 1 && warp < kSoftWarps) {
    for (int j = tid - 32; j < ckpad + (G - 1) * BN; j += (kSoftWarps - 1) * 32)
      s_bias[j] = (j < c_k && mrow[j] == 0) ? lnw[(size_t)h * c_k + j] * kLog2e : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total_keys = s_total[0];
  const int n_exact = (total_keys + TK - 1) / TK;  // K/V tiles of selected keys
  const int n_cent = (ckpad + TK - 1) / TK;          // K/V tiles of centroids
  const int T = n_exact + n_cent;

  if (warp == kWarpK || warp == kWarpV) {
    // =========================== producers: K (warp 8) / Q then V (warp 9), one elected thread ===
    const bool is_k = warp == kWarpK;
    if (elect_one()) {
      const CUtensorMap* maps = is_k ? tm.k : tm.v;
      const CUtensorMap* cmap = is_k ? &tm.kbar : &tm.vbar;
      const uint32_t sbuf = is_k ? sK : sV;
      const int b_full = is_k ? B::KFULL : B::VFULL, b_empty = is_k ? B::KEMPTY : B::VEMPTY;
      constexpr int SLABS = D / 64;  // 64-column (128-byte) slabs of a row
      if (!is_k) {
        // Q tile: rows row0.. of the permuted Q (rows past the tile belong to the next cluster or are
        // zero-filled past the end of the array; they are computed but never stored)
        mbar_expect_tx(bar(B::QFULL), (uint32_t)(halves * 128 * D * 2));
        for (int hf = 0; hf < halves; ++hf)
          for (int sl = 0; sl < SLABS; ++sl)
            for (int rb = 0; rb < 2; ++rb)
              tma_box(sQ + (uint32_t)(hf * (128 * D * 2) + sl * (128 * 128) + rb * (64 * 128)), &tm.q, sl * 64,
                      h * n_q + row0 + hf * 128 + rb * 64, bar(B::QFULL));
      }
      int cur = 0;  // cursor into the selection list
      const int rowbase = h * n_k;
      for (int t = 0; t < T; ++t) {
        const int st = t % NS;
        if (t >= NS) mbar_wait(bar(b_empty + st), ((t / NS) - 1) & 1);
        const uint32_t dst = sbuf + (uint32_t)st * L::kTileBytes;
        const uint32_t fb = bar(b_full + st);
        if (SVG_ABL & 16) {  // no K/V traffic at all
          mbar_arrive(fb);
          continue;
        }
        mbar_expect_tx(fb, (uint32_t)L::kTileBytes);
        if (SVG_ABL & 32) {  // same bytes, one 64-row box per slab
#pragma unroll
          for (int sl = 0; sl < SLABS; ++sl)
            for (int g = 0; g < G; ++g)
              tma_box(dst + (uint32_t)(g * (BN * 128) + sl * (TK * 128)), maps + 6, sl * 64, rowbase + (int)(((long long)(t * G + g) * 64 + blockIdx.x * 192) % (n_k - 64)), fb);
          continue;
        }
        if (t < n_exact) {
          int u = t * TK;
          const int uend = min(u + TK, total_keys);
          while (u < uend) {
            while (s_pre[cur + 1] <= u) ++cur;
            int len = min(s_pre[cur + 1], uend) - u;
            int src = rowbase + s_row[cur] + (u - s_pre[cur]);
            while (len > 0) {  // largest power-of-two box first
              const int b = min(31 - __clz(len), 6), nb = 1 << b;
              const uint32_t d0 = dst + (uint32_t)((u - t * TK) * 128);
#pragma unroll
              for (int sl = 0; sl < SLABS; ++sl) tma_box(d0 + (uint32_t)(sl * (TK * 128)), maps + b, sl * 64, src, fb);
              u += nb;
              src += nb;
              len -= nb;
            }
          }
          // ragged last tile: the remaining slots are filled with zeros (out-of-bounds boxes); their
          // logits are masked to -inf, and 0 * finite keeps the P.V accumulation clean
          int slot = uend - t * TK, pad = TK - slot;
          while (pad > 0) {
            const int b = min(31 - __clz(pad), 6), nb = 1 << b;
#pragma unroll
            for (int sl = 0; sl < SLABS; ++sl)
              tma_box(dst + (uint32_t)(slot * 128 + sl * (TK * 128)), maps + b, sl * 64, oob_row, fb);
            slot += nb;
            pad -= nb;
          }
        } else {
          // (with G = 2 the last centroid tile may run 64 rows into the next instance's centroids, or
          // past the array: zero filled; those columns carry a -inf bias)
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int sl = 0; sl < SLABS; ++sl)
              tma_box(dst + (uint32_t)(g * (BN * 128) + sl * (TK * 128)), cmap, sl * 64,
                      h * ckpad + (t - n_exact) * TK + g * BN, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp >= kWarpMma) {
    // =========================== MMA issuers: warp 10 -> half 0, warp 11 -> half 1 =============
    // One elected thread per half runs its own QK^T / P.V sequence, so a barrier round trip of one
    // half never stalls the other half's MMAs; K/V stages are released by both (count = halves).
    // With G = 2 and two halves ONE thread issues for both halves in a fixed order - P.V_A(t), QK_A(t+1),
    // P.V_B(t), QK_B(t+1) - so that the halves alternate on the tensor pipe (left to themselves they fall
    // into lockstep: both softmax at once, then both sets of MMAs).
    constexpr bool kOrdered = (G == 2 && HALVES == 2);
    const int hf0 = warp - kWarpMma;
    if (hf0 < (kOrdered ? 1 : halves) && elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(128, TK, 0);
      constexpr uint32_t idesc_pv = make_idesc(128, D, 1);
      auto issue_qk = [&](int hf, int t) {
        const uint32_t qb = sQ + (uint32_t)(hf * (128 * D * 2));
        const uint32_t tSb = tmem + (uint32_t)(hf * 128);
        const int st = t % NS;
        mbar_wait(bar(B::KFULL + st), (t / NS) & 1);
        tc_fence_after();
        const uint32_t kb = sK + (uint32_t)st * L::kTileBytes;
        const uint32_t tS = tSb + (uint32_t)(G == 1 ? (t & 1) * 64 : 0);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = make_desc(qb + (uint32_t)((kk >> 2) * (128 * 128) + (kk & 3) * 32), 16, 1024);
          const uint64_t bd = make_desc(kb + (uint32_t)((kk >> 2) * (TK * 128) + (kk & 3) * 32), 16, 1024);
          if (!(SVG_ABL & 4)) umma_ss(tS, ad, bd, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(bar(B::SFULL + hf * 2 + (G == 1 ? (t & 1) : 0)));
        umma_commit(bar(B::KEMPTY + st));
      };
      auto issue_pv = [&](int hf, int t) {  // the P.V of every chunk of K/V tile t
        const uint32_t tSb = tmem + (uint32_t)(hf * 128);
        const uint32_t tO = tmem + (uint32_t)(kOBase + hf * D);
        const int st = t % NS;
        mbar_wait(bar(B::VFULL + st), (t / NS) & 1);
        const uint32_t vb = sV + (uint32_t)st * L::kTileBytes;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int u = t * G + g;  // chunk
          mbar_wait(bar(B::PFULL + hf * 2 + (u & 1)), (u >> 1) & 1);
          tc_fence_after();
          const uint32_t tP = tSb + (uint32_t)((u & 1) * 64);
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            // V tile [TK keys x D] is the MN-major B operand: 16 keys per MMA = 2048 B along K,
            // LBO = stride between the 64-column slabs, SBO = stride between 8-key groups
            const uint64_t bd = make_desc(vb + (uint32_t)((g * (BN / 16) + kk) * 2048), TK * 128, 1024);
            if (!(SVG_ABL & 8)) umma_ts(tO, tP + (uint32_t)(kk * 8), bd, idesc_pv, (u > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(bar(B::ODONE + hf));
        }
        umma_commit(bar(B::VEMPTY + st));
      };
      mbar_wait(bar(B::QFULL), 0);
      if (kOrdered) {
        issue_qk(0, 0);
        issue_qk(1, 0);
        for (int t = 0; t < T; ++t) {
          issue_pv(0, t);
          if (t + 1 < T) issue_qk(0, t + 1);
          issue_pv(1, t);
          if (t + 1 < T) issue_qk(1, t + 1);
        }
        umma_commit(bar(B::OFINAL));
        umma_commit(bar(B::OFINAL + 1));
      } else {
        const int hf = hf0;
        issue_qk(hf, 0);
        for (int t = 0; t < T; ++t) {
          if (G == 1 && t + 1 < T) issue_qk(hf, t + 1);
          issue_pv(hf, t);
          // the N = 128 QK^T overwrites both S buffers: it follows the P.V of this tile's second chunk
          // (tensor-pipe order), and the softmax warps have read all of S(t) before they hand over P
          if (G == 2 && t + 1 < T) issue_qk(hf, t + 1);
        }
        umma_commit(bar(B::OFINAL + hf));
      }
    }
    __syncwarp();
  } else if (TPR == 2) {
    // =========================== softmax + epilogue, two threads per row ========================
    // Warp w: lane quarter w & 3 (rows), half (w >> 2) >> 1, column half ch = (w >> 2) & 1: the thread
    // owns columns 32 ch .. 32 ch + 31 of every chunk of its row.  Its 32 logits stay in registers, so
    // the exact path re-uses them (no TMEM re-read), and P is only stored after the pair has met at the
    // named barrier - by then both have loaded their S columns, which P overwrites.
    const int grp = warp >> 2, hf = grp >> 1, ch = grp & 1, quad = warp & 3;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tSb = tmem + lane_base + (uint32_t)(hf * 128);
    const uint32_t tO = tmem + lane_base + (uint32_t)(kOBase + hf * D + ch * (D / 2));
    const int b_sfull = B::SFULL + hf * 2, b_pfull = B::PFULL + hf * 2, b_odone = B::ODONE + hf;
    const int pair_bar = 1 + hf * 4 + quad;  // named barrier of the two warps of this row group
    const int row = hf * 128 + quad * 32 + lane;
    float* xch = reinterpret_cast<float*>(smem + L::kXchg) + row * 2;
    float m = -INFINITY, l = 0.f;
    uint32_t sa[32], pk[16];
    const int U = T * G, u_exact = n_exact * G;
    for (int t = 0; t < U; ++t) {
      const int st = t & 1;
      const int last_valid = total_keys - t * BN;
      const int kind = t >= u_exact ? 2 : (last_valid >= BN ? 0 : 1);
      const float* bias = s_bias + (kind == 2 ? (t - u_exact) * BN : 0);
      if (G == 1 || st == 0) {  // G = 2: one QK^T fills both S buffers of the half
        mbar_wait(bar(b_sfull + (G == 1 ? st : 0)), (t >> 1) & 1);
        tc_fence_after();
      }
      TMEM_LD32(tSb + (uint32_t)(st * 64 + ch * 32), sa);
      const float mu = (m == -INFINITY) ? 0.f : m;
      float sum = 0.f, xk = -INFINITY;
      tc_wait_ld();
      if (SVG_ABL & 1) {
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = sa[j] ^ sa[j + 16];
      } else if (kind == 0) {
        const uint64_t sc2 = pack2(scale_log2e, scale_log2e), nm2 = pack2(-mu, -mu);
        uint64_t acc01 = pack2(0.f, 0.f), acc23 = pack2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          float p[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t xx = ffma2(pack2(__uint_as_float(sa[j + 2 * q]), __uint_as_float(sa[j + 2 * q + 1])), sc2, nm2);
            if (q >= 4 - SVG_POLY2) {
              exp2_poly2(xx, p[2 * q], p[2 * q + 1]);
            } else {
              float a0, a1;
              unpack2(xx, a0, a1);
              p[2 * q] = ex2(a0);
              p[2 * q + 1] = ex2(a1);
            }
          }
          acc01 = fadd2(acc01, pack2(p[0], p[1]));
          acc23 = fadd2(acc23, pack2(p[2], p[3]));
          acc01 = fadd2(acc01, pack2(p[4], p[5]));
          acc23 = fadd2(acc23, pack2(p[6], p[7]));
#pragma unroll
          for (int q = 0; q < 4; ++q) pk[j / 2 + q] = pack_bf16x2(p[2 * q], p[2 * q + 1]);
        }
        float s0, s1, s2, s3;
        unpack2(acc01, s0, s1);
        unpack2(acc23, s2, s3);
        sum = (s0 + s1) + (s2 + s3);
      } else {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int c = ch * 32 + j;
          float b0, b1;
          if (kind == 2) {
            b0 = bias[c];
            b1 = bias[c + 1];
          } else {
            b0 = c < last_valid ? 0.f : -INFINITY;
            b1 = c + 1 < last_valid ? 0.f : -INFINITY;
          }
          const float v0 = fmaf(__uint_as_float(sa[j]), scale_log2e, b0);
          const float v1 = fmaf(__uint_as_float(sa[j + 1]), scale_log2e, b1);
          xk = fmaxf(xk, fmaxf(v0, v1));
          const float p0 = ex2(v0 - mu), p1 = ex2(v1 - mu);
          sum += p0 + p1;
          pk[j / 2] = pack_bf16x2(p0, p1);
        }
      }
      // same lazy maximum as the one-thread-per-row path; a full chunk triggers on its own 32 columns
      // (sum <= 2^13 bounds every logit by m + 13).  The OR over the pair also orders the pair's TMEM
      // loads before the P stores below.
      const bool maybe = kind == 0 ? !(sum <= 8192.f) || m == -INFINITY
                                   : (xk > m + kRescaleThreshold || (m == -INFINITY && xk > -INFINITY));
      uint32_t redo_u;
      asm volatile(
          "{\n\t"
          ".reg .pred p, q;\n\t"
          "setp.ne.b32 q, %1, 0;\n\t"
          "barrier.cta.red.or.pred p, %2, 64, q;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t"
          "}"
          : "=r"(redo_u)
          : "r"((uint32_t)maybe), "r"(pair_bar)
          : "memory");
      if (SVG_ABL & 2) redo_u = 0;
      float alpha = 1.f;
      if (redo_u) {
        // exact path for the row group: maximum of the chunk over both column halves, raise m where
        // needed, exponentials again from the logits still in registers
        float mt = xk;
        if (kind == 0) {
          mt = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j) mt = fmaxf(mt, __uint_as_float(sa[j]));
          mt *= scale_log2e;
        }
        xch[ch] = mt;
        asm volatile("barrier.cta.sync %0, 64;" ::"r"(pair_bar) : "memory");
        mt = fmaxf(mt, xch[ch ^ 1]);
        asm volatile("barrier.cta.sync %0, 64;" ::"r"(pair_bar) : "memory");  // slot free for the next exchange
        const bool bump = mt > m + kRescaleThreshold || (m == -INFINITY && mt > -INFINITY);
        if (bump) {
          alpha = ex2(m - mt);  // m = -inf -> 0
          m = mt;
        }
        const float mu2 = (m == -INFINITY) ? 0.f : m;
        sum = 0.f;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int c = ch * 32 + j;
          float v0 = __uint_as_float(sa[j]) * scale_log2e, v1 = __uint_as_float(sa[j + 1]) * scale_log2e;
          if (kind == 2) {
            v0 += bias[c];
            v1 += bias[c + 1];
          } else if (kind == 1) {
            if (c >= last_valid) v0 = -INFINITY;
            if (c + 1 >= last_valid) v1 = -INFINITY;
          }
          const float p0 = ex2(v0 - mu2), p1 = ex2(v1 - mu2);
          sum += p0 + p1;
          pk[j / 2] = pack_bf16x2(p0, p1);
        }
      }
      l = l * alpha + sum;
      TMEM_ST16(tSb + (uint32_t)(st * 64 + ch * 16), pk);  // this thread's 32 keys of P (bf16 pairs)
      // (loading the logits of chunk t+1 here, under the store and the hand-off, was measured slower:
      // 5.91 vs 5.29 ms per 8 heads)
      if (redo_u && t > 0) {
        // rescale this thread's half of the O columns; P.V of chunk t-1 must have landed first
        mbar_wait(bar(b_odone), (t - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D / 2; c += 32) {
          TMEM_LD32(tO + c, sa);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sa[j] = __float_as_uint(__uint_as_float(sa[j]) * alpha);
          TMEM_ST32(tO + c, sa);
        }
      }
      tc_wait_st();
      tc_fence_before();
      if (lane == 0) mbar_arrive(bar(b_pfull + st));
    }
    // ---- epilogue: row sum of the pair, then each thread normalises and scatters D/2 columns ------
    xch[ch] = l;
    asm volatile("barrier.cta.sync %0, 64;" ::"r"(pair_bar) : "memory");
    l += xch[ch ^ 1];
    mbar_wait(bar(B::OFINAL + hf), 0);
    tc_fence_after();
    const bool live = row < nrows;
    const int prow = min(row0 + row, n_q - 1);
    const int dst = q_perm ? q_perm[(size_t)h * n_q + prow] : prow;
    const float inv = 1.f / l;
    uint4* orow = reinterpret_cast<uint4*>(out + ((size_t)h * n_q + dst) * D + ch * (D / 2));
#pragma unroll
    for (int c = 0; c < D / 2; c += 32) {
      TMEM_LD32(tO + c, sa);
      tc_wait_ld();
      if (live) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(sa[8 * j]) * inv, __uint_as_float(sa[8 * j + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(sa[8 * j + 2]) * inv, __uint_as_float(sa[8 * j + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(sa[8 * j + 4]) * inv, __uint_as_float(sa[8 * j + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(sa[8 * j + 6]) * inv, __uint_as_float(sa[8 * j + 7]) * inv);
          orow[c / 8 + j] = w;
        }
      }
    }
    if (lse && live && ch == 0) lse[(size_t)h * n_q + dst] = (m + log2f(l)) * kLn2;
    tc_fence_before();
  } else if ((warp >> 2) < halves) {
    // =========================== softmax + epilogue (warps 0-7, thread == row) ==================
    const int hf = warp >> 2;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tSb = tmem + lane_base + (uint32_t)(hf * 128);
    const uint32_t tO = tmem + lane_base + (uint32_t)(kOBase + hf * D);
    const int b_sfull = B::SFULL + hf * 2, b_pfull = B::PFULL + hf * 2, b_odone = B::ODONE + hf;
    float m = -INFINITY, l = 0.f;
    // The S tile is consumed as two 32-column blocks; the TMEM load of the next block is always in
    // flight under the arithmetic of the current one (TMEM reads run at 64 B/clk/SM, as long as the
    // MMAs of the tile).  Exponentials are taken SPECULATIVELY against the running maximum m; the
    // block maxima are collected on the side and, only if some row of the warp has to raise m
    // (tile max > m + 2^8, rare after the first tiles), the tile is redone from TMEM the exact way.
    uint32_t sa[32], sb[32], pk[32];
    // chunk t (64 keys) lives in S buffer t & 1.  With G = 1 every chunk has its own QK^T and SFULL
    // phase; with G = 2 one QK^T fills both buffers and only even chunks wait (one barrier per half).
    const int U = T * G, u_exact = n_exact * G;  // chunks in all / chunks of selected keys (incl. padding)
    auto sfull_bar = [&](int t) -> uint32_t { return bar(b_sfull + (G == 1 ? (t & 1) : 0)); };
    mbar_wait(bar(b_sfull), 0);
    tc_fence_after();
    TMEM_LD32(tSb, sa);
    for (int t = 0; t < U; ++t) {
      const int st = t & 1;
      const uint32_t tS = tSb + (uint32_t)(st * 64);
      // chunk kind: 0 = 64 selected keys (raw logits), 1 = ragged or empty tail of the selected keys,
      // 2 = centroids
      const int last_valid = total_keys - t * BN;  // valid columns of an exact chunk (may be <= 0)
      const int kind = t >= u_exact ? 2 : (last_valid >= BN ? 0 : 1);
      const float* bias = s_bias + (kind == 2 ? (t - u_exact) * BN : 0);
      const float mu = (m == -INFINITY) ? 0.f : m;
      float sum0 = 0.f, sum1 = 0.f, sum2 = 0.f, sum3 = 0.f;
      float x2 = -INFINITY, x3 = -INFINITY;  // block maxima of the biased tiles (log2 domain)
      tc_wait_ld();                 // sa = columns 0-31 of tile t
      TMEM_LD32(tS + 32, sb);       // columns 32-63 load under the arithmetic on sa
      auto block = [&](uint32_t(&v)[32], int col0, int pk0) {
        if (kind == 0) {
          // three of four column pairs take their exponential on the MUFU, the fourth on the FMA pipe
          // (packed polynomial): the mix that minimises the block time with two softmax warps per SM
          // sub-partition (tools/micro/softmax_block.cu; the MUFU alone, 16/clk/SM, would need as long
          // as the tile's MMAs)
          const uint64_t sc2 = pack2(scale_log2e, scale_log2e), nm2 = pack2(-mu, -mu);
          uint64_t acc01 = pack2(0.f, 0.f), acc23 = pack2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            float vv[8], p[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) vv[e] = __uint_as_float(v[j + e]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint64_t xx = ffma2(pack2(vv[2 * q], vv[2 * q + 1]), sc2, nm2);
              if (q == 3) {
                exp2_poly2(xx, p[6], p[7]);
              } else {
                float a0, a1;
                unpack2(xx, a0, a1);
                p[2 * q] = ex2(a0);
                p[2 * q + 1] = ex2(a1);
              }
            }
            acc01 = fadd2(acc01, pack2(p[0], p[1]));
            acc23 = fadd2(acc23, pack2(p[2], p[3]));
            acc01 = fadd2(acc01, pack2(p[4], p[5]));
            acc23 = fadd2(acc23, pack2(p[6], p[7]));
#pragma unroll
            for (int q = 0; q < 4; ++q) pk[pk0 + j / 2 + q] = pack_bf16x2(p[2 * q], p[2 * q + 1]);
          }
          float s0, s1, s2, s3;
          unpack2(acc01, s0, s1);
          unpack2(acc23, s2, s3);
          sum0 += s0 + s1;
          sum1 += s2 + s3;
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float b0, b1;
            if (kind == 2) {
              b0 = bias[col0 + j];
              b1 = bias[col0 + j + 1];
            } else {
              b0 = col0 + j < last_valid ? 0.f : -INFINITY;
              b1 = col0 + j + 1 < last_valid ? 0.f : -INFINITY;
            }
            const float v0 = fmaf(__uint_as_float(v[j]), scale_log2e, b0);
            const float v1 = fmaf(__uint_as_float(v[j + 1]), scale_log2e, b1);
            x2 = fmaxf(x2, fmaxf(v0, v1));
            const float p0 = ex2(v0 - mu), p1 = ex2(v1 - mu);
            sum2 += p0 + p1;
            pk[pk0 + j / 2] = pack_bf16x2(p0, p1);
          }
        }
      };
      if (!(SVG_ABL & 1)) block(sa, 0, 0);
      tc_wait_ld();                 // sb landed
      // first block of the next tile: prefetch it under the arithmetic on sb if S(t+1) is already
      // there (warp-uniform decision), otherwise right after this block
      bool fetched = t + 1 >= U;
      if (!fetched && ((G == 2 && st == 0) ||
                       __all_sync(0xffffffffu, mbar_test(sfull_bar(t + 1), ((t + 1) >> 1) & 1)))) {
        tc_fence_after();
        TMEM_LD32(tSb + (uint32_t)((st ^ 1) * 64), sa);
        fetched = true;
      }
      if (!(SVG_ABL & 1)) block(sb, 32, 16);
      else {
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = sa[j] ^ sb[j];
      }
      float sum = (sum0 + sum1) + (sum2 + sum3);
      // Lazy running max: m only moves when a logit exceeds it by more than 2^kRescaleThreshold.  Full
      // exact tiles do not track their maximum (one FMNMX per logit on the softmax warps' critical
      // path): while every logit stays below m + 8 the 64 exponentials sum to at most 2^14, so a larger
      // (or non-finite) row sum is the trigger, and the tile maximum is taken on the redo path only.
      // Untriggered tiles may hold logits up to m + 14: harmless for fp32 sums and bf16 P.
      float alpha = 1.f;
      const float mt_known = fmaxf(x2, x3);
      const bool maybe = kind == 0 ? !(sum <= 16384.f) || m == -INFINITY
                                   : (mt_known > m + kRescaleThreshold || (m == -INFINITY && mt_known > -INFINITY));
      const bool redo = (SVG_ABL & 2) ? false : __any_sync(0xffffffffu, maybe);
      if (redo) {
        // exact path for the whole warp: tile maximum, raise m where needed, exponentials again
        tc_wait_ld();  // keep the prefetched block of tile t+1 intact in sa
        float mt = mt_known;
        if (kind == 0) {
          mt = -INFINITY;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            TMEM_LD32(tS + half * 32, sb);
            tc_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) mt = fmaxf(mt, __uint_as_float(sb[j]));
          }
          mt *= scale_log2e;
        }
        const bool bump = mt > m + kRescaleThreshold || (m == -INFINITY && mt > -INFINITY);
        if (bump) {
          alpha = ex2(m - mt);  // m = -inf -> 0
          m = mt;
        }
        const float mu2 = (m == -INFINITY) ? 0.f : m;
        sum = 0.f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          TMEM_LD32(tS + half * 32, sb);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float v0 = __uint_as_float(sb[j]) * scale_log2e, v1 = __uint_as_float(sb[j + 1]) * scale_log2e;
            if (kind == 2) {
              v0 += bias[half * 32 + j];
              v1 += bias[half * 32 + j + 1];
            } else if (kind == 1) {
              if (half * 32 + j >= last_valid) v0 = -INFINITY;
              if (half * 32 + j + 1 >= last_valid) v1 = -INFINITY;
            }
            const float p0 = ex2(v0 - mu2), p1 = ex2(v1 - mu2);
            sum += p0 + p1;
            pk[half * 16 + j / 2] = pack_bf16x2(p0, p1);
          }
        }
      }
      l = l * alpha + sum;
      TMEM_ST32(tS, pk);  // P (bf16 pairs) over the first 32 columns of this S buffer
      if (redo && t > 0) {
        // rescale the O accumulator; P.V of tile t-1 must have landed first
        mbar_wait(bar(b_odone), (t - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          TMEM_LD32(tO + c, sb);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sb[j] = __float_as_uint(__uint_as_float(sb[j]) * alpha);
          TMEM_ST32(tO + c, sb);
        }
      }
      // (handing P(t) over later, after the first block of chunk t + 1 so that the TMEM stores run under
      // arithmetic, was measured at 7.25 vs 5.61 ms per 8 heads: the chain P(t) -> P.V(t) -> QK^T(t+2) ->
      // S(t+2) is what the softmax of chunk t + 2 waits for)
      tc_wait_st();  // .sync.aligned: every lane's stores have landed when any lane is past this
      tc_fence_before();
      if (lane == 0) mbar_arrive(bar(b_pfull + st));
      if (!fetched) {
        mbar_wait(sfull_bar(t + 1), ((t + 1) >> 1) & 1);
        tc_fence_after();
        TMEM_LD32(tSb + (uint32_t)((st ^ 1) * 64), sa);
      }
    }
    // ---- epilogue: O / l -> bf16 -> global, scattered to original token order -----------------
    // The per-tile ODONE barrier cannot be used here: a parity wait only tells the current phase
    // from the one before it, and right after the last P hand-off P.V(T-2) may still be in flight
    // (inside the loop a thread holding S(t) knows P.V(t-2) has completed; nothing bounds the lag
    // here), so a wait for phase T-1 could be satisfied by phase T-3 and O read two tiles early.
    // OFINAL has a single phase, committed after the last P.V.
    mbar_wait(bar(B::OFINAL + hf), 0);
    tc_fence_after();
    const int r = tid;  // row within the CTA tile (warps 0-7 <-> rows 0-255)
    const bool live = r < nrows;
    const int prow = min(row0 + r, n_q - 1);
    const int dst = q_perm ? q_perm[(size_t)h * n_q + prow] : prow;
    const float inv = 1.f / l;
    uint4* orow = reinterpret_cast<uint4*>(out + ((size_t)h * n_q + dst) * D);
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      uint32_t o[32];
      TMEM_LD32(tO + c, o);
      tc_wait_ld();
      if (live) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(o[8 * j]) * inv, __uint_as_float(o[8 * j + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(o[8 * j + 2]) * inv, __uint_as_float(o[8 * j + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(o[8 * j + 4]) * inv, __uint_as_float(o[8 * j + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(o[8 * j + 6]) * inv, __uint_as_float(o[8 * j + 7]) * inv);
          orow[c / 8 + j] = w;
        }
      }
    }
    if (lse && live) lse[(size_t)h * n_q + dst] = (m + log2f(l)) * kLn2;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// [rows][d] bf16 row-major, box = 64 columns x box_rows rows, SWIZZLE_128B, zero fill out of bounds
bool encode_rows_map(CUtensorMap* tm, const void* base, uint64_t rows, int d, int box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess || !p) {
      (void)cudaGetLastError();
      return false;
    }
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[2] = {(cuuint64_t)d, rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int NS2, int G2, int NS1, int TPR2 = 1>
static int launch_attend_tc_ns(const SvgEarShape& s, const TmaSet& tm, const int32_t* q_perm,
                               const int32_t* k_sizes, const int32_t* k_offsets, const uint8_t* mask, bf16* out,
                               float* lse, AttendScratch& sc, int ckpad, int mt, float scale_log2e,
                               cudaStream_t st) {
  HelperFork fk(st, 1);
  if (!fk.ok()) return SVGEAR_ECUDA;
  cudaStream_t side = fk.side();
  // tiles with more than 128 live rows: one CTA per SM, two halves sharing every K/V tile
  const size_t smem2 = Smem<D, NS2, 2, G2, TPR2>::bytes(ckpad);
  SVG_CUDA_OK(cudaFuncSetAttribute(attend_tc_kernel<D, NS2, 2, G2, TPR2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  attend_tc_kernel<D, NS2, 2, G2, TPR2><<<dim3(mt, s.bh), threads_for(2, TPR2), smem2, st>>>(
      tm, s.bh * s.n_k, sc.lnw, q_perm, k_sizes, k_offsets, mask, sc.tile_list, sc.tile_count, mt, s.n_q, s.n_k,
      s.c_q, s.c_k, ckpad, scale_log2e, out, lse);
  SVG_LAUNCH_OK();
  // remainder tiles (<= 128 live rows): one half per CTA, two CTAs co-resident per SM so that one
  // CTA's softmax runs under the other's MMAs.  The two kernels write disjoint rows; the second is
  // forked onto a helper stream so that its CTAs fill the tail of the first instead of following it.
  const size_t smem1 = Smem<D, NS1, 1, 1>::bytes(ckpad);
  SVG_CUDA_OK(cudaFuncSetAttribute(attend_tc_kernel<D, NS1, 1, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
  attend_tc_kernel<D, NS1, 1, 1, 1><<<dim3(mt < s.c_q ? mt : s.c_q, s.bh), threads_for(1), smem1, side>>>(
      tm, s.bh * s.n_k, sc.lnw, q_perm, k_sizes, k_offsets, mask, sc.tile_list, sc.tile_count, mt, s.n_q, s.n_k,
      s.c_q, s.c_k, ckpad, scale_log2e, out, lse);
  SVG_LAUNCH_OK();
  return fk.join();
}

int launch_attend_tc(const SvgEarShape& s, const bf16* qp, const bf16* kp, const bf16* vp,
                     const int32_t* q_perm, const int32_t* k_sizes, const int32_t* k_offsets,
                     const uint8_t* mask, bf16* out, float* lse, AttendScratch& sc, int variant,
                     cudaStream_t st) {
  const int ckpad = ceil_div(s.c_k, 64) * 64;
  const int mt = AttendScratch::max_tiles(s.n_q, s.c_q, BM);
  const float scale_log2e = kLog2e / sqrtf((float)s.d);
  if ((long long)s.bh * s.n_k >= (1ll << 31) - 64 || (long long)s.bh * s.n_q >= (1ll << 31) - 512)
    return SVGEAR_EUNSUPPORTED;  // TMA row coordinates are int32
  TmaSet tm;
  bool ok = true;
  for (int i = 0; i < 7; ++i) {
    ok = ok && encode_rows_map(&tm.k[i], kp, (uint64_t)s.bh * s.n_k, s.d, 1 << i);
    ok = ok && encode_rows_map(&tm.v[i], vp, (uint64_t)s.bh * s.n_k, s.d, 1 << i);
  }
  ok = ok && encode_rows_map(&tm.kbar, sc.kbar_bf16, (uint64_t)s.bh * ckpad, s.d, 64);
  ok = ok && encode_rows_map(&tm.vbar, sc.vbar_bf16, (uint64_t)s.bh * ckpad, s.d, 64);
  ok = ok && encode_rows_map(&tm.q, qp, (uint64_t)s.bh * s.n_q, s.d, 64);
  if (!ok) return SVGEAR_ECUDA;
  const size_t cap = 227 * 1024;
#define SVG_TRY(DD, N2, GG, N1)                                                                           \
  if (s.d == DD && (GG == 1 || !force_g1) && Smem<DD, N2, 2, GG>::bytes(ckpad) <= cap &&                   \
      Smem<DD, N1, 1, 1>::bytes(ckpad) <= cap)                                                             \
    return launch_attend_tc_ns<DD, N2, GG, N1>(s, tm, q_perm, k_sizes, k_offsets, mask, out, lse, sc, ckpad, mt, \
                                               scale_log2e, st);
  // Default at d = 128: two threads per query row (16 softmax warps), 64-key tiles.  The measured
  // alternatives stay selectable - per call with the SVGEAR_ATTEND_* bits of svgear_sparse_attend's
  // exec_mode, per process with SVGEAR_ATTEND_TPR=1 (one thread per row) / SVGEAR_ATTEND_G=2 (128-key tiles,
  // one thread per row) for A/B measurements of whole layers (DESIGN 4.1).
  static const bool env_g2 = [] { const char* e = getenv("SVGEAR_ATTEND_G"); return e && e[0] == '2'; }();
  static const bool env_tpr1 = [] { const char* e = getenv("SVGEAR_ATTEND_TPR"); return e && e[0] == '1'; }();
  const bool force_g1 = !(env_g2 || (variant & SVGEAR_ATTEND_TILE128));
  const bool tpr2 = !(env_tpr1 || (variant & SVGEAR_ATTEND_ONE_THREAD_PER_ROW));
  if (tpr2 && force_g1 && s.d == 128 && Smem<128, 4, 2, 1, 2>::bytes(ckpad) <= cap && Smem<128, 2, 1, 1>::bytes(ckpad) <= cap)
    return launch_attend_tc_ns<128, 4, 1, 2, 2>(s, tm, q_perm, k_sizes, k_offsets, mask, out, lse, sc, ckpad, mt,
                                                scale_log2e, st);
  SVG_TRY(128, 2, 2, 2)
  SVG_TRY(128, 4, 1, 2)
  SVG_TRY(128, 3, 1, 2)
  SVG_TRY(128, 2, 1, 2)
  SVG_TRY(64, 3, 2, 4)
  SVG_TRY(64, 4, 1, 4)
  SVG_TRY(64, 2, 1, 2)
#undef SVG_TRY
  return SVGEAR_EUNSUPPORTED;
}

int attend_tc_rows_per_tile() { return BM; }

}  // namespace svg
