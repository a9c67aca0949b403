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
// One CTA = one 128-row query tile of one query cluster (tile list built by build_tiles_kernel);
// two CTAs are co-resident per SM (each: 256 TMEM columns, ~108 KB shared memory) so one CTA's
// softmax overlaps the other's MMAs.
//   warps 0-3 : softmax + epilogue, one thread per query row (TMEM lane == row)
//   warp  4   : K producer   (cp.async gathers into the canonical SWIZZLE_128B layout)
//   warp  5   : V producer
//   warp  6   : TMEM allocator + single-thread tcgen05.mma issuer
// TMEM columns: S0 [0,64)  S1 [64,128)  O [128,128+D).  P (bf16) overwrites its S buffer and is the
// A operand of the P.V MMA straight from TMEM; S is double buffered so QK^T of tile t+1 runs while
// the softmax of tile t is in flight.  The running maximum is only raised when it grows by more
// than 2^8 (lazy rescale), which keeps the O accumulator in TMEM untouched on almost every tile.
#include "tc_common.cuh"

namespace svg {

using namespace tc;

namespace {

constexpr int BM = 128;      // query rows per CTA
constexpr int BN = 64;       // keys per tile
constexpr int NTHREADS = 224;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct Smem {
  static constexpr int kQBytes = BM * D * 2;
  static constexpr int kTileBytes = BN * D * 2;
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;            // 2 stages
  static constexpr int kV = kK + 2 * kTileBytes;     // 2 stages
  static constexpr int kBars = kV + 2 * kTileBytes;  // 16 mbarriers + tmem ptr
  static constexpr int kLists = kBars + 256;
  static size_t bytes(int ckpad) { return 1024 + kLists + (size_t)(ckpad + 64) * 12; }
};

enum { B_QFULL = 0, B_KFULL = 1, B_KEMPTY = 3, B_VFULL = 5, B_VEMPTY = 7, B_SFULL = 9, B_PFULL = 11, B_ODONE = 13 };

}  // namespace

template <int D>
__global__ void __launch_bounds__(NTHREADS, 2)
    attend_tc_kernel(const bf16* __restrict__ qp, const bf16* __restrict__ kp, const bf16* __restrict__ vp,
                     const bf16* __restrict__ kbar, const bf16* __restrict__ vbar,
                     const float* __restrict__ lnw, const int32_t* __restrict__ q_perm,
                     const int32_t* __restrict__ k_sizes, const int32_t* __restrict__ k_offsets,
                     const uint8_t* __restrict__ mask, const int32_t* __restrict__ tile_list,
                     const int32_t* __restrict__ tile_count, int max_tiles, int n_q, int n_k, int c_q,
                     int c_k, int ckpad, float scale_log2e, bf16* __restrict__ out,
                     float* __restrict__ lse) {
  using L = Smem<D>;
  const int h = blockIdx.y;
  if ((int)blockIdx.x >= tile_count[h]) return;
  const int32_t* te = tile_list + ((size_t)h * max_tiles + blockIdx.x) * 4;
  const int qcl = te[0], row0 = te[1], nrows = te[2];

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase + L::kQ, sK = sbase + L::kK, sV = sbase + L::kV;
  const uint32_t bars = sbase + L::kBars;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBars + 128);
  int32_t* s_total = reinterpret_cast<int32_t*>(smem + L::kBars + 136);  // [0]=selected keys
  int32_t* s_pre = reinterpret_cast<int32_t*>(smem + L::kLists);          // [nsel+1] key prefix
  int32_t* s_row = s_pre + (ckpad + 64);                                    // [nsel] first row
  float* s_bias = reinterpret_cast<float*>(s_row + (ckpad + 64));          // [ckpad] log2 domain

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto bar = [&](int i) -> uint32_t { return bars + 8u * (uint32_t)i; };

  // ---- prologue: barriers, TMEM, per-cluster selection lists ------------------------------------
  if (tid == 0) {
    mbar_init(bar(B_QFULL), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_KFULL + s), 1);
      mbar_init(bar(B_KEMPTY + s), 1);
      mbar_init(bar(B_VFULL + s), 1);
      mbar_init(bar(B_VEMPTY + s), 1);
      mbar_init(bar(B_SFULL + s), 1);
      mbar_init(bar(B_PFULL + s), 128);
    }
    mbar_init(bar(B_ODONE), 1);
    fence_barrier_init();
  }
  if (warp == 6) tmem_alloc(smem_u32(tmem_slot), 256);
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
  } else if (warp >= 1 && warp <= 3) {
    for (int j = tid - 32; j < ckpad; j += 96)
      s_bias[j] = (j < c_k && mrow[j] == 0) ? lnw[(size_t)h * c_k + j] * kLog2e : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total_keys = s_total[0];
  const int n_exact = (total_keys + BN - 1) / BN;
  const int n_cent = ckpad / BN;
  const int T = n_exact + n_cent;

  if (warp == 4 || warp == 5) {
    // =========================== producers: K (warp 4) / V (warp 5) ===========================
    const bool is_k = warp == 4;
    const bf16* src_tok = (is_k ? kp : vp) + (size_t)h * n_k * D;
    const bf16* src_cen = (is_k ? kbar : vbar) + (size_t)h * ckpad * D;
    const uint32_t sbuf = is_k ? sK : sV;
    const int b_full = is_k ? B_KFULL : B_VFULL, b_empty = is_k ? B_KEMPTY : B_VEMPTY;
    constexpr int CPR = D / 8;          // 16-byte chunks per row
    constexpr int RPI = 32 / CPR;       // rows covered by one warp-wide cp.async
    const int sub = lane / CPR, chunk = lane % CPR;
    if (is_k) {
      // Q tile first (contiguous rows of the permuted Q, clamped at the end of the instance)
      const bf16* qsrc = qp + (size_t)h * n_q * D;
      for (int r0 = 0; r0 < BM; r0 += RPI) {
        const int r = r0 + sub;
        const int row = min(row0 + r, n_q - 1);
        cp_async16(sQ + (uint32_t)((chunk >> 3) * (BM * 128)) + swz(r, chunk & 7),
                   qsrc + (size_t)row * D + chunk * 8);
      }
      cp_async_commit();
      cp_async_wait_all();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(B_QFULL));
    }
    uint32_t xo[8 / RPI];  // ((chunk & 7) ^ (row & 7)) << 4 for the 8/RPI row phases of this lane
#pragma unroll
    for (int j = 0; j < 8 / RPI; ++j) xo[j] = (uint32_t)(((chunk & 7) ^ ((j * RPI + sub) & 7)) << 4);
    int cur0 = 0, cur1 = 0;  // cursors into the selection list for slots lane and lane+32
    const int last_key = max(total_keys - 1, 0);
    for (int t = 0; t < T; ++t) {
      const int st = t & 1;
      if (t >= 2) mbar_wait(bar(b_empty + st), ((t >> 1) + 1) & 1);
      // source row of tile slots `lane` and `lane + 32`
      const bf16* base;
      int r_lo, r_hi;
      if (t < n_exact) {
        base = src_tok;
        int u0 = min(t * BN + lane, last_key), u1 = min(t * BN + lane + 32, last_key);
        while (s_pre[cur0 + 1] <= u0) ++cur0;
        if (cur1 < cur0) cur1 = cur0;
        while (s_pre[cur1 + 1] <= u1) ++cur1;
        r_lo = s_row[cur0] + (u0 - s_pre[cur0]);
        r_hi = s_row[cur1] + (u1 - s_pre[cur1]);
      } else {
        base = src_cen;
        r_lo = (t - n_exact) * BN + lane;
        r_hi = r_lo + 32;
      }
      // lane-constant parts of the swizzled destination: the XOR pattern repeats every 8 rows
      const uint32_t dst = sbuf + (uint32_t)st * L::kTileBytes + (uint32_t)((chunk >> 3) * (BN * 128)) +
                           (uint32_t)(sub * 128);
      const char* src = reinterpret_cast<const char*>(base) + chunk * 16;
#pragma unroll
      for (int r0 = 0; r0 < BN; r0 += RPI) {
        const int srow = __shfl_sync(0xffffffffu, r0 < 32 ? r_lo : r_hi, (r0 & 31) + sub);
        cp_async16(dst + (uint32_t)(r0 * 128) + xo[(r0 / RPI) % (8 / RPI)], src + (size_t)srow * (D * 2));
      }
      cp_async_commit();
      cp_async_wait_all();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(b_full + st));
    }
  } else if (warp == 6) {
    // =========================== MMA issuer (one elected thread) ===============================
    if (elect_one()) {
      constexpr uint32_t idesc_qk = make_idesc(BM, BN, 0);
      constexpr uint32_t idesc_pv = make_idesc(BM, D, 1);
      const uint32_t tS[2] = {tmem, tmem + 64};
      const uint32_t tO = tmem + 128;
      auto issue_qk = [&](int t) {
        const int st = t & 1;
        mbar_wait(bar(B_KFULL + st), (t >> 1) & 1);
        tc_fence_after();
        const uint32_t kb = sK + (uint32_t)st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = make_desc(sQ + (uint32_t)((kk >> 2) * (BM * 128) + (kk & 3) * 32), 16, 1024);
          const uint64_t bd = make_desc(kb + (uint32_t)((kk >> 2) * (BN * 128) + (kk & 3) * 32), 16, 1024);
          umma_ss(tS[st], ad, bd, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(bar(B_SFULL + st));
        umma_commit(bar(B_KEMPTY + st));
      };
      mbar_wait(bar(B_QFULL), 0);
      issue_qk(0);
      for (int t = 0; t < T; ++t) {
        const int st = t & 1;
        if (t + 1 < T) issue_qk(t + 1);
        mbar_wait(bar(B_VFULL + st), (t >> 1) & 1);
        mbar_wait(bar(B_PFULL + st), (t >> 1) & 1);
        tc_fence_after();
        const uint32_t vb = sV + (uint32_t)st * L::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // V tile [64 keys x D] is the MN-major B operand: 16 keys per MMA = 2048 B along K,
          // LBO = stride between the 64-column slabs, SBO = stride between 8-key groups
          const uint64_t bd = make_desc(vb + (uint32_t)(kk * 2048), BN * 128, 1024);
          umma_ts(tO, tS[st] + (uint32_t)(kk * 8), bd, idesc_pv, (t > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(bar(B_VEMPTY + st));
        umma_commit(bar(B_ODONE));
      }
    }
    __syncwarp();
  } else {
    // =========================== softmax + epilogue (warps 0-3, thread == row) ==================
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t tS[2] = {tmem + lane_base, tmem + lane_base + 64};
    const uint32_t tO = tmem + lane_base + 128;
    float m = -INFINITY, l = 0.f;
    for (int t = 0; t < T; ++t) {
      const int st = t & 1;
      mbar_wait(bar(B_SFULL + st), (t >> 1) & 1);
      tc_fence_after();
      uint32_t sa[32], sb[32];
      TMEM_LD32(tS[st], sa);
      TMEM_LD32(tS[st] + 32, sb);
      tc_wait_ld();
      float mt = -INFINITY;
      float cmul = 1.f;  // multiplier still to be applied to sa/sb inside the exponential
      if (t < n_exact - 1) {
        // full exact tile: keep the raw logits, fold the scale into the exp2 FFMA below
#pragma unroll
        for (int j = 0; j < 32; ++j) mt = fmaxf(mt, fmaxf(__uint_as_float(sa[j]), __uint_as_float(sb[j])));
        mt *= scale_log2e;
        cmul = scale_log2e;
      } else if (t < n_exact) {
        const int valid = total_keys - t * BN;  // 1..64 valid columns in the last exact tile
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = j < valid ? __uint_as_float(sa[j]) * scale_log2e : -INFINITY;
          float y = j + 32 < valid ? __uint_as_float(sb[j]) * scale_log2e : -INFINITY;
          sa[j] = __float_as_uint(x);
          sb[j] = __float_as_uint(y);
          mt = fmaxf(mt, fmaxf(x, y));
        }
      } else {
        const float* bias = s_bias + (t - n_exact) * BN;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = fmaf(__uint_as_float(sa[j]), scale_log2e, bias[j]);
          float y = fmaf(__uint_as_float(sb[j]), scale_log2e, bias[j + 32]);
          sa[j] = __float_as_uint(x);
          sb[j] = __float_as_uint(y);
          mt = fmaxf(mt, fmaxf(x, y));
        }
      }
      // lazy running max: only move it when it grows by more than 2^kRescaleThreshold
      float alpha = 1.f;
      const bool bump = mt > m + kRescaleThreshold || (m == -INFINITY && mt > -INFINITY);
      if (bump) {
        alpha = ex2(m - mt);  // m = -inf -> 0
        m = mt;
      }
      const float mu = (m == -INFINITY) ? 0.f : m;
      float sum = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float p0 = ex2(fmaf(__uint_as_float(sa[2 * j]), cmul, -mu)), p1 = ex2(fmaf(__uint_as_float(sa[2 * j + 1]), cmul, -mu));
        sum += p0 + p1;
        pk[j] = pack_bf16x2(p0, p1);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float p0 = ex2(fmaf(__uint_as_float(sb[2 * j]), cmul, -mu)), p1 = ex2(fmaf(__uint_as_float(sb[2 * j + 1]), cmul, -mu));
        sum += p0 + p1;
        pk[16 + j] = pack_bf16x2(p0, p1);
      }
      l = l * alpha + sum;
      TMEM_ST32(tS[st], pk);  // P (bf16 pairs) over the first 32 columns of this S buffer
      if (t > 0 && __any_sync(0xffffffffu, bump)) {
        // rescale the O accumulator; P.V of tile t-1 must have landed first
        mbar_wait(bar(B_ODONE), (t - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          TMEM_LD32(tO + c, o);
          tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          TMEM_ST32(tO + c, o);
        }
      }
      tc_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_PFULL + st));
    }
    // ---- epilogue: O / l -> bf16 -> global, scattered to original token order -----------------
    mbar_wait(bar(B_ODONE), (T - 1) & 1);
    tc_fence_after();
    const int r = tid;
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
  if (warp == 6) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int launch_attend_tc(const SvgEarShape& s, const bf16* qp, const bf16* kp, const bf16* vp,
                     const int32_t* q_perm, const int32_t* k_sizes, const int32_t* k_offsets,
                     const uint8_t* mask, bf16* out, float* lse, AttendScratch& sc, cudaStream_t st) {
  const int ckpad = ceil_div(s.c_k, 64) * 64;
  const int mt = AttendScratch::max_tiles(s.n_q, s.c_q, BM);
  const float scale_log2e = kLog2e / sqrtf((float)s.d);
  if (s.d == 128) {
    const size_t smem = Smem<128>::bytes(ckpad);
    if (smem > 227 * 1024) return SVGEAR_EUNSUPPORTED;
    SVG_CUDA_OK(cudaFuncSetAttribute(attend_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attend_tc_kernel<128><<<dim3(mt, s.bh), NTHREADS, smem, st>>>(
        qp, kp, vp, sc.kbar_bf16, sc.vbar_bf16, sc.lnw, q_perm, k_sizes, k_offsets, mask, sc.tile_list,
        sc.tile_count, mt, s.n_q, s.n_k, s.c_q, s.c_k, ckpad, scale_log2e, out, lse);
  } else {
    const size_t smem = Smem<64>::bytes(ckpad);
    if (smem > 227 * 1024) return SVGEAR_EUNSUPPORTED;
    SVG_CUDA_OK(cudaFuncSetAttribute(attend_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attend_tc_kernel<64><<<dim3(mt, s.bh), NTHREADS, smem, st>>>(
        qp, kp, vp, sc.kbar_bf16, sc.vbar_bf16, sc.lnw, q_perm, k_sizes, k_offsets, mask, sc.tile_list,
        sc.tile_count, mt, s.n_q, s.n_k, s.c_q, s.c_k, ckpad, scale_log2e, out, lse);
  }
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
