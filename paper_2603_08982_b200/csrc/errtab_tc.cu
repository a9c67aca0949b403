// Value-aware / plain block error table on the tensor cores (tcgen05 + TMEM), sm_100a.
//
// Same quantity and arithmetic as error_table_kernel in stats_route.cu (which documents the
// algebra and cites the reference, estimator.py:187-253 / 120-148):
//     E[i,j] = |q_i| * w̄_ij^2 * sum_{t in cluster j} ( A_t - 2 x B_t + x^2 C_t ),  x = expm1(g_it),
//     g_it = q̄_i . (k_t - k̄_j) / sqrt(d)
// but the C_q x N_k x d contraction g runs on the tensor cores:
//   * key_stats_kernel writes, per key, kd = k_t - k̄_j split into bf16 (hi, lo) and the scalars
//     (A_t, B_t, C_t);
//   * q̄ is split into bf16 (hi, lo); g = qh.dh + qh.dl + ql.dh accumulates in fp32 in TMEM
//     (the dropped ql.dl term is 2^-18 relative);
//   * the epilogue owns one query cluster per thread (TMEM lane) and walks the key columns of a
//     key cluster in order, so the per-block sum and its running-max rescale stay in registers and
//     each E[i,j] is written exactly once — no atomics, deterministic.  The epilogue is the bound of
//     this kernel (fp32 issue slots), so its common case is written in packed arithmetic: when every
//     |g| of a chunk is <= 1 (a warp-uniform test on the chunk's largest |g|), expm1 is a degree-8
//     polynomial and two keys go through each fma.rn.f32x2 with no stabiliser; per-key scalars sit in
//     shared memory as separate arrays so that neighbouring keys load as register pairs.  Chunks
//     with larger logits take the scalar path with the running-maximum rescale.
// CTA = (instance, 128 query clusters, a range of key clusters); key clusters stream through in
// chunks of <= 128 keys (N = chunk rounded up to 16), two TMEM buffers, two epilogue warp groups.
//   warps 0-3 / 4-7 : epilogue groups (even / odd key clusters of the range)
//   warp 8 : producer — q̄ tiles once (cp.async), then ONE elected thread streams the chunks: the
//            k - k̄ tiles as 16-row TMA boxes (rows of a cluster are contiguous), the per-key scalars as
//            three bulk copies, all completing on mbarriers, so nothing blocks on a load
//   warp 9 : TMEM allocator + MMA issuer
#include "tc_common.cuh"

namespace svg {

using namespace tc;

namespace {
constexpr int EM = 128;       // query clusters per CTA (M)
constexpr int ECH = 128;      // max keys per chunk
constexpr int ERANGE = 48;    // key clusters per CTA
constexpr int ETHREADS = 320;
enum { EB_AFULL = 0, EB_BFULL = 1, EB_BEMPTY = 3, EB_ACCFULL = 5, EB_ACCEMPTY = 7, EB_STATEMPTY = 9 /* [2 groups][2 buffers] */,
       EB_STATFULL = 13 /* [2 groups][2 buffers] */ };

template <int D>
struct ESmem {
  static constexpr int kTile = EM * D * 2;        // one [128 x d] bf16 tile
  static constexpr int kA = 0;                    // qh, ql
  static constexpr int kB = kA + 2 * kTile;       // 2 stages x (dh, dl)
  static constexpr int kStat = kB + 4 * kTile;
  static constexpr int kBars = kStat + 4 * ECH * 16;  // stats: 2 groups x 2 buffers x (A[128], -2B[128], C[128]) f32
  static constexpr size_t bytes() { return 1024 + kBars + 256; }
};

#define TMEM_LD16(taddr, r)                                                                       \
  asm volatile(                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "                                                   \
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"           \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),       \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),   \
        "=r"(r[14]), "=r"(r[15])                                                                  \
      : "r"(taddr)                                                                                \
      : "memory")

// Per-key scalars live in three planes (A, -2B, C) of `pstride` floats per instance.  Inside a plane
// the keys of cluster j start at a 16-byte aligned position pos_j = align4(offset_j) + 4 j, so that a
// chunk of a cluster is one aligned bulk copy (cp.async.bulk needs 16-byte alignment and size).
__host__ __device__ __forceinline__ size_t stat_plane_stride(int n_k, int c_k) {
  return (((size_t)n_k + 3) & ~(size_t)3) + 4 * (size_t)c_k + 8;  // a multiple of 4 floats: planes stay 16-byte aligned
}
__device__ __forceinline__ int stat_pos(int offset_j, int j) { return ((offset_j + 3) & ~3) + 4 * j; }

// 1-D bulk copy global -> shared, completes `bytes` on `bar` (16-byte aligned addresses and size)
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ float expm1_fast(float g) {
  // |g| < 0.125: degree-4 Taylor (relative error < 3e-6); otherwise 2^(g log2 e) - 1 (< 1e-6)
  const float poly = g * fmaf(g, fmaf(g, fmaf(g, 1.f / 24.f, 1.f / 6.f), 0.5f), 1.f);
  const float big = ex2(g * 1.4426950408889634f) - 1.f;
  return fabsf(g) < 0.125f ? poly : big;
}
}  // namespace

// per key: kd = k - k̄_j as bf16 (hi, lo); (A, B, C) = (|v̄-v|^2, (v̄-v).v, |v|^2)  [plain: 0,0,1]
// stored as three planes A, -2B, C (layout: stat_plane_stride / stat_pos above)
template <int D>
__global__ void __launch_bounds__(128)
    key_stats_kernel(int mode, const float* __restrict__ kc, const float* __restrict__ vc,
                     const bf16* __restrict__ kp, const bf16* __restrict__ vp,
                     const int32_t* __restrict__ k_sizes, const int32_t* __restrict__ k_offsets, int n_k,
                     int c_k, bf16* __restrict__ kd_hi, bf16* __restrict__ kd_lo, float* __restrict__ kstat) {
  const int h = blockIdx.y, j = blockIdx.x;
  constexpr int EPL = D / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nj = k_sizes[(size_t)h * c_k + j], o = k_offsets[(size_t)h * c_k + j];
  float kb[EPL], vb[EPL];
#pragma unroll
  for (int u = 0; u < EPL; ++u) {
    kb[u] = kc[((size_t)h * c_k + j) * D + lane * EPL + u];
    vb[u] = mode == SVGEAR_EST_VALUE_AWARE ? vc[((size_t)h * c_k + j) * D + lane * EPL + u] : 0.f;
  }
  for (int r = warp; r < nj; r += 4) {
    const size_t row = (size_t)h * n_k + o + r;
    float kf[EPL], vf[EPL];
    if constexpr (EPL == 4) {
      const uint2 ku = __ldg(reinterpret_cast<const uint2*>(kp + row * D + lane * 4));
      kf[0] = __uint_as_float(ku.x << 16); kf[1] = __uint_as_float(ku.x & 0xffff0000u);
      kf[2] = __uint_as_float(ku.y << 16); kf[3] = __uint_as_float(ku.y & 0xffff0000u);
      if (mode == SVGEAR_EST_VALUE_AWARE) {
        const uint2 vu = __ldg(reinterpret_cast<const uint2*>(vp + row * D + lane * 4));
        vf[0] = __uint_as_float(vu.x << 16); vf[1] = __uint_as_float(vu.x & 0xffff0000u);
        vf[2] = __uint_as_float(vu.y << 16); vf[3] = __uint_as_float(vu.y & 0xffff0000u);
      }
    } else {
      const uint32_t ku = __ldg(reinterpret_cast<const uint32_t*>(kp + row * D + lane * 2));
      kf[0] = __uint_as_float(ku << 16); kf[1] = __uint_as_float(ku & 0xffff0000u);
      if (mode == SVGEAR_EST_VALUE_AWARE) {
        const uint32_t vu = __ldg(reinterpret_cast<const uint32_t*>(vp + row * D + lane * 2));
        vf[0] = __uint_as_float(vu << 16); vf[1] = __uint_as_float(vu & 0xffff0000u);
      }
    }
    float a = 0.f, b = 0.f, cc = 0.f;
    uint32_t hi[EPL / 2], lo[EPL / 2];
#pragma unroll
    for (int u = 0; u < EPL; u += 2) {
      const float d0 = kf[u] - kb[u], d1 = kf[u + 1] - kb[u + 1];
      const bf16 h0 = __float2bfloat16_rn(d0), h1 = __float2bfloat16_rn(d1);
      hi[u / 2] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
      lo[u / 2] = pack_bf16x2(d0 - __bfloat162float(h0), d1 - __bfloat162float(h1));
    }
    if (mode == SVGEAR_EST_VALUE_AWARE) {
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const float dv = vb[u] - vf[u];
        a = fmaf(dv, dv, a);
        b = fmaf(dv, vf[u], b);
        cc = fmaf(vf[u], vf[u], cc);
      }
      a = warp_sum(a); b = warp_sum(b); cc = warp_sum(cc);
    } else {
      cc = 1.f;
    }
    if constexpr (EPL == 4) {
      *reinterpret_cast<uint2*>(kd_hi + row * D + lane * 4) = make_uint2(hi[0], hi[1]);
      *reinterpret_cast<uint2*>(kd_lo + row * D + lane * 4) = make_uint2(lo[0], lo[1]);
    } else {
      *reinterpret_cast<uint32_t*>(kd_hi + row * D + lane * 2) = hi[0];
      *reinterpret_cast<uint32_t*>(kd_lo + row * D + lane * 2) = lo[0];
    }
    if (lane == 0) {  // planes A, -2B, C (separate arrays: neighbouring keys load as register pairs)
      const size_t ps = stat_plane_stride(n_k, c_k);
      float* dst = kstat + (size_t)h * 3 * ps + stat_pos(o, j) + r;
      dst[0] = a;
      dst[ps] = -2.f * b;
      dst[2 * ps] = cc;
    }
  }
}

// q̄ -> bf16 (hi, lo), zero padded to a multiple of 128 rows: [bh][2][cqpad][d]
__global__ void split_q_kernel(const float* __restrict__ qc, int d, int c_q, int cqpad, bf16* __restrict__ qsplit) {
  const int h = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= cqpad * d) return;
  const float v = (idx / d) < c_q ? qc[(size_t)h * c_q * d + idx] : 0.f;
  const bf16 hi = __float2bfloat16_rn(v);
  qsplit[((size_t)h * 2 + 0) * cqpad * d + idx] = hi;
  qsplit[((size_t)h * 2 + 1) * cqpad * d + idx] = __float2bfloat16_rn(v - __bfloat162float(hi));
}

template <int D>
__global__ void __launch_bounds__(ETHREADS, 1)
    error_table_tc_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                          const bf16* __restrict__ qsplit, const float* __restrict__ kstat,
                          const int32_t* __restrict__ q_sizes, const int32_t* __restrict__ k_sizes,
                          const int32_t* __restrict__ k_offsets, const float* __restrict__ sbar,
                          const float* __restrict__ mref, int n_k, int c_q, int c_k, int cqpad, float scale,
                          double* __restrict__ err) {
  using L = ESmem<D>;
  const int h = blockIdx.z, mt = blockIdx.y;
  const int j_lo = blockIdx.x * ERANGE, j_hi = min(c_k, j_lo + ERANGE);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase + L::kA, sB = sbase + L::kB, bars = sbase + L::kBars;
  const uint32_t sStat = sbase + L::kStat;
  const float* stat_smem = reinterpret_cast<const float*>(smem + L::kStat);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBars + 192);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto bar = [&](int i) -> uint32_t { return bars + 8u * (uint32_t)i; };

  if (tid == 0) {
    mbar_init(bar(EB_AFULL), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(EB_BFULL + s), 1);
      mbar_init(bar(EB_BEMPTY + s), 1);
      mbar_init(bar(EB_ACCFULL + s), 1);
      mbar_init(bar(EB_ACCEMPTY + s), 128);
      mbar_init(bar(EB_STATEMPTY + 2 * s), 128);
      mbar_init(bar(EB_STATEMPTY + 2 * s + 1), 128);
      mbar_init(bar(EB_STATFULL + 2 * s), 1);
      mbar_init(bar(EB_STATFULL + 2 * s + 1), 1);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(smem_u32(tmem_slot), 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int32_t* ksz = k_sizes + (size_t)h * c_k;
  const int32_t* kof = k_offsets + (size_t)h * c_k;

  if (warp == 8) {
    // =========================== producer ========================================================
    constexpr int CPR = D / 8, RPI = 32 / CPR;
    const int sub = lane / CPR, chunk = lane % CPR;
    for (int p = 0; p < 2; ++p) {
      const bf16* src = qsplit + (((size_t)h * 2 + p) * cqpad + (size_t)mt * EM) * D;
      for (int r0 = 0; r0 < EM; r0 += RPI) {
        const int r = r0 + sub;
        cp_async16(sA + (uint32_t)(p * L::kTile + (chunk >> 3) * (EM * 128)) + swz(r, chunk & 7),
                   src + (size_t)r * D + chunk * 8);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar(EB_AFULL));
    if (elect_one()) {
      const size_t ps = stat_plane_stride(n_k, c_k);
      const float* planes = kstat + (size_t)h * 3 * ps;
      int u = 0, guses[2] = {0, 0};
      for (int j = j_lo; j < j_hi; ++j) {
        const int nj = ksz[j], o = kof[j];
        const int g = (j - j_lo) & 1;
        const int pos = stat_pos(o, j);
        for (int s0 = 0; s0 < nj; s0 += ECH, ++u) {
          const int gu = guses[g]++;  // use number of this chunk within its epilogue group
          const int st = u & 1;
          if (u >= 2) mbar_wait(bar(EB_BEMPTY + st), ((u >> 1) + 1) & 1);
          const int valid = min(ECH, nj - s0);
          const int nn = ((valid + 15) >> 4) << 4;
          const uint32_t fb = bar(EB_BFULL + st);
          mbar_expect_tx(fb, (uint32_t)(2 * nn * D * 2));
          const int row = h * n_k + o + s0;
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const CUtensorMap* tm = p == 0 ? &map_hi : &map_lo;
            const uint32_t dst = sB + (uint32_t)((st * 2 + p) * L::kTile);
            for (int rb = 0; rb < nn; rb += 16)
#pragma unroll
              for (int sl = 0; sl < D / 64; ++sl)
                tma_box(dst + (uint32_t)(sl * (EM * 128) + rb * 128), tm, sl * 64, row + rb, fb);
          }
          // per-key scalars: stat buffer (group g, use parity); its previous user was use gu-2
          const int sb = g * 2 + (gu & 1);
          if (gu >= 2) mbar_wait(bar(EB_STATEMPTY + sb), ((gu >> 1) + 1) & 1);
          const uint32_t nbytes = (uint32_t)(((valid + 3) >> 2) << 4);
          const uint32_t sf = bar(EB_STATFULL + sb);
          mbar_expect_tx(sf, 3 * nbytes);
#pragma unroll
          for (int pl = 0; pl < 3; ++pl)
            bulk_copy(sStat + (uint32_t)((sb * 3 + pl) * ECH * 4), planes + (size_t)pl * ps + pos + s0, nbytes, sf);
        }
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // =========================== MMA issuer ======================================================
    if (elect_one()) {
      mbar_wait(bar(EB_AFULL), 0);
      int u = 0, uses[2] = {0, 0};
      for (int j = j_lo; j < j_hi; ++j) {
        const int nj = ksz[j];
        const int g = (j - j_lo) & 1;  // TMEM buffer / epilogue group of this key cluster
        for (int s0 = 0; s0 < nj; s0 += ECH, ++u) {
          const int st = u & 1;
          const int nn = ((min(ECH, nj - s0) + 15) >> 4) << 4;
          const uint32_t idesc = make_idesc(EM, nn, 0);
          if (uses[g] >= 1) mbar_wait(bar(EB_ACCEMPTY + g), (uses[g] - 1) & 1);
          mbar_wait(bar(EB_BFULL + st), (u >> 1) & 1);
          tc_fence_after();
          // g = qh.dh + qh.dl + ql.dh
#pragma unroll
          for (int prod = 0; prod < 3; ++prod) {
            const uint32_t at = sA + (uint32_t)((prod == 2 ? 1 : 0) * L::kTile);
            const uint32_t bt = sB + (uint32_t)((st * 2 + (prod == 1 ? 1 : 0)) * L::kTile);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint64_t ad = make_desc(at + (uint32_t)((kk >> 2) * (EM * 128) + (kk & 3) * 32), 16, 1024);
              const uint64_t bd = make_desc(bt + (uint32_t)((kk >> 2) * (EM * 128) + (kk & 3) * 32), 16, 1024);
              umma_ss(tmem + (uint32_t)(g * 128), ad, bd, idesc, (prod > 0 || kk > 0) ? 1u : 0u);
            }
          }
          umma_commit(bar(EB_BEMPTY + st));
          umma_commit(bar(EB_ACCFULL + g));
          ++uses[g];
        }
      }
    }
    __syncwarp();
  } else {
    // =========================== epilogue groups =================================================
    const int g = warp >> 2;
    const int i = mt * EM + (warp & 3) * 32 + lane;  // query cluster of this thread
    const bool live = i < c_q;
    const uint32_t tcol = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(g * 128);
    const float mr = live ? mref[(size_t)h * c_q + i] : 0.f;
    const double nq = live ? (double)q_sizes[(size_t)h * c_q + i] : 0.0;
    int uses = 0, u = 0;  // u = global chunk counter (selects the stage the producer used)
    for (int j = j_lo; j < j_hi; ++j) {
      const int nj = ksz[j];
      if (((j - j_lo) & 1) != g) {  // the other group's cluster: just advance the chunk counter
        u += (nj + ECH - 1) / ECH;
        continue;
      }
      const size_t e = ((size_t)h * c_q + (live ? i : 0)) * c_k + j;
      const float sb = sbar[e];  // issued early; consumed after the chunks
      float M = 0.f, em = 1.f, em2 = 1.f, acc = 0.f;
      for (int s0 = 0; s0 < nj; s0 += ECH, ++uses, ++u) {
        const int valid = min(ECH, nj - s0);
        const int sbuf = g * 2 + (uses & 1);
        const float* ksA = stat_smem + sbuf * (3 * ECH);
        const float* ksB = ksA + ECH;  // -2B
        const float* ksC = ksB + ECH;
        mbar_wait(bar(EB_STATFULL + sbuf), (uses >> 1) & 1);
        mbar_wait(bar(EB_ACCFULL + g), uses & 1);
        tc_fence_after();
        // pass 1: largest |g| of the chunk for this query cluster (columns beyond the chunk masked)
        float amax = 0.f;
        for (int c0 = 0; c0 < valid; c0 += 16) {
          uint32_t a[16];
          TMEM_LD16(tcol + c0, a);
          tc_wait_ld();
          if (c0 + 16 <= valid) {
#pragma unroll
            for (int q = 0; q < 16; ++q) amax = fmaxf(amax, fabsf(__uint_as_float(a[q])));
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) amax = fmaxf(amax, c0 + q < valid ? fabsf(__uint_as_float(a[q])) : 0.f);
          }
        }
        if (!__any_sync(0xffffffffu, amax * scale > 1.0f)) {
          // ---- packed path: |g| <= 1 for every lane of the warp.  x = expm1(g) by the degree-8 series
          // (g^9/9! < 2.8e-6), two keys per instruction, no stabiliser: S = sum A - 2B x + C x^2, then
          // acc += exp(-2M) S (M is the block's running maximum; it only moves in the scalar path).
          const uint64_t sc2 = pack2(scale, scale);
          uint64_t s2 = pack2(0.f, 0.f);
          for (int c0 = 0; c0 < valid; c0 += 16) {
            uint32_t a[16];
            TMEM_LD16(tcol + c0, a);
            tc_wait_ld();
            if (c0 + 16 > valid) {
#pragma unroll
              for (int q = 0; q < 16; ++q) a[q] = c0 + q < valid ? a[q] : 0u;  // g = 0 where the scalars are 0
            }
#pragma unroll
            for (int q4 = 0; q4 < 16; q4 += 4) {
              float4 A4 = *reinterpret_cast<const float4*>(ksA + c0 + q4);
              float4 B4 = *reinterpret_cast<const float4*>(ksB + c0 + q4);
              float4 C4 = *reinterpret_cast<const float4*>(ksC + c0 + q4);
              if (c0 + q4 + 4 > valid) {  // past the chunk: whatever follows in the plane (or stale) -> 0
                const int left = valid - (c0 + q4);
                if (left < 4) { A4.w = B4.w = C4.w = 0.f; }
                if (left < 3) { A4.z = B4.z = C4.z = 0.f; }
                if (left < 2) { A4.y = B4.y = C4.y = 0.f; }
                if (left < 1) { A4.x = B4.x = C4.x = 0.f; }
              }
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const uint64_t g2 = fmul2(pack2(__uint_as_float(a[q4 + 2 * hh]), __uint_as_float(a[q4 + 2 * hh + 1])), sc2);
                uint64_t pz = ffma2(g2, pack2(1.f / 40320.f, 1.f / 40320.f), pack2(1.f / 5040.f, 1.f / 5040.f));
                pz = ffma2(pz, g2, pack2(1.f / 720.f, 1.f / 720.f));
                pz = ffma2(pz, g2, pack2(1.f / 120.f, 1.f / 120.f));
                pz = ffma2(pz, g2, pack2(1.f / 24.f, 1.f / 24.f));
                pz = ffma2(pz, g2, pack2(1.f / 6.f, 1.f / 6.f));
                pz = ffma2(pz, g2, pack2(0.5f, 0.5f));
                pz = ffma2(pz, g2, pack2(1.f, 1.f));
                const uint64_t x2 = fmul2(pz, g2);
                const uint64_t A2 = hh ? pack2(A4.z, A4.w) : pack2(A4.x, A4.y);
                const uint64_t B2 = hh ? pack2(B4.z, B4.w) : pack2(B4.x, B4.y);
                const uint64_t C2 = hh ? pack2(C4.z, C4.w) : pack2(C4.x, C4.y);
                s2 = fadd2(s2, ffma2(ffma2(C2, x2, B2), x2, A2));
              }
            }
          }
          float s_lo, s_hi;
          unpack2(s2, s_lo, s_hi);
          acc = fmaf(em2, s_lo + s_hi, acc);
        } else {
          // ---- scalar path: chunk maximum of g -> raise the running maximum once, then accumulate at
          // the fixed maximum M:  xs = exp(g - M) - exp(-M) = em * expm1(g)
          float gmax = -INFINITY;
          for (int c0 = 0; c0 < valid; c0 += 16) {
            uint32_t a[16];
            TMEM_LD16(tcol + c0, a);
            tc_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q)
              gmax = fmaxf(gmax, c0 + q < valid ? __uint_as_float(a[q]) : -INFINITY);
          }
          gmax *= scale;
          if (gmax > M) {
            const float r = __expf(M - gmax);
            acc *= r * r;
            M = gmax;
            em = __expf(-M);
            em2 = em * em;
          }
          for (int c0 = 0; c0 < valid; c0 += 16) {
            uint32_t a[16];
            TMEM_LD16(tcol + c0, a);
            tc_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float gg = fminf(__uint_as_float(a[q]) * scale, 85.f);
              const float xs = expm1_fast(gg) * em;
              // A em^2 - 2B (em xs) + C xs^2, Horner in xs
              const float term = fmaf(fmaf(ksC[c0 + q], xs, ksB[c0 + q] * em), xs, ksA[c0 + q] * em2);
              acc += c0 + q < valid ? term : 0.f;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(bar(EB_ACCEMPTY + g));
        mbar_arrive(bar(EB_STATEMPTY + sbuf));
      }
      if (live) {
        const double lift = 2.0 * ((double)sb - (double)mr + (double)M);
        err[e] = nq * ((double)fmaxf(acc, 0.f) * exp(lift));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

size_t errtab_stat_floats(const SvgEarShape& s) { return (size_t)s.bh * 3 * stat_plane_stride(s.n_k, s.c_k) + 64; }

size_t errtab_tc_scratch_bytes(const SvgEarShape& s) {
  const int cqpad = ceil_div(s.c_q, EM) * EM;
  return align_up((size_t)s.bh * s.n_k * s.d * 2, 256) * 2 + align_up(errtab_stat_floats(s) * 4, 256) +
         align_up((size_t)s.bh * 2 * cqpad * s.d * 2, 256) + 1024;
}

// key-side half of the estimator (needs only the key clustering): k - k̄ split + per-key scalars
int launch_key_stats(const SvgEarShape& s, int mode, const float* kc, const float* vc, const bf16* kp,
                     const bf16* vp, const int32_t* k_sizes, const int32_t* k_offsets, bf16* kd_hi, bf16* kd_lo,
                     float* kstat, cudaStream_t st) {
  if (s.d == 128)
    key_stats_kernel<128><<<dim3(s.c_k, s.bh), 128, 0, st>>>(mode, kc, vc, kp, vp, k_sizes, k_offsets, s.n_k,
                                                            s.c_k, kd_hi, kd_lo, kstat);
  else
    key_stats_kernel<64><<<dim3(s.c_k, s.bh), 128, 0, st>>>(mode, kc, vc, kp, vp, k_sizes, k_offsets, s.n_k,
                                                           s.c_k, kd_hi, kd_lo, kstat);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

int launch_error_table_tc(const SvgEarShape& s, int mode, const float* qc, const float* kc, const float* vc,
                          const bf16* kp, const bf16* vp, const int32_t* q_sizes, const int32_t* k_sizes,
                          const int32_t* k_offsets, const float* sbar, const float* mref, bf16* kd_hi,
                          bf16* kd_lo, float* kstat, bf16* qsplit, double* err, bool key_stats_done,
                          cudaStream_t st) {
  const int cqpad = ceil_div(s.c_q, EM) * EM;
  const float scale = 1.0f / sqrtf((float)s.d);
  split_q_kernel<<<dim3(ceil_div(cqpad * s.d, 256), s.bh), 256, 0, st>>>(qc, s.d, s.c_q, cqpad, qsplit);
  SVG_LAUNCH_OK();
  if (!key_stats_done) {
    const int rc = launch_key_stats(s, mode, kc, vc, kp, vp, k_sizes, k_offsets, kd_hi, kd_lo, kstat, st);
    if (rc) return rc;
  }
  CUtensorMap map_hi, map_lo;  // [bh*n_k][d] bf16, box = 64 columns x 16 rows
  if (!encode_rows_map(&map_hi, kd_hi, (uint64_t)s.bh * s.n_k, s.d, 16) ||
      !encode_rows_map(&map_lo, kd_lo, (uint64_t)s.bh * s.n_k, s.d, 16))
    return SVGEAR_ECUDA;
  dim3 grid(ceil_div(s.c_k, ERANGE), cqpad / EM, s.bh);
  if (s.d == 128) {
    const size_t smem = ESmem<128>::bytes();
    SVG_CUDA_OK(cudaFuncSetAttribute(error_table_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    error_table_tc_kernel<128><<<grid, ETHREADS, smem, st>>>(map_hi, map_lo, qsplit, kstat, q_sizes, k_sizes,
                                                             k_offsets, sbar, mref, s.n_k, s.c_q, s.c_k, cqpad,
                                                             scale, err);
  } else {
    const size_t smem = ESmem<64>::bytes();
    SVG_CUDA_OK(cudaFuncSetAttribute(error_table_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    error_table_tc_kernel<64><<<grid, ETHREADS, smem, st>>>(map_hi, map_lo, qsplit, kstat, q_sizes, k_sizes,
                                                            k_offsets, sbar, mref, s.n_k, s.c_q, s.c_k, cqpad,
                                                            scale, err);
  }
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
