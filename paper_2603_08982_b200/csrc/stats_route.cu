// Block statistics, the value-aware error table and budgeted routing (subsystem 2).
//
// Reference semantics:
//   estimator.estimate_errors_streaming  estimator.py:187-253   (value-aware, Eq.8)
//   estimator.estimate_errors            estimator.py:120-148   (plain, Eq.5)
//   estimator.to_ratios                  estimator.py:83-96     order (-ratio,-error,qc,kc)
//   router._greedy_fill                  router.py:100-110
//   router._apply_single_item_fallback   router.py:113-121
//   router.route_score                   router.py:253-280
//
// Error table arithmetic.  With g_it = (q̄_i.(k_t - k̄_j))/sqrt(d) for key t of cluster j,
//   || w̄_ij v̄_j - e_it v_t ||^2 = w̄_ij^2 || (v̄_j - v_t) - expm1(g_it) v_t ||^2
//                                = w̄_ij^2 ( A_t - 2 x B_t + x^2 C_t ),   x = expm1(g_it)
// with per-key scalars A_t = |v̄_j - v_t|^2, B_t = (v̄_j - v_t).v_t, C_t = |v_t|^2 that do not
// depend on the query cluster.  This is the reference's quantity exactly (w̄ = exp(s̄_ij - m_ref),
// e = exp(logit - m_ref) = w̄ exp(g)), but evaluated from DIFFERENCES so that fp32 keeps the
// small residuals of tight clusters; a running maximum M of g (the reference's m_loc - s̄_ij)
// keeps every exponential <= 1, and the final rescale exp(2(s̄_ij - m_ref + M)) is applied in
// float64, the type of the reference's table.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace svg {

// ------------------------------------------------------------------------------------------------
// centroid logits s̄ = q̄ k̄^T / sqrt(d) and their row maxima (estimator.py:216-217)
// ------------------------------------------------------------------------------------------------
constexpr int kLogitRows = 8;  // query clusters per block (each k̄ row is read once per block)
__global__ void __launch_bounds__(256)
    centroid_logits_kernel(const float* __restrict__ qc, const float* __restrict__ kc, int d,
                           int c_q, int c_k, float scale, float* __restrict__ sbar,
                           float* __restrict__ mref) {
  const int h = blockIdx.y, i0 = blockIdx.x * kLogitRows;
  __shared__ float sq[kLogitRows][128];
  __shared__ float smax[8][kLogitRows];
  const int tid = threadIdx.x;
  for (int e = tid; e < kLogitRows * d; e += 256) {
    const int r = e / d, k = e % d;
    sq[r][k] = (i0 + r < c_q) ? qc[((size_t)h * c_q + i0 + r) * d + k] : 0.f;
  }
  __syncthreads();
  float mx[kLogitRows];
#pragma unroll
  for (int r = 0; r < kLogitRows; ++r) mx[r] = -INFINITY;
  for (int j = tid; j < c_k; j += 256) {
    const float4* kp = reinterpret_cast<const float4*>(kc + ((size_t)h * c_k + j) * d);
    float s[kLogitRows];
#pragma unroll
    for (int r = 0; r < kLogitRows; ++r) s[r] = 0.f;
    for (int q = 0; q < d / 4; ++q) {
      const float4 kv = __ldg(kp + q);
#pragma unroll
      for (int r = 0; r < kLogitRows; ++r) {
        s[r] = fmaf(sq[r][4 * q], kv.x, s[r]);
        s[r] = fmaf(sq[r][4 * q + 1], kv.y, s[r]);
        s[r] = fmaf(sq[r][4 * q + 2], kv.z, s[r]);
        s[r] = fmaf(sq[r][4 * q + 3], kv.w, s[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kLogitRows; ++r) {
      if (i0 + r < c_q) {
        const float v = s[r] * scale;
        sbar[((size_t)h * c_q + i0 + r) * c_k + j] = v;
        mx[r] = fmaxf(mx[r], v);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kLogitRows; ++r) {
    const float m = warp_max(mx[r]);
    if ((tid & 31) == 0) smax[tid >> 5][r] = m;
  }
  __syncthreads();
  if (tid < kLogitRows && i0 + tid < c_q) {
    float m = smax[0][tid];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, smax[w][tid]);
    mref[(size_t)h * c_q + i0 + tid] = m;
  }
}

// ------------------------------------------------------------------------------------------------
// error table: one block per key cluster; thread <-> query cluster (q̄_i in registers); key tiles
// of 32 rows staged in shared memory as fp32 differences k_t - k̄_j.
// ------------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256, 1)
    error_table_kernel(int mode, const float* __restrict__ qc, const float* __restrict__ kc,
                       const float* __restrict__ vc, const bf16* __restrict__ kp,
                       const bf16* __restrict__ vp, const int32_t* __restrict__ q_sizes,
                       const int32_t* __restrict__ k_sizes, const int32_t* __restrict__ k_offsets,
                       const float* __restrict__ sbar, const float* __restrict__ mref, int n_k,
                       int c_q, int c_k, float scale, double* __restrict__ err) {
  constexpr int TK = 32;
  const int h = blockIdx.y, j = blockIdx.x;
  __shared__ float4 skd[TK][D / 4];  // k_t - k̄_j
  __shared__ float sA[TK], sB[TK], sC[TK];
  __shared__ float skb[D], svb[D];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nj = k_sizes[(size_t)h * c_k + j], o = k_offsets[(size_t)h * c_k + j];
  if (tid < D) {
    skb[tid] = kc[((size_t)h * c_k + j) * D + tid];
    svb[tid] = (mode == SVGEAR_EST_VALUE_AWARE) ? vc[((size_t)h * c_k + j) * D + tid] : 0.f;
  }
  __syncthreads();

  const int nthr = blockDim.x, nwarp = blockDim.x >> 5;
  for (int ibase = 0; ibase < c_q; ibase += nthr) {
    const int i = ibase + tid;
    const bool act = i < c_q;
    float qr[D];
    {
      const float4* qp = reinterpret_cast<const float4*>(qc + ((size_t)h * c_q + (act ? i : 0)) * D);
#pragma unroll
      for (int q = 0; q < D / 4; ++q) {
        float4 v = __ldg(qp + q);
        qr[4 * q] = v.x; qr[4 * q + 1] = v.y; qr[4 * q + 2] = v.z; qr[4 * q + 3] = v.w;
      }
    }
    float M = 0.f;    // running max(0, g)
    float acc = 0.f;  // sum at scale exp(-2M)
    for (int t0 = 0; t0 < nj; t0 += TK) {
      const int nt = min(TK, nj - t0);
      __syncthreads();
      // stage the tile: each warp takes rows warp, warp+8, ...; lanes split the row
      for (int r = warp; r < TK; r += nwarp) {
        float a = 0.f, b = 0.f, cc = 0.f;
        if (r < nt) {
          const size_t row = (size_t)h * n_k + o + t0 + r;
          constexpr int EPL = D / 32;
          float kf[EPL], vf[EPL];
          if (EPL == 4) {
            uint2 ku = __ldg(reinterpret_cast<const uint2*>(kp + row * D + lane * 4));
            kf[0] = __uint_as_float(ku.x << 16); kf[1] = __uint_as_float(ku.x & 0xffff0000u);
            kf[2] = __uint_as_float(ku.y << 16); kf[3] = __uint_as_float(ku.y & 0xffff0000u);
            if (mode == SVGEAR_EST_VALUE_AWARE) {
              uint2 vu = __ldg(reinterpret_cast<const uint2*>(vp + row * D + lane * 4));
              vf[0] = __uint_as_float(vu.x << 16); vf[1] = __uint_as_float(vu.x & 0xffff0000u);
              vf[2] = __uint_as_float(vu.y << 16); vf[3] = __uint_as_float(vu.y & 0xffff0000u);
            }
          } else {
            uint32_t ku = __ldg(reinterpret_cast<const uint32_t*>(kp + row * D + lane * 2));
            kf[0] = __uint_as_float(ku << 16); kf[1] = __uint_as_float(ku & 0xffff0000u);
            if (mode == SVGEAR_EST_VALUE_AWARE) {
              uint32_t vu = __ldg(reinterpret_cast<const uint32_t*>(vp + row * D + lane * 2));
              vf[0] = __uint_as_float(vu << 16); vf[1] = __uint_as_float(vu & 0xffff0000u);
            }
          }
          float* dst = reinterpret_cast<float*>(&skd[r][0]) + lane * EPL;
#pragma unroll
          for (int u = 0; u < EPL; ++u) {
            dst[u] = kf[u] - skb[lane * EPL + u];
            if (mode == SVGEAR_EST_VALUE_AWARE) {
              float dv = svb[lane * EPL + u] - vf[u];
              a = fmaf(dv, dv, a);
              b = fmaf(dv, vf[u], b);
              cc = fmaf(vf[u], vf[u], cc);
            }
          }
          a = warp_sum(a); b = warp_sum(b); cc = warp_sum(cc);
          if (mode != SVGEAR_EST_VALUE_AWARE) { a = 0.f; b = 0.f; cc = 1.f; }
        } else {
          float* dst = reinterpret_cast<float*>(&skd[r][0]) + lane * (D / 32);
#pragma unroll
          for (int u = 0; u < D / 32; ++u) dst[u] = 0.f;
        }
        if (lane == 0) { sA[r] = a; sB[r] = b; sC[r] = cc; }
      }
      __syncthreads();
      if (act) {
        for (int t = 0; t < nt; ++t) {
          float g0 = 0.f, g1 = 0.f;
#pragma unroll
          for (int q = 0; q < D / 4; q += 2) {
            float4 k0 = skd[t][q], k1 = skd[t][q + 1];
            g0 = fmaf(qr[4 * q], k0.x, g0); g0 = fmaf(qr[4 * q + 1], k0.y, g0);
            g0 = fmaf(qr[4 * q + 2], k0.z, g0); g0 = fmaf(qr[4 * q + 3], k0.w, g0);
            g1 = fmaf(qr[4 * q + 4], k1.x, g1); g1 = fmaf(qr[4 * q + 5], k1.y, g1);
            g1 = fmaf(qr[4 * q + 6], k1.z, g1); g1 = fmaf(qr[4 * q + 7], k1.w, g1);
          }
          const float g = (g0 + g1) * scale;
          if (g > M) {
            const float r = expf(M - g);
            acc *= r * r;
            M = g;
          }
          const float em = expf(-M);          // 1 when M == 0
          const float xs = (g < 20.f) ? expm1f(g) * em : (expf(g - M) - em);
          acc += (sA[t] * em) * em - 2.f * (em * xs) * sB[t] + (xs * xs) * sC[t];
        }
      }
    }
    if (act) {
      const size_t e = ((size_t)h * c_q + i) * c_k + j;
      const double lift = 2.0 * ((double)sbar[e] - (double)mref[(size_t)h * c_q + i] + (double)M);
      double v = (double)fmaxf(acc, 0.f) * exp(lift);
      err[e] = (double)q_sizes[(size_t)h * c_q + i] * v;
    }
  }
}

int launch_error_table_tc(const SvgEarShape& s, int mode, const float* qc, const float* kc, const float* vc,
                          const bf16* kp, const bf16* vp, const int32_t* q_sizes, const int32_t* k_sizes,
                          const int32_t* k_offsets, const float* sbar, const float* mref, bf16* kd_hi,
                          bf16* kd_lo, float* kstat, bf16* qsplit, double* err, bool key_stats_done,
                          cudaStream_t st);
int launch_key_stats(const SvgEarShape& s, int mode, const float* kc, const float* vc, const bf16* kp,
                     const bf16* vp, const int32_t* k_sizes, const int32_t* k_offsets, bf16* kd_hi, bf16* kd_lo,
                     float* kstat, cudaStream_t st);

// key-side half of the tensor-core estimator, for callers that overlap it with the query side
int launch_error_table_keys(const SvgEarShape& s, int mode, const float* kc, const float* vc, const bf16* kp,
                            const bf16* vp, const int32_t* k_sizes, const int32_t* k_offsets, ErrScratch& sc,
                            cudaStream_t st) {
  return launch_key_stats(s, mode, kc, vc, kp, vp, k_sizes, k_offsets, sc.kd_hi, sc.kd_lo, sc.kstat, st);
}

size_t errtab_stat_floats(const SvgEarShape& s);

bool ErrScratch::carve(Carver& cv, const SvgEarShape& s) {
  const int cqpad = ceil_div(s.c_q, 128) * 128;
  sbar = cv.take<float>((size_t)s.bh * s.c_q * s.c_k);
  kd_hi = cv.take<bf16>((size_t)s.bh * s.n_k * s.d);
  kd_lo = cv.take<bf16>((size_t)s.bh * s.n_k * s.d);
  kstat = cv.take<float>(errtab_stat_floats(s));  // planes A, -2B, C, clusters 16-byte aligned (errtab_tc.cu)
  qsplit = cv.take<bf16>((size_t)s.bh * 2 * cqpad * s.d);
  return cv.ok;
}

int launch_error_table(const SvgEarShape& s, int exec_mode, int mode, const float* qc, const float* kc,
                       const float* vc, const bf16* kp, const bf16* vp, const int32_t* q_sizes,
                       const int32_t* k_sizes, const int32_t* k_offsets, double* err,
                       float* stabilizers, ErrScratch& sc, cudaStream_t st, bool key_stats_done) {
  const float scale = 1.0f / sqrtf((float)s.d);
  float* sbar = sc.sbar;
  centroid_logits_kernel<<<dim3(ceil_div(s.c_q, kLogitRows), s.bh), 256, 0, st>>>(qc, kc, s.d, s.c_q, s.c_k, scale, sbar,
                                                           stabilizers);
  SVG_LAUNCH_OK();
  if (exec_mode == SVGEAR_EXEC_BF16_TENSOR)
    return launch_error_table_tc(s, mode, qc, kc, vc, kp, vp, q_sizes, k_sizes, k_offsets, sbar, stabilizers,
                                 sc.kd_hi, sc.kd_lo, sc.kstat, sc.qsplit, err, key_stats_done, st);
  const int passes = ceil_div(s.c_q, 256);
  const int thr = min(256, max(128, ceil_div(ceil_div(s.c_q, passes), 32) * 32));
  if (s.d == 128)
    error_table_kernel<128><<<dim3(s.c_k, s.bh), thr, 0, st>>>(
        mode, qc, kc, vc, kp, vp, q_sizes, k_sizes, k_offsets, sbar, stabilizers, s.n_k, s.c_q,
        s.c_k, scale, err);
  else
    error_table_kernel<64><<<dim3(s.c_k, s.bh), thr, 0, st>>>(
        mode, qc, kc, vc, kp, vp, q_sizes, k_sizes, k_offsets, sbar, stabilizers, s.n_k, s.c_q,
        s.c_k, scale, err);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

// ------------------------------------------------------------------------------------------------
// cluster mass for score routing: row softmax of s̄ + ln|k_c| in float64 (router.py:193-206,267)
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    score_mass_kernel(const float* __restrict__ qc, const float* __restrict__ kc,
                      const int32_t* __restrict__ k_sizes, int d, int c_q, int c_k, double scale,
                      double* __restrict__ mass) {
  const int h = blockIdx.y, i = blockIdx.x;
  __shared__ double sq[128];
  __shared__ double sred[8];
  __shared__ double s_bcast;
  const int tid = threadIdx.x;
  if (tid < d) sq[tid] = (double)qc[((size_t)h * c_q + i) * d + tid];
  __syncthreads();
  double* row = mass + ((size_t)h * c_q + i) * c_k;
  double mx = -INFINITY;
  for (int j = tid; j < c_k; j += 256) {
    const float* kp = kc + ((size_t)h * c_k + j) * d;
    double s = 0.0;
    for (int k = 0; k < d; ++k) s = fma(sq[k], (double)__ldg(kp + k), s);
    s = s * scale + log((double)k_sizes[(size_t)h * c_k + j]);
    row[j] = s;
    mx = fmax(mx, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) sred[tid >> 5] = mx;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 8; ++w) mx = fmax(mx, sred[w]);
    s_bcast = mx;
  }
  __syncthreads();
  mx = s_bcast;
  double sum = 0.0;
  for (int j = tid; j < c_k; j += 256) {
    double w = exp(row[j] - mx);
    row[j] = w;
    sum += w;
  }
  sum = warp_sum(sum);
  __syncthreads();
  if ((tid & 31) == 0) sred[tid >> 5] = sum;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sred[w];
    s_bcast = s;
  }
  __syncthreads();
  sum = s_bcast;
  for (int j = tid; j < c_k; j += 256) row[j] = row[j] / sum;
}

int launch_score_mass(const SvgEarShape& s, const float* qc, const float* kc,
                      const int32_t* k_sizes, double* mass, cudaStream_t st) {
  score_mass_kernel<<<dim3(s.c_q, s.bh), 256, 0, st>>>(qc, kc, k_sizes, s.d, s.c_q, s.c_k,
                                                      1.0 / sqrt((double)s.d), mass);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

// ------------------------------------------------------------------------------------------------
// routing: exact greedy walk without a sort.
//
// Walk order = descending priority P(b) = (ord(primary_b), ord(value_b), ~b) compared
// lexicographically, where primary = value/(|q||k|) for error-aware routing (ratio_mode 0) or
// primary = value for mass routing (ratio_mode 1), and ord() is the order-preserving map of a
// float64 onto uint64.  Because the index is part of the key the order is total, exactly the
// reference's sort key (-ratio, -error, qc, kc).
//   phase 1  MSD radix select on P with weighted (block-size) histograms finds the first block
//            that does not fit = end of the "take while it fits" prefix;
//   phase 2  fillRemainder: repeatedly take the highest-priority block after the cursor whose
//            weight still fits (block-wide lexicographic arg-max), until none fits;
//   phase 3  best-single-fitting-block fallback.
// One thread-block CLUSTER per instance (the scans are issue bound, so a single CTA per instance left
// the kernel at ~1 SM per head): every CTA scans its slice of the blocks into a local histogram, the
// non-empty bins are merged into rank 0's totals through distributed shared memory, rank 0 picks the
// digit and broadcasts it.  Integer atomics only.
// ------------------------------------------------------------------------------------------------
struct Prio {
  unsigned long long a;  // ord64(primary key)
  unsigned int c;        // ~block index   (the secondary key ord64(value) is fetched on demand)
};
__device__ __forceinline__ unsigned long long ord64(double v) {
  unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
// Radix-select digit schedule over the 160-bit key (a:64 | b:64 | c:32), most significant first,
// 11-bit digits: a -> 6 passes, b -> 6 passes, c -> 3 passes.
constexpr int kRouteBins = 2048;
constexpr int kRoutePasses = 15;
constexpr int kRouteMaxCluster = 8;
__device__ __forceinline__ void pass_geom(int pass, int& field, int& shift, int& width) {
  if (pass < 12) {
    field = pass / 6;
    const int q = pass % 6;
    shift = q < 5 ? 53 - 11 * q : 0;
    width = q < 5 ? 11 : 9;
  } else {
    field = 2;
    const int q = pass - 12;
    shift = q == 0 ? 21 : (q == 1 ? 10 : 0);
    width = q == 2 ? 10 : 11;
  }
}

// primary keys, computed once by the whole grid (the float64 division is the expensive part)
__global__ void route_keys_kernel(const double* __restrict__ val, const int32_t* __restrict__ q_sizes,
                                  const int32_t* __restrict__ k_sizes, int c_q, int c_k, int ratio_mode,
                                  unsigned long long* __restrict__ keys) {
  const int h = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= c_q * c_k) return;
  const double v = val[(size_t)h * c_q * c_k + b];
  double key = v;
  if (ratio_mode == 0) {
    const long long w = (long long)q_sizes[(size_t)h * c_q + b / c_k] * (long long)k_sizes[(size_t)h * c_k + b % c_k];
    key = v / (double)w;
  }
  keys[(size_t)h * c_q * c_k + b] = ord64(key);
}

__global__ void __launch_bounds__(1024)
    route_kernel(int c_q, int c_k, const double* __restrict__ val_all,
                 const unsigned long long* __restrict__ keys_all, const int32_t* __restrict__ q_sizes_all,
                 const int32_t* __restrict__ k_sizes_all, long long capacity, int overshoot, int fallback,
                 uint8_t* __restrict__ mask_all, long long* __restrict__ entries_all, int pieces,
                 int piece_bits) {
  cg::cluster_group cluster = cg::this_cluster();
  const int R = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int h = blockIdx.x / R;
  const int nb = c_q * c_k;
  const double* val = val_all + (size_t)h * nb;
  const unsigned long long* keys = keys_all + (size_t)h * nb;
  const int32_t* qs = q_sizes_all + (size_t)h * c_q;
  uint8_t* mask = mask_all + (size_t)h * nb;
  // Weighted histograms use native 32-bit shared atomics: a block weight (up to 34 bits) is split
  // into `pieces` fields of `piece_bits` bits, each summed in its own counter array (64-bit shared
  // atomics compile to CAS loops and dominated this kernel).
  extern __shared__ int32_t s_dyn[];
  int32_t* s_ks = s_dyn;                                                        // [c_k]
  unsigned int* s_hc = reinterpret_cast<unsigned int*>(s_dyn + ((c_k + 3) & ~3));  // [bins]
  unsigned int* s_hp = s_hc + kRouteBins;                                         // [pieces][bins]
  // cluster totals (live on rank 0; with one CTA per instance the local arrays are the totals)
  unsigned int* s_tc = R > 1 ? s_hp + pieces * kRouteBins : s_hc;                 // [bins]
  unsigned int* s_tp = s_tc + kRouteBins;                                         // [pieces][bins]
  auto bin_weight = [&](int dg) -> unsigned long long {
    unsigned long long t = 0;
    for (int q = 0; q < pieces; ++q) t += (unsigned long long)s_tp[q * kRouteBins + dg] << (q * piece_bits);
    return t;
  };
  auto bin_add = [&](unsigned int dg, unsigned long long wsum, unsigned int cnt) {
    const unsigned long long m = (1ull << piece_bits) - 1ull;
    for (int q = 0; q < pieces; ++q) {
      const unsigned int part = (unsigned int)((wsum >> (q * piece_bits)) & m);
      if (part) atomicAdd(&s_hp[q * kRouteBins + dg], part);
    }
    atomicAdd(&s_hc[dg], cnt);
  };
  __shared__ unsigned long long s_pa, s_pb;  // digits chosen so far (others zero)
  __shared__ unsigned int s_pc;
  __shared__ Prio s_red[32];
  __shared__ long long s_redw[32];
  __shared__ double s_redd[32];
  __shared__ long long s_base;
  __shared__ int s_flag;
  // per-CTA partial results collected on rank 0 (phase 2 double-buffered by iteration parity)
  __shared__ Prio s_cbest[2][kRouteMaxCluster];
  __shared__ long long s_cbw[2][kRouteMaxCluster];
  __shared__ double s_csum[kRouteMaxCluster], s_cbv[kRouteMaxCluster];
  __shared__ long long s_cent[kRouteMaxCluster];
  __shared__ int s_cbi[kRouteMaxCluster];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x;
  const int gtid = rank * nthr + tid, gthr = R * nthr;  // this thread's slot among the cluster's threads
  for (int j = tid; j < c_k; j += nthr) s_ks[j] = k_sizes_all[(size_t)h * c_k + j];
  if (tid == 0) { s_pa = 0; s_pb = 0; s_pc = 0; s_base = 0; s_flag = 0; }
  __syncthreads();

  auto getb = [&](unsigned int c) -> unsigned long long { return ord64(val[~c]); };
  auto pgt = [&](const Prio& x, const Prio& y) -> bool {  // x strictly earlier in the walk than y
    if (x.a != y.a) return x.a > y.a;
    if (x.c == y.c) return false;
    const unsigned long long xb = getb(x.c), yb = getb(y.c);
    if (xb != yb) return xb > yb;
    return x.c > y.c;
  };
  // iterate this thread's blocks b = gtid, gtid + gthr, ... keeping (row, col) incrementally
#define FOR_BLOCKS(BODY)                                             \
  {                                                                  \
    int qi_ = gtid / c_k, kj_ = gtid % c_k;                          \
    const int dq_ = gthr / c_k, dk_ = gthr % c_k;                    \
    for (int b = gtid; b < nb; b += gthr) {                          \
      const long long w = (long long)qs[qi_] * (long long)s_ks[kj_]; \
      BODY                                                           \
      qi_ += dq_; kj_ += dk_;                                        \
      if (kj_ >= c_k) { kj_ -= c_k; ++qi_; }                         \
    }                                                                \
  }

  // ---- phase 1: first block that does not fit ---------------------------------------------------
  bool all_fit = false;
  int last_field = 0, last_shift = 64;
  for (int pass = 0; pass < kRoutePasses; ++pass) {
    int field, shift, width;
    pass_geom(pass, field, shift, width);
    for (int k = tid; k < kRouteBins * (pieces + 1); k += nthr) s_hc[k] = 0u;  // counts + all pieces
    if (R > 1 && rank == 0)
      for (int k = tid; k < kRouteBins * (pieces + 1); k += nthr) s_tc[k] = 0u;
    cluster.sync();  // totals are zero before any CTA merges into them
    const unsigned long long pa = s_pa, pb = s_pb;
    const unsigned int pc = s_pc;
    const int hs = shift + width;
    {
      // run-length accumulation: consecutive candidates usually share the digit in the top passes
      unsigned int rd = 0xffffffffu, rc = 0;
      unsigned long long rw = 0;
      FOR_BLOCKS({
        const unsigned long long ka = keys[b];
        bool cand;
        unsigned int dg;
        if (field == 0) {
          cand = hs >= 64 ? true : (ka >> hs) == (pa >> hs);
          dg = (unsigned int)(ka >> shift) & ((1u << width) - 1u);
        } else if (ka != pa) {
          cand = false; dg = 0;
        } else {
          const unsigned long long kb = getb(~(unsigned int)b);
          if (field == 1) {
            cand = hs >= 64 ? true : (kb >> hs) == (pb >> hs);
            dg = (unsigned int)(kb >> shift) & ((1u << width) - 1u);
          } else {
            const unsigned int kc = ~(unsigned int)b;
            cand = kb == pb && (hs >= 32 ? true : (kc >> hs) == (pc >> hs));
            dg = (kc >> shift) & ((1u << width) - 1u);
          }
        }
        if (cand) {
          // a run is flushed when the digit changes or before a piece field could overflow
          if (dg != rd || rc >= 64u) {
            if (rc) bin_add(rd, rw, rc);
            rd = dg; rw = 0; rc = 0;
          }
          rw += (unsigned long long)w;
          rc += 1;
        }
      })
      if (rc) bin_add(rd, rw, rc);
    }
    __syncthreads();
    if (R > 1) {  // merge the non-empty local bins into rank 0's totals
      unsigned int* t0 = cluster.map_shared_rank(s_tc, 0);
      for (int k = tid; k < kRouteBins * (pieces + 1); k += nthr) {
        const unsigned int x = s_hc[k];
        if (x) atomicAdd(t0 + k, x);
      }
      cluster.sync();
    }
    if (rank == 0 && warp == 0) {
      // first bin (from the top) where the running weight exceeds the capacity: each lane owns 64
      // consecutive bins, lane 0 the highest
      const int nbins = 1 << width;
      const int per = kRouteBins / 32;
      const int hi = nbins - 1 - lane * per;
      unsigned long long mine = 0;
      for (int q = 0; q < per; ++q) {
        const int dg = hi - q;
        if (dg >= 0) mine += bin_weight(dg);
      }
      unsigned long long inc = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const long long base0 = s_base;
      const bool crosses = base0 + (long long)inc > capacity;
      const unsigned bal = __ballot_sync(0xffffffffu, crosses);
      const unsigned long long group_total = __shfl_sync(0xffffffffu, inc, 31);
      if (bal == 0) {
        if (lane == 0) { s_flag = 1; s_base = base0 + (long long)group_total; }
      } else {
        const int owner = __ffs(bal) - 1;
        if (lane == owner) {
          long long run = base0 + (long long)(inc - mine);
          int found = -1;
          for (int q = 0; q < per; ++q) {
            const int dg = hi - q;
            if (dg < 0) break;
            if (s_tc[dg] == 0) continue;
            const long long bwt = (long long)bin_weight(dg);
            if (run + bwt > capacity) { found = dg; break; }
            run += bwt;
          }
          s_base = run;
          if (field == 0) s_pa |= (unsigned long long)found << shift;
          else if (field == 1) s_pb |= (unsigned long long)found << shift;
          else s_pc |= (unsigned int)found << shift;
          s_flag = (s_tc[found] == 1) ? 2 : 0;  // unique candidate -> it is the boundary block
        }
      }
      __syncwarp();
      if (lane == 0)
        for (int r = 1; r < R; ++r) {  // broadcast the decision
          *cluster.map_shared_rank(&s_pa, r) = s_pa;
          *cluster.map_shared_rank(&s_pb, r) = s_pb;
          *cluster.map_shared_rank(&s_pc, r) = s_pc;
          *cluster.map_shared_rank(&s_base, r) = s_base;
          *cluster.map_shared_rank(&s_flag, r) = s_flag;
        }
    }
    cluster.sync();
    last_field = field; last_shift = shift;
    if (s_flag == 1) { all_fit = true; break; }
    if (s_flag == 2) break;
  }
  // locate the boundary block (the unique element matching every chosen digit)
  Prio bound;
  bound.a = 0; bound.c = 0;
  long long remaining = capacity - s_base;
  __syncthreads();
  if (!all_fit) {
    const unsigned long long pa = s_pa, pb = s_pb;
    const unsigned int pc = s_pc;
    FOR_BLOCKS({
      const unsigned long long ka = keys[b];
      bool hit;
      if (last_field == 0) hit = (ka >> last_shift) == (pa >> last_shift);
      else if (ka != pa) hit = false;
      else {
        const unsigned long long kb = getb(~(unsigned int)b);
        if (last_field == 1) hit = (kb >> last_shift) == (pb >> last_shift);
        else hit = kb == pb && ((~(unsigned int)b) >> last_shift) == (pc >> last_shift);
      }
      if (hit)  // exactly one writer in the cluster
        for (int r = 0; r < R; ++r) {
          Prio* dst = cluster.map_shared_rank(&s_red[0], r);
          dst->a = ka; dst->c = ~(unsigned int)b;
        }
      (void)w;
    })
    cluster.sync();
    bound = s_red[0];
  }
  __syncthreads();
  // ---- mask of the prefix -------------------------------------------------------------------------
  FOR_BLOCKS({
    Prio p; p.a = keys[b]; p.c = ~(unsigned int)b;
    mask[b] = all_fit ? 1 : (pgt(p, bound) ? 1 : 0);
    (void)w;
  })
  // ---- phase 2: fillRemainder tail ------------------------------------------------------------------
  if (!all_fit && overshoot == SVGEAR_FILL_REMAINDER) {
    Prio cur = bound;
    for (int it = 0;; ++it) {
      Prio best;
      best.a = 0; best.c = 0;
      long long bw = 0;
      FOR_BLOCKS({
        if (w <= remaining) {
          Prio p; p.a = keys[b]; p.c = ~(unsigned int)b;
          if (pgt(cur, p) && (best.a == 0 || pgt(p, best))) { best = p; bw = w; }
        }
      })
      // block arg-max (a == 0 marks "none": ord64 of a non-negative key always has the top bit set)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Prio q;
        q.a = __shfl_xor_sync(0xffffffffu, best.a, o);
        q.c = __shfl_xor_sync(0xffffffffu, best.c, o);
        const long long qw = __shfl_xor_sync(0xffffffffu, bw, o);
        if (q.a != 0 && (best.a == 0 || pgt(q, best))) { best = q; bw = qw; }
      }
      __syncthreads();
      if (lane == 0) { s_red[warp] = best; s_redw[warp] = bw; }
      __syncthreads();
      if (warp == 0) {
        const int nw = nthr >> 5;
        Prio q = s_red[lane < nw ? lane : 0];
        long long qw = s_redw[lane < nw ? lane : 0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          Prio r;
          r.a = __shfl_xor_sync(0xffffffffu, q.a, o);
          r.c = __shfl_xor_sync(0xffffffffu, q.c, o);
          const long long rw = __shfl_xor_sync(0xffffffffu, qw, o);
          if (r.a != 0 && (q.a == 0 || pgt(r, q))) { q = r; qw = rw; }
        }
        if (lane == 0) {  // this CTA's candidate -> rank 0
          *cluster.map_shared_rank(&s_cbest[it & 1][rank], 0) = q;
          *cluster.map_shared_rank(&s_cbw[it & 1][rank], 0) = qw;
        }
      }
      cluster.sync();
      {  // every thread reduces the R candidates in rank order (same result everywhere)
        const Prio* cb = cluster.map_shared_rank(&s_cbest[it & 1][0], 0);
        const long long* cw = cluster.map_shared_rank(&s_cbw[it & 1][0], 0);
        best = cb[0];
        bw = cw[0];
        for (int r = 1; r < R; ++r) {
          const Prio q = cb[r];
          if (q.a != 0 && (best.a == 0 || pgt(q, best))) { best = q; bw = cw[r]; }
        }
      }
      if (best.a == 0) break;  // nothing fits any more
      if (gtid == 0) mask[~best.c] = 1;
      remaining -= bw;
      cur = best;
      __syncthreads();
    }
  }
  cluster.sync();  // rank 0's tail writes to the mask are visible to the whole cluster
  // ---- phase 3: single-item fallback + entry count ----------------------------------------------
  double sum_sel = 0.0;
  long long ent = 0;
  double bestv = -INFINITY;
  int besti = 0x7fffffff;
  FOR_BLOCKS({
    const bool sel = mask[b] != 0;
    if (sel) ent += w;
    if (fallback) {
      const double v = val[b];
      if (sel) sum_sel += v;
      if (w <= capacity && v > bestv) { bestv = v; besti = b; }
    }
  })
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum_sel += __shfl_xor_sync(0xffffffffu, sum_sel, o);
    ent += __shfl_xor_sync(0xffffffffu, ent, o);
    double ov = __shfl_xor_sync(0xffffffffu, bestv, o);
    int oi = __shfl_xor_sync(0xffffffffu, besti, o);
    if (ov > bestv || (ov == bestv && oi < besti)) { bestv = ov; besti = oi; }
  }
  if (lane == 0) {
    s_redd[warp] = sum_sel;
    s_redw[warp] = ent;
    s_red[warp].a = (unsigned long long)__double_as_longlong(bestv);
    s_red[warp].c = (unsigned int)besti;
  }
  __syncthreads();
  if (tid == 0) {  // this CTA's partial results -> rank 0
    const int nw = nthr >> 5;
    double s = 0.0;
    long long e = 0;
    double bv = -INFINITY;
    int bx = 0x7fffffff;
    for (int w2 = 0; w2 < nw; ++w2) {
      s += s_redd[w2];
      e += s_redw[w2];
      double ov = __longlong_as_double((long long)s_red[w2].a);
      int oi = (int)s_red[w2].c;
      if (ov > bv || (ov == bv && oi < bx)) { bv = ov; bx = oi; }
    }
    *cluster.map_shared_rank(&s_csum[rank], 0) = s;
    *cluster.map_shared_rank(&s_cent[rank], 0) = e;
    *cluster.map_shared_rank(&s_cbv[rank], 0) = bv;
    *cluster.map_shared_rank(&s_cbi[rank], 0) = bx;
  }
  cluster.sync();
  if (rank == 0 && tid == 0) {
    double s = 0.0;
    long long e = 0;
    double bv = -INFINITY;
    int bx = 0x7fffffff;
    for (int r = 0; r < R; ++r) {
      s += s_csum[r];
      e += s_cent[r];
      if (s_cbv[r] > bv || (s_cbv[r] == bv && s_cbi[r] < bx)) { bv = s_cbv[r]; bx = s_cbi[r]; }
    }
    int swap = (fallback && bx != 0x7fffffff && bv > s) ? 1 : 0;
    if (entries_all)
      entries_all[h] = swap ? (long long)qs[bx / c_k] * (long long)s_ks[bx % c_k] : e;
    for (int r = 0; r < R; ++r) {
      *cluster.map_shared_rank(&s_flag, r) = swap;
      *cluster.map_shared_rank(&s_base, r) = swap ? (long long)bx : -1;
    }
  }
  cluster.sync();
  if (s_flag) {
    const int keep = (int)s_base;
    for (int b = gtid; b < nb; b += gthr) mask[b] = (b == keep) ? 1 : 0;
  }
#undef FOR_BLOCKS
}

// ------------------------------------------------------------------------------------------------
// perClusterTopP routing (router.py:172-190 with score_top_p_budget, router.py:209-250): every
// query-cluster row gets its own entry budget — the entries of the minimal set of key clusters whose
// softmax mass reaches p — and spends it with the same greedy error-to-cost walk + single-block
// fallback, restricted to the row.  One CTA per (row, instance): two bitonic sorts of the row in
// shared memory (mass order, then (-ratio, -error, index) order), and an exact sequential walk by
// one thread (cumulative sums in the reference's left-to-right order).
// ------------------------------------------------------------------------------------------------
struct TopPKey {
  double a;  // primary, descending
  double b;  // secondary, descending
  int idx;   // tertiary, ascending (padding: INT_MAX)
};
__device__ __forceinline__ bool topp_before(const TopPKey& x, const TopPKey& y) {
  if (x.a != y.a) return x.a > y.a;
  if (x.b != y.b) return x.b > y.b;
  return x.idx < y.idx;
}
__device__ void topp_sort(TopPKey* keys, int npad) {
  for (int k = 2; k <= npad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          TopPKey x = keys[i], y = keys[l];
          if (topp_before(y, x) == up) { keys[i] = y; keys[l] = x; }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256)
    route_top_p_kernel(const double* __restrict__ err, const double* __restrict__ mass,
                       const int32_t* __restrict__ q_sizes, const int32_t* __restrict__ k_sizes, int c_q,
                       int c_k, int npad, double p, int overshoot, int fallback,
                       uint8_t* __restrict__ mask, unsigned long long* __restrict__ entries) {
  extern __shared__ __align__(16) unsigned char topp_smem[];
  TopPKey* keys = reinterpret_cast<TopPKey*>(topp_smem);
  __shared__ long long s_cap;
  __shared__ int s_single;  // fallback block (or -1)
  const int h = blockIdx.y, i = blockIdx.x, tid = threadIdx.x;
  const double* erow = err + ((size_t)h * c_q + i) * c_k;
  const double* mrow = mass + ((size_t)h * c_q + i) * c_k;
  const int32_t* ks = k_sizes + (size_t)h * c_k;
  const long long qs = q_sizes[(size_t)h * c_q + i];
  uint8_t* out = mask + ((size_t)h * c_q + i) * c_k;
  // ---- (1) row budget: minimal mass prefix reaching p (router.py:225-236) -------------------------
  for (int j = tid; j < npad; j += 256) {
    TopPKey k;
    k.a = j < c_k ? mrow[j] : -INFINITY;
    k.b = 0.0;
    k.idx = j < c_k ? j : 0x7fffffff;
    keys[j] = k;
  }
  __syncthreads();
  topp_sort(keys, npad);
  if (tid == 0) {
    long long cap = 0;
    if (p >= 1.0) {
      for (int j = 0; j < c_k; ++j) cap += qs * ks[j];
    } else {
      double cum = 0.0;
      int cut = c_k;  // searchsorted(cumsum, p, side="left"): first position with cumsum >= p
      for (int r = 0; r < c_k; ++r) {
        cum += keys[r].a;
        if (cum >= p) { cut = r; break; }
      }
      const int last = min(cut, c_k - 1);
      for (int r = 0; r <= last; ++r) cap += qs * ks[keys[r].idx];
      s_single = last;
    }
    s_cap = cap;
    s_single = min(c_k - 1, p >= 1.0 ? c_k - 1 : s_single);
  }
  __syncthreads();
  if (err == nullptr) {
    // score_top_p as a policy of its own (router.py:209-236): the prefix itself is the mask
    const int last = s_single;
    for (int j = tid; j < c_k; j += 256) out[j] = 0;
    __syncthreads();
    for (int r = tid; r <= last; r += 256) out[keys[r].idx] = 1;
    if (tid == 0 && entries) atomicAdd(&entries[h], (unsigned long long)s_cap);
    return;
  }
  // ---- (2) row order (-ratio, -error, index) (estimator.py:83-96 restricted to the row) ------------
  for (int j = tid; j < npad; j += 256) {
    TopPKey k;
    if (j < c_k) {
      const double e = erow[j];
      k.a = e / (double)(qs * ks[j]);
      k.b = e;
      k.idx = j;
    } else {
      k.a = -INFINITY;
      k.b = -INFINITY;
      k.idx = 0x7fffffff;
    }
    keys[j] = k;
  }
  for (int j = tid; j < c_k; j += 256) out[j] = 0;
  __syncthreads();
  topp_sort(keys, npad);
  // ---- (3) greedy walk + single-block fallback (router.py:100-121), one thread ---------------------
  if (tid == 0) {
    const long long cap = s_cap;
    long long left = cap;
    double total = 0.0;
    int ntake = 0;
    for (int r = 0; r < c_k; ++r) {
      const int j = keys[r].idx;
      const long long w = qs * ks[j];
      if (w <= left) {
        left -= w;
        total += keys[r].b;
        keys[r].idx = j | 0x40000000;  // mark taken
        ++ntake;
      } else if (overshoot == SVGEAR_STOP_AT_FIRST_OVERFLOW) {
        break;
      }
    }
    int single = -1;
    if (fallback) {
      double best = 0.0;
      int bj = -1;
      for (int j = 0; j < c_k; ++j) {  // first maximum in index order among the blocks that fit
        if (qs * ks[j] <= cap) {
          const double e = erow[j];
          if (bj < 0 || e > best) { best = e; bj = j; }
        }
      }
      if (bj >= 0 && best > total) single = bj;
    }
    s_single = single;
    unsigned long long ent = 0;
    if (single >= 0) {
      out[single] = 1;
      ent = (unsigned long long)(qs * ks[single]);
    } else {
      ent = (unsigned long long)(cap - left);
    }
    if (entries) atomicAdd(&entries[h], ent);
    (void)ntake;
  }
  __syncthreads();
  if (s_single < 0) {
    for (int r = tid; r < c_k; r += 256)
      if (keys[r].idx & 0x40000000) out[keys[r].idx & 0x3fffffff] = 1;
  }
}

int launch_route_top_p(const SvgEarShape& s, const double* err, const double* mass, const int32_t* q_sizes,
                       const int32_t* k_sizes, double p, int overshoot, int fallback, uint8_t* mask,
                       int64_t* entries, cudaStream_t st) {
  int npad = 1;
  while (npad < s.c_k) npad <<= 1;
  const size_t smem = (size_t)npad * sizeof(TopPKey);
  if (smem > 200 * 1024) return SVGEAR_EUNSUPPORTED;
  if (entries) SVG_CUDA_OK(cudaMemsetAsync(entries, 0, (size_t)s.bh * sizeof(int64_t), st));
  SVG_CUDA_OK(cudaFuncSetAttribute(route_top_p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  route_top_p_kernel<<<dim3(s.c_q, s.bh), 256, smem, st>>>(err, mass, q_sizes, k_sizes, s.c_q, s.c_k, npad, p,
                                                          overshoot, fallback, mask,
                                                          (unsigned long long*)entries);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

int launch_route(int bh, int c_q, int c_k, const double* val, const int32_t* q_sizes,
                 const int32_t* k_sizes, int64_t capacity, int overshoot, int fallback,
                 int ratio_mode, uint8_t* mask, int64_t* entries, unsigned long long* keys,
                 cudaStream_t st) {
  route_keys_kernel<<<dim3(ceil_div(c_q * c_k, 256), bh), 256, 0, st>>>(val, q_sizes, k_sizes, c_q, c_k,
                                                                      ratio_mode, keys);
  SVG_LAUNCH_OK();
  // piece_bits: every counter receives at most nb partial sums of < 2^piece_bits ... but a flushed
  // run holds up to 64 blocks, so a field sum stays below 2^32 when nb * 2^piece_bits <= 2^32
  int lg = 0;
  while ((1ll << lg) < (long long)c_q * c_k) ++lg;
  int piece_bits = 31 - lg;
  if (piece_bits > 17) piece_bits = 17;
  if (piece_bits < 6) return SVGEAR_EUNSUPPORTED;
  const int pieces = (40 + piece_bits - 1) / piece_bits;  // run sums: 34-bit weights x 64 blocks
  // CTAs per instance: one for small tables, otherwise the largest cluster size for which every
  // instance's cluster is co-resident (a 1024-thread CTA of this kernel owns an SM's registers, and
  // clusters do not straddle GPCs, so the driver is asked rather than assuming 148 / bh)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(1024);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SVG_CUDA_OK(cudaFuncSetAttribute(
      route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)(((size_t)((c_k + 3) & ~3) + (size_t)kRouteBins * (pieces + 1) * 2) * sizeof(int32_t))));
  int cluster = 1;
  if ((long long)c_q * c_k > 16384) {
    for (int r = kRouteMaxCluster; r > 1; --r) {
      cfg.gridDim = dim3(bh * r);
      cfg.dynamicSmemBytes = ((size_t)((c_k + 3) & ~3) + (size_t)kRouteBins * (pieces + 1) * 2) * sizeof(int32_t);
      attr[0].val.clusterDim.x = r;
      int fit = 0;
      if (cudaOccupancyMaxActiveClusters(&fit, route_kernel, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        continue;
      }
      if (fit >= bh) { cluster = r; break; }
    }
  }
  const size_t smem = ((size_t)((c_k + 3) & ~3) + (size_t)kRouteBins * (pieces + 1) * (cluster > 1 ? 2 : 1)) * sizeof(int32_t);
  cfg.gridDim = dim3(bh * cluster);
  cfg.dynamicSmemBytes = smem;
  attr[0].val.clusterDim.x = cluster;
  SVG_CUDA_OK(cudaLaunchKernelEx(&cfg, route_kernel, c_q, c_k, val, (const unsigned long long*)keys, q_sizes, k_sizes,
                                 (long long)capacity, overshoot, fallback, mask,
                                 reinterpret_cast<long long*>(entries), pieces, piece_bits));
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // namespace svg
