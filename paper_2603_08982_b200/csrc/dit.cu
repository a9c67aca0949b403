// The callers either side of the operator inside a DiT attention block (
// PAPER.md:398, :766): between the fused QKV projection and svgear_forward, and between
// svgear_forward and the output projection.  Both kernels are pure HBM streaming (one read and one
// write of every element); the projections themselves are plain library GEMMs on the caller's side.
//
//   qkv_prologue_kernel : [b][s][3][h][d] bf16 -> q, k, v [b][h][s][d] bf16 with RMSNorm of q and k
//                         (per head or over all heads of a token) and rotary embedding fused;
//                         one CTA per token, fp32 arithmetic, one rounding at the store.
//   heads_to_tokens_kernel : [b][h][s][d] -> [b][s][h][d] (what the output projection reads).
#include "common.cuh"

namespace svg {
namespace {

constexpr int kProThreads = 256;
constexpr int kProMaxChunks = 4;  // 16-byte chunks per thread per operand: h*d <= 8192
constexpr int kProTokens = 8;     // consecutive tokens per CTA (norm weights staged once per CTA)

// NORM: 0 none, 1 per head (over d), 2 over the whole token (h*d).  ROPE: 0 none, 1 interleaved
// pairs (x[2i], x[2i+1]), 2 half split (x[i], x[i+d/2]).
// A CTA handles kProTokens consecutive tokens, one at a time: the norm weights (2*h*d floats, as
// many bytes as a token's q and k) are staged in shared memory once per CTA instead of being
// fetched from L2 for every token — with per-token fetches the kernel ran at 60 % of the HBM rate
// of its norm-free instantiation.
template <int D, int NORM, int ROPE, int CH>  // CH = 16-byte chunks per thread per operand
__global__ void __launch_bounds__(kProThreads, 3)
qkv_prologue_kernel(const bf16* __restrict__ qkv, int tokens, int s, int h, const float* __restrict__ wq,
                    const float* __restrict__ wk, float eps, int rope_len,
                    const float* __restrict__ rope_cos, const float* __restrict__ rope_sin,
                    bf16* __restrict__ q, bf16* __restrict__ k, bf16* __restrict__ v) {
  constexpr int CPH = D / 8;  // chunks per head row
  extern __shared__ float4 s_w[];  // [2][h*D/4] when NORM != 0
  __shared__ float red2[2][2][kProThreads / 32];
  const int chunks = h * CPH;
  const int cc = threadIdx.x % CPH;  // chunk inside the head row (same for every i: 256 % CPH == 0)
  if (NORM != 0) {
    for (int e = threadIdx.x; e < 2 * chunks; e += kProThreads) {
      s_w[e] = __ldg(reinterpret_cast<const float4*>(wq) + e);
      s_w[2 * chunks + e] = __ldg(reinterpret_cast<const float4*>(wk) + e);
    }
    __syncthreads();
  }
  const int tok0 = blockIdx.x * kProTokens;
  const int tok1 = min(tok0 + kProTokens, tokens);
  for (int tok = tok0; tok < tok1; ++tok) {
    const int sidx = tok % s, bidx = tok / s;
    const uint4* row = reinterpret_cast<const uint4*>(qkv) + (size_t)tok * 3 * chunks;
    // every load of the token (q, k and v chunks) is issued before the first use
    uint4 raw[3][CH];
#pragma unroll
    for (int op = 0; op < 3; ++op)
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int c = threadIdx.x + i * kProThreads;
        raw[op][i] = c < chunks ? __ldg(row + op * chunks + c) : make_uint4(0u, 0u, 0u, 0u);
      }
    const bool rotate = ROPE != 0 && sidx < rope_len;
    float cs[8], sn[8];  // per-element rotation factors of this thread's chunk position
    if (rotate) {
      const float* ct = rope_cos + (size_t)sidx * (D / 2);
      const float* st = rope_sin + (size_t)sidx * (D / 2);
      if (ROPE == 1) {
        const float4 c4 = __ldg(reinterpret_cast<const float4*>(ct + cc * 4));
        const float4 s4 = __ldg(reinterpret_cast<const float4*>(st + cc * 4));
        cs[0] = cs[1] = c4.x; cs[2] = cs[3] = c4.y; cs[4] = cs[5] = c4.z; cs[6] = cs[7] = c4.w;
        sn[0] = -s4.x; sn[1] = s4.x; sn[2] = -s4.y; sn[3] = s4.y;
        sn[4] = -s4.z; sn[5] = s4.z; sn[6] = -s4.w; sn[7] = s4.w;
      } else {
        const int f = (cc * 8) % (D / 2);
        const float sign = (cc * 8 < D / 2) ? -1.f : 1.f;
        const float4 c0 = __ldg(reinterpret_cast<const float4*>(ct + f));
        const float4 c1 = __ldg(reinterpret_cast<const float4*>(ct + f + 4));
        const float4 s0 = __ldg(reinterpret_cast<const float4*>(st + f));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(st + f + 4));
        cs[0] = c0.x; cs[1] = c0.y; cs[2] = c0.z; cs[3] = c0.w;
        cs[4] = c1.x; cs[5] = c1.y; cs[6] = c1.z; cs[7] = c1.w;
        sn[0] = sign * s0.x; sn[1] = sign * s0.y; sn[2] = sign * s0.z; sn[3] = sign * s0.w;
        sn[4] = sign * s1.x; sn[5] = sign * s1.y; sn[6] = sign * s1.z; sn[7] = sign * s1.w;
      }
    }
    // v: layout change only
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int c = threadIdx.x + i * kProThreads;
      if (c < chunks)
        *reinterpret_cast<uint4*>(v + (((size_t)bidx * h + c / CPH) * s + sidx) * D + cc * 8) = raw[2][i];
    }
    float ss[2][CH];
    float total[2] = {0.f, 0.f};
    if (NORM != 0) {
#pragma unroll
      for (int op = 0; op < 2; ++op)
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          float f[8];
          unpack8(raw[op][i], f);
          float a = 0.f;
#pragma unroll
          for (int t = 0; t < 8; ++t) a += f[t] * f[t];
          ss[op][i] = a;
        }
      if (NORM == 2) {  // one block-wide reduction for both operands (buffers alternate per token)
        float mq = 0.f, mk = 0.f;
#pragma unroll
        for (int i = 0; i < CH; ++i) { mq += ss[0][i]; mk += ss[1][i]; }
        mq = warp_sum(mq);
        mk = warp_sum(mk);
        float(*rd)[kProThreads / 32] = red2[(tok - tok0) & 1];
        if ((threadIdx.x & 31) == 0) { rd[0][threadIdx.x >> 5] = mq; rd[1][threadIdx.x >> 5] = mk; }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kProThreads / 32; ++i) { total[0] += rd[0][i]; total[1] += rd[1][i]; }
      }
    }
#pragma unroll
    for (int op = 0; op < 2; ++op) {
      bf16* dst = op == 0 ? q : k;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int c = threadIdx.x + i * kProThreads;
        float x[8], y[8];
        unpack8(raw[op][i], x);
        if (NORM != 0) {
          float sq = ss[op][i];
          if (NORM == 1) {  // the CPH lanes of one head row are an aligned lane group
#pragma unroll
            for (int o = CPH / 2; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          }
          const float r = NORM == 1 ? rsqrtf(sq / (float)D + eps) : rsqrtf(total[op] / (float)(h * D) + eps);
          float4 w0 = make_float4(0.f, 0.f, 0.f, 0.f), w1 = w0;
          if (c < chunks) {
            w0 = s_w[op * 2 * chunks + 2 * c];
            w1 = s_w[op * 2 * chunks + 2 * c + 1];
          }
          y[0] = x[0] * r * w0.x; y[1] = x[1] * r * w0.y; y[2] = x[2] * r * w0.z; y[3] = x[3] * r * w0.w;
          y[4] = x[4] * r * w1.x; y[5] = x[5] * r * w1.y; y[6] = x[6] * r * w1.z; y[7] = x[7] * r * w1.w;
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) y[t] = x[t];
        }
        if (ROPE == 1) {
          if (rotate) {
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = y[t] * cs[t] + y[t ^ 1] * sn[t];
          } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = y[t];
          }
        } else if (ROPE == 2) {
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const float partner = __shfl_xor_sync(0xffffffffu, y[t], CPH / 2);
            x[t] = rotate ? y[t] * cs[t] + partner * sn[t] : y[t];
          }
        } else {
#pragma unroll
          for (int t = 0; t < 8; ++t) x[t] = y[t];
        }
        if (c < chunks) {
          uint4 o;
          o.x = pack_bf16x2(x[0], x[1]);
          o.y = pack_bf16x2(x[2], x[3]);
          o.z = pack_bf16x2(x[4], x[5]);
          o.w = pack_bf16x2(x[6], x[7]);
          *reinterpret_cast<uint4*>(dst + (((size_t)bidx * h + c / CPH) * s + sidx) * D + cc * 8) = o;
        }
      }
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256)
heads_to_tokens_kernel(const uint4* __restrict__ x, uint4* __restrict__ out, int s, int h, size_t total) {
  constexpr int CPH = D / 8;
  const size_t i = (size_t)blockIdx.x * 256 + threadIdx.x;  // chunk index in [b][s][h][CPH]
  if (i >= total) return;
  const int cc = (int)(i % CPH);
  const size_t r = i / CPH;
  const int head = (int)(r % h);
  const size_t bs = r / h;
  const int sidx = (int)(bs % s);
  const size_t bidx = bs / s;
  out[i] = __ldg(x + ((bidx * h + head) * s + sidx) * CPH + cc);
}

template <int D, int NORM, int ROPE, int CH>
int launch_prologue_ch(int tokens, cudaStream_t st, const bf16* qkv, int s, int h, const float* wq,
                       const float* wk, float eps, int rope_len, const float* rc, const float* rs, bf16* q,
                       bf16* k, bf16* v) {
  const int grid = ceil_div(tokens, kProTokens);
  const size_t smem = NORM != 0 ? (size_t)2 * h * D * sizeof(float) : 0;  // <= 64 KB (h*d <= 8192)
  if (smem > 48 * 1024)
    SVG_CUDA_OK(cudaFuncSetAttribute(qkv_prologue_kernel<D, NORM, ROPE, CH>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  qkv_prologue_kernel<D, NORM, ROPE, CH><<<grid, kProThreads, smem, st>>>(qkv, tokens, s, h, wq, wk, eps, rope_len,
                                                                          rc, rs, q, k, v);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

template <int D, int NORM, int ROPE>
int launch_prologue_chunks(int tokens, cudaStream_t st, const bf16* qkv, int s, int h, const float* wq,
                           const float* wk, float eps, int rope_len, const float* rc, const float* rs, bf16* q,
                           bf16* k, bf16* v) {
  const int ch = ceil_div(h * (D / 8), kProThreads);  // 1..kProMaxChunks
  if (ch <= 1) return launch_prologue_ch<D, NORM, ROPE, 1>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  if (ch == 2) return launch_prologue_ch<D, NORM, ROPE, 2>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  if (ch == 3) return launch_prologue_ch<D, NORM, ROPE, 3>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  return launch_prologue_ch<D, NORM, ROPE, kProMaxChunks>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
}

template <int D, int NORM>
int launch_prologue_rope(int rope_mode, int tokens, cudaStream_t st, const bf16* qkv, int s, int h,
                         const float* wq, const float* wk, float eps, int rope_len, const float* rc,
                         const float* rs, bf16* q, bf16* k, bf16* v) {
  if (rope_mode == 0) return launch_prologue_chunks<D, NORM, 0>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  if (rope_mode == 1) return launch_prologue_chunks<D, NORM, 1>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  return launch_prologue_chunks<D, NORM, 2>(tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
}

template <int D>
int launch_prologue(int norm_mode, int rope_mode, int tokens, cudaStream_t st, const bf16* qkv, int s,
                    int h, const float* wq, const float* wk, float eps, int rope_len, const float* rc,
                    const float* rs, bf16* q, bf16* k, bf16* v) {
  if (norm_mode == 0) return launch_prologue_rope<D, 0>(rope_mode, tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  if (norm_mode == 1) return launch_prologue_rope<D, 1>(rope_mode, tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
  return launch_prologue_rope<D, 2>(rope_mode, tokens, st, qkv, s, h, wq, wk, eps, rope_len, rc, rs, q, k, v);
}

bool has_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return n > 0;
}

}  // namespace
}  // namespace svg

using namespace svg;

extern "C" {

int svgear_qkv_prologue(int32_t b, int32_t s, int32_t h, int32_t d, const void* qkv,
                        int32_t norm_mode, const float* q_norm_weight, const float* k_norm_weight,
                        float eps, int32_t rope_mode, int32_t rope_len, const float* rope_cos,
                        const float* rope_sin, void* q, void* k, void* v, void* stream) {
  if (!qkv || !q || !k || !v) return SVGEAR_EINVAL;
  if (norm_mode < SVGEAR_NORM_NONE || norm_mode > SVGEAR_NORM_TOKEN) return SVGEAR_EINVAL;
  if (rope_mode < SVGEAR_ROPE_NONE || rope_mode > SVGEAR_ROPE_HALF_SPLIT) return SVGEAR_EINVAL;
  if (norm_mode != SVGEAR_NORM_NONE && (!q_norm_weight || !k_norm_weight || !(eps >= 0.f))) return SVGEAR_EINVAL;
  if (rope_mode != SVGEAR_ROPE_NONE && (rope_len < 0 || (rope_len > 0 && (!rope_cos || !rope_sin)))) return SVGEAR_EINVAL;
  if (b < 1 || s < 1 || h < 1 || (d != 64 && d != 128)) return SVGEAR_ESHAPE;
  if ((int64_t)h * d > (int64_t)kProThreads * kProMaxChunks * 8) return SVGEAR_ESHAPE;
  if ((int64_t)b * s > 0x7fffffffLL || rope_len > s) return SVGEAR_ESHAPE;
  if (!has_device()) return SVGEAR_ECUDA;
  const int tokens = b * s;
  cudaStream_t st = (cudaStream_t)stream;
  if (d == 128)
    return launch_prologue<128>(norm_mode, rope_mode, tokens, st, (const bf16*)qkv, s, h, q_norm_weight,
                                k_norm_weight, eps, rope_len, rope_cos, rope_sin, (bf16*)q, (bf16*)k, (bf16*)v);
  return launch_prologue<64>(norm_mode, rope_mode, tokens, st, (const bf16*)qkv, s, h, q_norm_weight,
                             k_norm_weight, eps, rope_len, rope_cos, rope_sin, (bf16*)q, (bf16*)k, (bf16*)v);
}

int svgear_heads_to_tokens(int32_t b, int32_t s, int32_t h, int32_t d, const void* x, void* out,
                           void* stream) {
  if (!x || !out) return SVGEAR_EINVAL;
  if (b < 1 || s < 1 || h < 1 || (d != 64 && d != 128)) return SVGEAR_ESHAPE;
  const size_t total = (size_t)b * s * h * (d / 8);
  if ((total + 255) / 256 > 0x7fffffffULL) return SVGEAR_ESHAPE;
  if (!has_device()) return SVGEAR_ECUDA;
  const unsigned grid = (unsigned)((total + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (d == 128)
    heads_to_tokens_kernel<128><<<grid, 256, 0, st>>>((const uint4*)x, (uint4*)out, s, h, total);
  else
    heads_to_tokens_kernel<64><<<grid, 256, 0, st>>>((const uint4*)x, (uint4*)out, s, h, total);
  SVG_LAUNCH_OK();
  return SVGEAR_OK;
}

}  // extern "C"
