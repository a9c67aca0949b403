// Executor, fp32 check mode (CUDA cores) + the metadata shared with the tcgen05 executor.
//
// Reference semantics: /root/reference/pkg/src/routedattn/attention.py
//   exact_block_pass   :57-101   softmax over the keys of the selected blocks of a query cluster
//   compensation_pass  :104-157  every unselected key cluster j enters as ONE key with logit
//                                q.k̄_j/sqrt(d) + ln|k_j| and value v̄_j
// Both passes share a single online softmax here (they are one softmax mathematically: the
// reference seeds the second pass with (m = lse, l = 1, acc = O), attention.py:142-144), so the
// output is written once.  Rows whose cluster selects nothing start from (m=-inf, l=0).
#include "common.cuh"

namespace svg {

// ------------------------------------------------------------------------------------------------
// q-row tiles that do not cross a query-cluster boundary: (cluster, first row, rows)
// ------------------------------------------------------------------------------------------------
// split_rows > 0 (tensor-core executor): tiles with more than split_rows rows fill the list from the
// front (tile_count[h] of them), the others — at most one per query cluster — from the back
// (tile_count[bh + h] of them, entry r at index max_tiles - 1 - r), so that each of the two executor
// kernels launches over its own compact list.  split_rows == 0: one list, tile_count[h] entries.
__global__ void __launch_bounds__(1024)
    build_tiles_kernel(int c_q, int rows_per_tile, int max_tiles, int split_rows, const int32_t* __restrict__ q_sizes,
                       const int32_t* __restrict__ q_offsets, int32_t* __restrict__ tile_list,
                       int32_t* __restrict__ tile_count) {
  const int h = blockIdx.x;
  __shared__ int s_warp[2][32];
  __shared__ int s_carry[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 2) s_carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < c_q; base += 1024) {
    const int i = base + tid;
    const int nq = i < c_q ? q_sizes[(size_t)h * c_q + i] : 0;
    const int nt = ceil_div(nq, rows_per_tile);
    const int last_rows = nq - (nt - 1) * rows_per_tile;
    const int nback = (split_rows > 0 && nt > 0 && last_rows <= split_rows) ? 1 : 0;
    const int nfront = nt - nback;
    int inc0 = nfront, inc1 = nback;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(0xffffffffu, inc0, o), y1 = __shfl_up_sync(0xffffffffu, inc1, o);
      if (lane >= o) { inc0 += y0; inc1 += y1; }
    }
    if (lane == 31) { s_warp[0][warp] = inc0; s_warp[1][warp] = inc1; }
    __syncthreads();
    if (warp < 2) {
      int w = s_warp[warp][lane], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      s_warp[warp][lane] = wi - w;
    }
    __syncthreads();
    const int pos0 = s_carry[0] + s_warp[0][warp] + inc0 - nfront;
    const int pos1 = s_carry[1] + s_warp[1][warp] + inc1 - nback;
    if (i < c_q) {
      const int o = q_offsets[(size_t)h * c_q + i];
      for (int t = 0; t < nt; ++t) {
        const bool back = nback && t == nt - 1;
        const int slot = back ? max_tiles - 1 - pos1 : pos0 + t;
        int32_t* e = tile_list + ((size_t)h * max_tiles + slot) * 4;
        e[0] = i;
        e[1] = o + t * rows_per_tile;
        e[2] = min(rows_per_tile, nq - t * rows_per_tile);
        e[3] = 0;
      }
    }
    __syncthreads();
    if (tid == 1023) { s_carry[0] = pos0 + nfront; s_carry[1] = pos1 + nback; }
    __syncthreads();
  }
  if (tid == 0) {
    tile_count[h] = s_carry[0];
    tile_count[gridDim.x + h] = s_carry[1];
  }
}

// bf16 copies of the key/value centroids (zero-padded to a multiple of 64 rows) and ln|k_c|
__global__ void prep_centroids_kernel(const float* __restrict__ kc, const float* __restrict__ vc,
                                      const int32_t* __restrict__ k_sizes, int d, int c_k, int ckpad,
                                      bf16* __restrict__ kb, bf16* __restrict__ vb,
                                      float* __restrict__ lnw) {
  const int h = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ckpad * d) return;
  const int j = idx / d;
  float kv = 0.f, vv = 0.f;
  if (j < c_k) {
    kv = kc[(size_t)h * c_k * d + idx];
    vv = vc[(size_t)h * c_k * d + idx];
  }
  kb[(size_t)h * ckpad * d + idx] = __float2bfloat16_rn(kv);
  vb[(size_t)h * ckpad * d + idx] = __float2bfloat16_rn(vv);
  if (idx % d == 0 && j < c_k) lnw[(size_t)h * c_k + j] = (float)log((double)k_sizes[(size_t)h * c_k + j]);
}

// ------------------------------------------------------------------------------------------------
// fp32 executor: block = 4 warps x 4 query rows; key tiles of 32 (lane <-> key)
// ------------------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128)
    attend_fp32_kernel(const bf16* __restrict__ qp, const bf16* __restrict__ kp,
                       const bf16* __restrict__ vp, const int32_t* __restrict__ q_perm,
                       const int32_t* __restrict__ k_sizes, const int32_t* __restrict__ k_offsets,
                       const float* __restrict__ kc, const float* __restrict__ vc,
                       const float* __restrict__ lnw, const uint8_t* __restrict__ mask,
                       const int32_t* __restrict__ tile_list, const int32_t* __restrict__ tile_count,
                       int max_tiles, int n_q, int n_k, int c_q, int c_k, float scale,
                       float* __restrict__ out, float* __restrict__ lse) {
  const int h = blockIdx.y;
  if ((int)blockIdx.x >= tile_count[h]) return;
  const int32_t* te = tile_list + ((size_t)h * max_tiles + blockIdx.x) * 4;
  const int qcl = te[0], row0 = te[1], nrows = te[2];
  constexpr int R = 16, TK = 32, CPL = D / 32;
  __shared__ float sQ[R][D];
  __shared__ float sK[TK][D + 1];
  __shared__ float sV[TK][D];
  __shared__ float sP[R][TK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < R * D; i += 128) {
    const int r = i / D, k = i % D;
    const int row = min(row0 + r, n_q - 1);
    sQ[r][k] = __bfloat162float(qp[((size_t)h * n_q + row) * D + k]);
  }
  float m[4], l[4], acc[4][CPL];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int u = 0; u < CPL; ++u) acc[r][u] = 0.f;
  }
  const uint8_t* mrow = mask + ((size_t)h * c_q + qcl) * c_k;

  // one tile of up to 32 "keys": phase 0 = real keys of a selected cluster, phase 1 = centroids
  auto process = [&](float bias_or_ninf) {
    // S = Q K^T for this warp's 4 rows, lane's key
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int k = 0; k < D; ++k) {
      const float kv = sK[lane][k];
      s[0] = fmaf(sQ[warp * 4 + 0][k], kv, s[0]);
      s[1] = fmaf(sQ[warp * 4 + 1][k], kv, s[1]);
      s[2] = fmaf(sQ[warp * 4 + 2][k], kv, s[2]);
      s[3] = fmaf(sQ[warp * 4 + 3][k], kv, s[3]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float sv = s[r] * scale + bias_or_ninf;  // -inf masks the column
      const float mt = warp_max(sv);
      const float mn = fmaxf(m[r], mt);
      const float ms = (mn == -INFINITY) ? 0.f : mn;
      const float alpha = expf(m[r] - ms);  // m = -inf -> 0
      const float p = expf(sv - ms);
      l[r] = l[r] * alpha + warp_sum(p);
      m[r] = mn;
      sP[warp * 4 + r][lane] = p;
#pragma unroll
      for (int u = 0; u < CPL; ++u) acc[r][u] *= alpha;
    }
    __syncwarp();
    for (int t = 0; t < TK; ++t) {
      float vv[CPL];
#pragma unroll
      for (int u = 0; u < CPL; ++u) vv[u] = sV[t][lane * CPL + u];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float p = sP[warp * 4 + r][t];
#pragma unroll
        for (int u = 0; u < CPL; ++u) acc[r][u] = fmaf(p, vv[u], acc[r][u]);
      }
    }
  };

  // ---- exact blocks, ascending key-cluster order (attention.py:86-91)
  for (int j = 0; j < c_k; ++j) {
    if (!mrow[j]) continue;
    const int nj = k_sizes[(size_t)h * c_k + j], o = k_offsets[(size_t)h * c_k + j];
    for (int t0 = 0; t0 < nj; t0 += TK) {
      __syncthreads();
      for (int i = tid; i < TK * D; i += 128) {
        const int r = i / D, k = i % D;
        const int row = min(o + t0 + r, n_k - 1);
        sK[r][k] = __bfloat162float(kp[((size_t)h * n_k + row) * D + k]);
        sV[r][k] = __bfloat162float(vp[((size_t)h * n_k + row) * D + k]);
      }
      __syncthreads();
      process((t0 + lane < nj) ? 0.f : -INFINITY);
    }
  }
  // ---- compensation: unselected clusters as single keys (attention.py:136-155)
  for (int j0 = 0; j0 < c_k; j0 += TK) {
    __syncthreads();
    for (int i = tid; i < TK * D; i += 128) {
      const int r = i / D, k = i % D;
      const int j = min(j0 + r, c_k - 1);
      sK[r][k] = kc[((size_t)h * c_k + j) * D + k];
      sV[r][k] = vc[((size_t)h * c_k + j) * D + k];
    }
    __syncthreads();
    const int j = j0 + lane;
    const bool use = j < c_k && !mrow[j];
    process(use ? lnw[(size_t)h * c_k + j] : -INFINITY);
  }
  // ---- write (optionally scattering rows back to original token order)
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int rr = warp * 4 + r;
    if (rr < nrows) {
      const int prow = row0 + rr;
      const int dst = q_perm ? q_perm[(size_t)h * n_q + prow] : prow;
      const float inv = 1.f / l[r];
#pragma unroll
      for (int u = 0; u < CPL; ++u)
        out[((size_t)h * n_q + dst) * D + lane * CPL + u] = acc[r][u] * inv;
      if (lse && lane == 0) lse[(size_t)h * n_q + dst] = m[r] + logf(l[r]);
    }
  }
}

size_t AttendScratch::bytes(const SvgEarShape& s) {
  const int ckpad = ceil_div(s.c_k, 64) * 64 + 64;
  const int mt = max_tiles(s.n_q, s.c_q, 16);
  size_t b = 0;
  b += align_up((size_t)s.bh * mt * 4 * 4, 256);
  b += align_up((size_t)s.bh * 8, 256);
  b += align_up((size_t)s.bh * ckpad * s.d * 2, 256) * 2;
  b += align_up((size_t)s.bh * s.c_k * 4, 256);
  return b + 2048;
}

bool AttendScratch::carve(Carver& cv, const SvgEarShape& s) {
  const int ckpad = ceil_div(s.c_k, 64) * 64 + 64;
  const int mt = max_tiles(s.n_q, s.c_q, 16);
  tile_list = cv.take<int32_t>((size_t)s.bh * mt * 4);
  tile_count = cv.take<int32_t>((size_t)2 * s.bh);  // [front counts | back counts]
  kbar_bf16 = cv.take<bf16>((size_t)s.bh * ckpad * s.d);
  vbar_bf16 = cv.take<bf16>((size_t)s.bh * ckpad * s.d);
  lnw = cv.take<float>((size_t)s.bh * s.c_k);
  return cv.ok;
}

int launch_attend(const SvgEarShape& s, int exec_mode, const bf16* qp, const bf16* kp,
                  const bf16* vp, const int32_t* q_perm, const int32_t* q_sizes,
                  const int32_t* q_offsets, const int32_t* k_sizes, const int32_t* k_offsets,
                  const float* kc, const float* vc, const uint8_t* mask, void* out, float* lse,
                  AttendScratch& sc, cudaStream_t st) {
  const int variant = exec_mode & (SVGEAR_ATTEND_ONE_THREAD_PER_ROW | SVGEAR_ATTEND_TILE128);
  exec_mode &= ~variant;
  const int ckpad = ceil_div(s.c_k, 64) * 64;  // rows of the bf16 centroid arrays (zero padded)
  const float scale = 1.0f / sqrtf((float)s.d);
  prep_centroids_kernel<<<dim3(ceil_div(ckpad * s.d, 256), s.bh), 256, 0, st>>>(
      kc, vc, k_sizes, s.d, s.c_k, ckpad, sc.kbar_bf16, sc.vbar_bf16, sc.lnw);
  SVG_LAUNCH_OK();
  const int rows = exec_mode == SVGEAR_EXEC_FP32_CHECK ? 16 : attend_tc_rows_per_tile();
  const int mt = AttendScratch::max_tiles(s.n_q, s.c_q, rows);
  build_tiles_kernel<<<s.bh, 1024, 0, st>>>(s.c_q, rows, mt, exec_mode == SVGEAR_EXEC_FP32_CHECK ? 0 : 128, q_sizes,
                                            q_offsets, sc.tile_list, sc.tile_count);
  SVG_LAUNCH_OK();
  if (exec_mode == SVGEAR_EXEC_FP32_CHECK) {
    if (s.d == 128)
      attend_fp32_kernel<128><<<dim3(mt, s.bh), 128, 0, st>>>(
          qp, kp, vp, q_perm, k_sizes, k_offsets, kc, vc, sc.lnw, mask, sc.tile_list, sc.tile_count,
          mt, s.n_q, s.n_k, s.c_q, s.c_k, scale, (float*)out, lse);
    else
      attend_fp32_kernel<64><<<dim3(mt, s.bh), 128, 0, st>>>(
          qp, kp, vp, q_perm, k_sizes, k_offsets, kc, vc, sc.lnw, mask, sc.tile_list, sc.tile_count,
          mt, s.n_q, s.n_k, s.c_q, s.c_k, scale, (float*)out, lse);
    SVG_LAUNCH_OK();
    return SVGEAR_OK;
  }
  return launch_attend_tc(s, qp, kp, vp, q_perm, k_sizes, k_offsets, mask, (bf16*)out, lse, sc, variant, st);
}

}  // namespace svg
