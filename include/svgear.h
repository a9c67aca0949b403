/*
 * svgear.h — C ABI of libsvgear.so: the B200 (sm_100a) implementation of the SVG-EAR
 * attention hot path.
 *
 * The reference (`routedattn`, numpy/CPU, /root/reference/pkg/src/routedattn) has no FFI: the
 * operator is the four-call Python composition
 *     prepare -> build_error_table -> route_error_aware -> sparse_attend
 * (README.md:94-98, cli.py:119-134).  Each entry point below replaces one of those calls (cited
 * per function) for a BATCH of independent (Q,K,V) instances ("heads"; `bh` = batch*heads), so a
 * maintainer can bind it from Python with ctypes.
 *
 * Conventions
 *  - plain pointers and sizes only; every pointer is a CUDA DEVICE pointer unless named `host_*`;
 *  - the caller owns every buffer including the workspace; the library allocates no device memory
 *    and outputs are written exactly once.  The only process-wide state is two helper streams (with
 *    their fork/join events) created on first use: svgear_forward runs the key-side k-means, and
 *    the attention executor its remainder-tile kernel, concurrently with the caller's stream and
 *    joins them back before returning, so every result is ordered on `stream` alone;
 *  - all work is enqueued on `stream` (a cudaStream_t passed as void*), nothing synchronises the
 *    host; results are deterministic run to run (no floating-point atomics);
 *  - token matrices are row-major bf16 `[bh][n][d]`, d in {64,128}, d_v == d;
 *  - index outputs are int32; block tables are row-major `[bh][c_q][c_k]`;
 *  - return value: SVGEAR_OK (0) or a negative status; svgear_strerror() names it.
 *  - there is NO CPU fallback: without a CUDA device every compute entry returns SVGEAR_ECUDA.
 */
#ifndef SVGEAR_H_
#define SVGEAR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVGEAR_VERSION 111 /* 0.1.2: greedy tail of the device seeding; executor variants */

enum {
  SVGEAR_OK = 0,
  SVGEAR_EINVAL = -1,      /* bad argument value (null pointer, budget, mode, iteration count)   */
  SVGEAR_ESHAPE = -2,      /* unsupported / inconsistent shape (d, cluster counts vs tokens)      */
  SVGEAR_ECUDA = -3,       /* a CUDA call failed (or no device)                                   */
  SVGEAR_EWORKSPACE = -4,  /* workspace too small; see svgear_workspace_bytes                     */
  SVGEAR_EUNSUPPORTED = -5 /* valid in the reference but not implemented on this path             */
};

/* estimator modes — analysis.build_error_table(mode) (analysis.py:242-249) */
enum { SVGEAR_EST_VALUE_AWARE = 0, SVGEAR_EST_PLAIN = 1 };
/* greedy walk policy — router.DensityBudget.overshoot (router.py:29-30, 100-110) */
enum { SVGEAR_FILL_REMAINDER = 0, SVGEAR_STOP_AT_FIRST_OVERFLOW = 1 };
/* executor arithmetic — sparse_attend(dtype=...) (attention.py:160-168) */
enum {
  SVGEAR_EXEC_BF16_TENSOR = 0, /* tcgen05 bf16 MMA, fp32 softmax/accumulate, bf16 output          */
  SVGEAR_EXEC_FP32_CHECK = 1   /* CUDA-core fp32 everywhere, fp32 output (the "fp32 check mode")  */
};

/* OR-ed into svgear_kmeans' exec_mode: evaluate every token against every centre in every Lloyd
 * iteration.  Without it the tensor-core mode skips tokens whose distance bounds (Hamerly) prove
 * that their cluster cannot change — the assignments are identical, only the work differs. */
enum { SVGEAR_KMEANS_FULL_EVAL = 0x100 };

/* OR-ed into svgear_sparse_attend's exec_mode (SVGEAR_EXEC_BF16_TENSOR only): select a measured
 * alternative of the fused attention kernel instead of the default (two threads per query row, 64-key
 * tiles).  Same semantics, results equal up to the fp32 summation order of the row sums; kept callable so
 * that the parity suite covers them (DESIGN.md 4.1 has their timings). */
enum {
  SVGEAR_ATTEND_ONE_THREAD_PER_ROW = 0x200, /* 8 softmax warps, thread == query row                 */
  SVGEAR_ATTEND_TILE128 = 0x400             /* one N = 128 QK^T per 128-key tile (one thread per row) */
};

/* Problem shape of one call (all `bh` instances share it). */
typedef struct SvgEarShape {
  int32_t bh;  /* number of independent (Q,K,V) instances = batch * heads                         */
  int32_t n_q; /* query tokens per instance                                                       */
  int32_t n_k; /* key/value tokens per instance                                                   */
  int32_t d;   /* head dimension, 64 or 128                                                       */
  int32_t c_q; /* query clusters, 1 <= c_q <= n_q                                                 */
  int32_t c_k; /* key clusters,   1 <= c_k <= n_k, c_k <= 4096                                    */
} SvgEarShape;

/* Optional extra outputs of svgear_forward (any member may be NULL).  These are the fields of the
 * reference's ClusterModel (clustering.py:29-39), BlockErrorTable (estimator.py:50-73) and
 * AttentionResult (attention.py:48-54) that the parity tests compare. */
typedef struct SvgEarAux {
  int32_t* q_assign;    /* [bh][n_q]  raw-order cluster id                                         */
  int32_t* k_assign;    /* [bh][n_k]                                                               */
  int32_t* q_perm;      /* [bh][n_q]  permuted[i] = tokens[perm[i]] (stable sort by cluster)       */
  int32_t* k_perm;      /* [bh][n_k]                                                               */
  int32_t* q_sizes;     /* [bh][c_q]                                                               */
  int32_t* k_sizes;     /* [bh][c_k]                                                               */
  int32_t* q_offsets;   /* [bh][c_q]  exclusive cumsum of sizes                                    */
  int32_t* k_offsets;   /* [bh][c_k]                                                               */
  float* q_centroids;   /* [bh][c_q][d]                                                            */
  float* k_centroids;   /* [bh][c_k][d]                                                            */
  float* v_centroids;   /* [bh][c_k][d]                                                            */
  int32_t* q_iters;     /* [bh] Lloyd iterations executed                                          */
  int32_t* k_iters;     /* [bh]                                                                    */
  double* error_table;  /* [bh][c_q][c_k] stabilised block error sums                              */
  float* stabilizers;   /* [bh][c_q] per-row reference logit the sums were taken at                */
  int64_t* mask_entries;/* [bh] entries covered by selected blocks (BlockMask.density_entries)     */
  float* lse;           /* [bh][n_q] final log-sum-exp per query, ORIGINAL token order             */
  void* kmeans_done_event; /* optional cudaEvent_t (not an output array): recorded on `stream` once both
                           Lloyd loops and the permuted copies of this call are complete, so a caller
                           can start another call's latency-bound clustering under this call's
                           attention kernel                                                        */
} SvgEarAux;

const char* svgear_strerror(int status);
int svgear_version(void);
/* Diagnostic: number of CUDA kernels this library has launched in this process so far. */
int64_t svgear_launch_count(void);

/* Bytes of device workspace sufficient for ANY entry point below at this shape. */
int svgear_workspace_bytes(const SvgEarShape* shape, size_t* bytes);

/* Lloyd k-means for `bh` token matrices from explicit start centres.
 * Replaces clustering.kmeans / _lloyd (clustering.py:104-207) for restarts=1 with the start
 * centres given (the reference draws them with host-side numpy k-means++, clustering.py:65-84;
 * the Python shim reproduces that draw or accepts warm-start centres).
 * Semantics kept: distance = max(|x|^2 - 2x.c + |c|^2, 0); ties -> lowest cluster index; empty
 * clusters repaired in ascending order from the farthest token of a cluster with >=2 members;
 * convergence is tested before the centroid update; final centroids are the member means;
 * permutation = stable sort by cluster.  Distances are evaluated in fp32 (reference: float64):
 * exec_mode SVGEAR_EXEC_BF16_TENSOR forms x.c on the tensor cores (tcgen05) from a 2-way bf16
 * split of the fp32 centroids with fp32 accumulation; SVGEAR_EXEC_FP32_CHECK uses fp32 FMAs.
 *   x            [bh][n][d] bf16          init_centroids [bh][c][d] f32
 *   assign,perm  [bh][n] i32              sizes,offsets  [bh][c] i32
 *   centroids    [bh][c][d] f32           iters [bh] i32, inertia [bh] f64 (either may be NULL) */
int svgear_kmeans(int32_t exec_mode, int32_t bh, int32_t n, int32_t d, int32_t c, const void* x,
                  const float* init_centroids, int32_t max_iters, int32_t* assign, int32_t* perm,
                  int32_t* sizes, int32_t* offsets, float* centroids, int32_t* iters,
                  double* inertia, void* workspace, size_t workspace_bytes, void* stream);

/* Device-side start centres for svgear_kmeans when the caller has none: k-means++ D^2 sampling
 * (the reference's seeding rule, clustering.py:65-84) over a strided subsample of
 * m = min(n, oversample*c, 4096) tokens (sample i = token floor(i*n/m)) with a counter-based hash RNG
 * keyed by (seed, first_instance + b).  This is NOT the reference's numpy draw (the Python shim
 * reproduces that one on the host for parity runs); it is deterministic.  Two kernels: the Gram
 * matrix of the subsample on the tensor cores (tcgen05), then the sequential D^2 rounds, which
 * read only the Gram rows of the centres drawn so far.  The last min(c/2, (n/c)^2/512) centres are
 * drawn greedily (8 D^2 candidates per round, the one that lowers the potential most is kept).
 *   centroids [bh][c][d] f32 (out); workspace: >= bh*m*m*2 bytes (svgear_workspace_bytes covers
 *   oversample <= 8)                                                                             */
int svgear_kmeans_seed(int32_t bh, int32_t n, int32_t d, int32_t c, const void* x,
                       int32_t oversample, uint32_t seed, int32_t first_instance, float* centroids,
                       void* workspace, size_t workspace_bytes, void* stream);

/* The reference's own k-means++ draw, bit for bit, on the device: clustering._kmeans_pp_init
 * (clustering.py:65-84) under numpy's Generator(PCG64) — rng.integers(n) for the first centre, then
 * rng.choice(n, p=d2/total) per centre, with every float64 operation in numpy's order (pairwise row
 * sums and d2.sum(), sequential cumsum, searchsorted(side="right")), and the lowest unused index
 * when all distances are zero.  The result equals the centres the reference starts from for the
 * same generator state, at any size, without a host stage; it is the parity path (the sequential
 * cumsum costs one dependent float64 add per token per centre), not the production seeding.
 *   pcg64_states [bh][4] u64 (DEVICE): {state_hi, state_lo, inc_hi, inc_lo} of each instance's PCG64
 *     right after seeding, i.e. numpy.random.PCG64(SeedSequence(entropy=side_seed,
 *     spawn_key=(restart,))).state (clustering.py:178-180; has_uint32 == 0)
 *   centroids [bh][c][d] f32 (out)      picks [bh][c] i32 token indices (out, may be NULL)
 *   workspace: svgear_kmeans_seed_reference_workspace(bh, n) bytes                              */
int svgear_kmeans_seed_reference(int32_t bh, int32_t n, int32_t d, int32_t c, const void* x,
                                 const uint64_t* pcg64_states, float* centroids, int32_t* picks,
                                 void* workspace, size_t workspace_bytes, void* stream);
int svgear_kmeans_seed_reference_workspace(int32_t bh, int32_t n, size_t* bytes);

/* out[b][i][:] = x[b][perm[b][i]][:]   — clustering.permute_rows (clustering.py:210-212). */
int svgear_permute_rows(int32_t bh, int32_t n, int32_t d, const void* x, const int32_t* perm,
                        void* out, void* stream);

/* Per-cluster means of a cluster-contiguous bf16 matrix, accumulated in ascending row order in
 * float64 and rounded once to f32 — clustering.segment_means (clustering.py:247-257). */
int svgear_segment_means(int32_t bh, int32_t n, int32_t d, int32_t c, const void* x_permuted,
                         const int32_t* sizes, const int32_t* offsets, float* means, void* stream);

/* Block error table — estimator.estimate_errors_streaming / estimate_errors
 * (estimator.py:187-253, 120-148) selected by `mode` as analysis.build_error_table does.
 *   k_permuted, v_permuted [bh][n_k][d] bf16 cluster-contiguous (v may be NULL for PLAIN)
 *   error_table [bh][c_q][c_k] f64 (stabilised at `stabilizers`, multiplied by |q_c|)
 *   stabilizers [bh][c_q] f32 = row max of centroid logits                                      */
int svgear_error_table(const SvgEarShape* shape, int32_t exec_mode, int32_t mode,
                       const float* q_centroids,
                       const float* k_centroids, const float* v_centroids, const void* k_permuted,
                       const void* v_permuted, const int32_t* q_sizes, const int32_t* k_sizes,
                       const int32_t* k_offsets, double* error_table, float* stabilizers,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Greedy error-to-cost routing under an entry budget — router.route_error_aware_entries
 * (router.py:124-142): order (-ratio,-error,qc,kc) (estimator.py:83-96), walk with
 * fillRemainder / stopAtFirstOverflow (router.py:100-110), best-single-block fallback
 * (router.py:113-121).  `capacity_entries` = entry_capacity(rho, n_q*n_k) (router.py:93-97),
 * computed by the caller in double precision exactly as the reference does.
 *   mask [bh][c_q][c_k] u8 (1 = exact block)      entries [bh] i64 (may be NULL)               */
int svgear_route_error_aware(int32_t bh, int32_t c_q, int32_t c_k, const double* error_table,
                             const int32_t* q_sizes, const int32_t* k_sizes,
                             int64_t capacity_entries, int32_t overshoot,
                             int32_t single_item_fallback, uint8_t* mask, int64_t* entries,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Cluster-mass (SVG2-style) routing at the same entry budget — router.route_score
 * (router.py:253-280): per-row softmax of q̄.k̄/sqrt(d) + ln|k_c|, order (-mass, index).        */
int svgear_route_score(const SvgEarShape* shape, const float* q_centroids,
                       const float* k_centroids, const int32_t* q_sizes, const int32_t* k_sizes,
                       int64_t capacity_entries, int32_t overshoot, uint8_t* mask,
                       int64_t* entries, void* workspace, size_t workspace_bytes, void* stream);

/* The top-p baseline as a routing policy of its own — router.score_top_p (router.py:209-236): row i
 * selects the minimal set of key clusters, in descending softmax mass (ties to the lower index),
 * whose cumulative mass reaches p; p = 1 selects every block.
 *   mask [bh][c_q][c_k] u8      entries [bh] i64 (may be NULL)      workspace >= bh*c_q*c_k*8 bytes */
int svgear_route_score_top_p(const SvgEarShape* shape, const float* q_centroids,
                             const float* k_centroids, const int32_t* q_sizes, const int32_t* k_sizes,
                             double p, uint8_t* mask, int64_t* entries, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Error-aware routing under the per-query-cluster top-p budget — router.route_error_aware with
 * DensityBudget.top_p(p) (router.py:172-190): row i may spend the entries of the minimal set of
 * key clusters whose softmax mass (q̄.k̄/sqrt(d) + ln|k_c|, router.py:193-250) reaches p; inside
 * the row the same (-ratio, -error, index) order, walk policy and single-block fallback apply.
 *   p in (0, 1]      mask [bh][c_q][c_k] u8      entries [bh] i64 (may be NULL)                  */
int svgear_route_error_aware_top_p(const SvgEarShape* shape, const double* error_table,
                                   const float* q_centroids, const float* k_centroids,
                                   const int32_t* q_sizes, const int32_t* k_sizes, double p,
                                   int32_t overshoot, int32_t single_item_fallback, uint8_t* mask,
                                   int64_t* entries, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* Block-sparse executor with centroid compensation folded into one online softmax —
 * attention.sparse_attend = exact_block_pass + compensation_pass (attention.py:57-192).
 *   q_permuted/k_permuted/v_permuted cluster-contiguous bf16; mask [bh][c_q][c_k] u8
 *   q_perm: if non-NULL, output row i is scattered to original index q_perm[i]
 *           (clustering.inverse_permute_rows, clustering.py:215-219); if NULL the output keeps
 *           the reference's permuted row order.
 *   out: bf16 [bh][n_q][d] for SVGEAR_EXEC_BF16_TENSOR, f32 for SVGEAR_EXEC_FP32_CHECK
 *   lse: [bh][n_q] f32 or NULL (same row order as out)                                          */
int svgear_sparse_attend(const SvgEarShape* shape, int32_t exec_mode, const void* q_permuted,
                         const void* k_permuted, const void* v_permuted, const int32_t* q_perm,
                         const int32_t* q_sizes, const int32_t* q_offsets, const int32_t* k_sizes,
                         const int32_t* k_offsets, const float* k_centroids,
                         const float* v_centroids, const uint8_t* mask, void* out, float* lse,
                         void* workspace, size_t workspace_bytes, void* stream);

/* The whole operator on one stream: k-means(Q), k-means(K), permute, error table, routing,
 * fused attention; output in ORIGINAL token order.  Equivalent per instance to
 * prepare -> build_error_table -> route_error_aware(global density) -> sparse_attend ->
 * inverse_permute_rows (cli.py:119-134).
 *   q,k,v [bh][n][d] bf16      q_init [bh][c_q][d] f32, k_init [bh][c_k][d] f32
 *   out  [bh][n_q][d] (bf16 / f32 per exec_mode)     mask [bh][c_q][c_k] u8
 *   top_p == 0: global entry budget `capacity_entries`; 0 < top_p <= 1: per-query-cluster top-p
 *   budget as in svgear_route_error_aware_top_p (capacity_entries is then ignored)
 *   aux may be NULL                                                                              */
int svgear_forward(const SvgEarShape* shape, const void* q, const void* k, const void* v,
                   const float* q_init, const float* k_init, int32_t kmeans_iters,
                   int32_t estimator_mode, int64_t capacity_entries, int32_t overshoot,
                   int32_t single_item_fallback, int32_t exec_mode, double top_p, void* out,
                   uint8_t* mask, const SvgEarAux* aux, void* workspace, size_t workspace_bytes,
                   void* stream);

/* svgear_forward with the device-side k-means++ seeding folded in: equivalent to
 * svgear_kmeans_seed(q side, seed) + svgear_kmeans_seed(k side, seed + 0x9E37) followed by
 * svgear_forward, but each side's seeding runs on the stream of that side's Lloyd loop, so the
 * query side does not wait for the (longer) key-side seeding.  NOT the reference's numpy draw: for
 * parity runs hand svgear_forward the reference's start centres.
 *   oversample: subsample size per centre, 1..8 (8 is what the operator uses)
 *   first_instance: instance b of this call draws as instance first_instance + b of the whole batch,
 *   so a caller that splits a batch into groups (one call per group, e.g. on concurrent streams, or
 *   head ranges on different GPUs) gets the centres of the unsplit call
 *   q_init [bh][c_q][d], k_init [bh][c_k][d] f32: OUT, the start centres that were drawn          */
int svgear_forward_seeded(const SvgEarShape* shape, const void* q, const void* k, const void* v,
                          int32_t oversample, uint32_t seed, int32_t first_instance, float* q_init,
                          float* k_init, int32_t kmeans_iters, int32_t estimator_mode,
                          int64_t capacity_entries, int32_t overshoot, int32_t single_item_fallback,
                          int32_t exec_mode, double top_p, void* out, uint8_t* mask,
                          const SvgEarAux* aux, void* workspace, size_t workspace_bytes, void* stream);

/* ---- the callers either side of the operator in a DiT attention block ----
 * The reference stops at single (Q,K,V) matrices; the paper's deployment feeds
 * the operator from a fused QKV projection with q/k RMSNorm and rotary embedding, and feeds its
 * output to the output projection.  The projections are the caller's (library GEMMs); these two
 * entries are the HBM-bound layout/normalisation steps between them and svgear_forward.          */
enum { SVGEAR_NORM_NONE = 0, SVGEAR_NORM_HEAD = 1 /* RMS over d */, SVGEAR_NORM_TOKEN = 2 /* RMS over h*d */ };
enum { SVGEAR_ROPE_NONE = 0, SVGEAR_ROPE_INTERLEAVED = 1 /* pairs (2i,2i+1) */, SVGEAR_ROPE_HALF_SPLIT = 2 /* pairs (i,i+d/2) */ };

/* qkv [b][s][3][h][d] bf16 (the projection output) -> q, k, v [b][h][s][d] bf16.
 *   q, k: y = x * rsqrt(mean(x^2) + eps) * weight (weights f32 [h*d]; mean over d or over h*d),
 *   then tokens with index < rope_len are rotated by rope_cos/rope_sin f32 [rope_len][d/2]
 *   (tokens >= rope_len, e.g. appended text tokens, are not rotated); fp32 arithmetic, one rounding.
 *   h*d <= 8192.                                                                                 */
int svgear_qkv_prologue(int32_t b, int32_t s, int32_t h, int32_t d, const void* qkv,
                        int32_t norm_mode, const float* q_norm_weight, const float* k_norm_weight,
                        float eps, int32_t rope_mode, int32_t rope_len, const float* rope_cos,
                        const float* rope_sin, void* q, void* k, void* v, void* stream);

/* x [b][h][s][d] bf16 (the operator's output) -> out [b][s][h][d] bf16 (the output projection's input) */
int svgear_heads_to_tokens(int32_t b, int32_t s, int32_t h, int32_t d, const void* x, void* out,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SVGEAR_H_ */
