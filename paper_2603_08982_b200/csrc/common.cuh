// Shared device/host helpers for libsvgear (sm_100a only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/svgear.h"

// SVGEAR_DEBUG=1 in the environment names the failing CUDA call on stderr (diagnostic only).
#define SVG_CUDA_OK(call)                                    \
  do {                                                       \
    cudaError_t e__ = (call);                                \
    if (e__ != cudaSuccess) {                                \
      svg::report_cuda_error(e__, __FILE__, __LINE__);       \
      return SVGEAR_ECUDA;                                   \
    }                                                        \
  } while (0)

#define SVG_LAUNCH_OK()                                      \
  do {                                                       \
    ++svg::g_launches;                                       \
    if (cudaPeekAtLastError() != cudaSuccess) {              \
      svg::report_cuda_error(cudaGetLastError(), __FILE__, __LINE__); \
      return SVGEAR_ECUDA;                                   \
    }                                                        \
  } while (0)

namespace svg {

extern long long g_launches;  // diagnostic: kernels launched by this library in this process
void report_cuda_error(cudaError_t e, const char* file, int line);

typedef __nv_bfloat16 bf16;

constexpr int kMaxClusters = 4096;
constexpr int kSortChunk = 2048;  // tokens per counting-sort chunk

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Bump allocator over the caller-provided workspace.
struct Carver {
  char* base;
  size_t off;
  size_t cap;
  bool ok;
  __host__ Carver(void* p, size_t bytes) : base((char*)p), off(0), cap(bytes), ok(true) {}
  template <typename T>
  __host__ T* take(size_t count) {
    off = align_up(off, 256);
    T* r = (T*)(base + off);
    off += count * sizeof(T);
    if (off > cap) ok = false;
    return r;
  }
};

__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

// 8 bf16 (one 16-byte chunk) -> 8 floats
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fork/join onto a process-wide helper stream (api.cu).  Independent pieces of one call (the two
// k-means sides; the two attention kernels) run concurrently: the constructor makes helper stream
// `slot` wait for everything enqueued on `main` so far, join() makes `main` wait for the helper.
// The helper streams and events are created once (stream creation can serialise with running
// work); a per-slot mutex keeps concurrent host threads from interleaving their fork/join pairs.
// Event based, so the pattern is capturable in a CUDA graph.
class HelperFork {
 public:
  // `main` keys the lane (one set of helper streams per caller stream); the helper forks from and joins
  // back to `from` (default: main) — a helper can itself be forked from another helper of the lane
  HelperFork(cudaStream_t main, int slot, cudaStream_t from = nullptr);
  ~HelperFork();
  bool ok() const { return ok_; }
  cudaStream_t side() const { return side_; }
  int join();  // SVGEAR_OK or SVGEAR_ECUDA; idempotent
 private:
  cudaStream_t main_, side_;
  int slot_;
  bool ok_, joined_;
};

// ---- stage launchers (defined in the per-stage .cu files) -------------------------------------

struct KmeansScratch {
  int32_t* prev_assign;   // [bh][n]
  float* own_d2;          // [bh][n]
  float* cnorm;           // [bh][c]
  double* chunk_inertia;  // [bh][nchunks]
  int32_t* done;          // [bh]
  bf16* pieces;           // [bh][pieces][cpad][d]  split-bf16 centroids (tensor-core assignment)
  float* cnorm_pad;       // [bh][cpad]
  float* xnorm;           // [bh][n]
  // exact bound-based skipping (tensor-core mode): per-token bounds, active lists, centre movement
  float* ub;              // [bh][n]  >= distance to the assigned centre
  float* lb;              // [bh][n]  <= distance to every other centre
  int32_t* active;        // [bh][n]  tokens to re-evaluate this iteration (first nactive[h])
  int32_t* nactive;       // [bh]
  float* move;            // [bh][c]  |c_new - c_old| of the last update
  uint8_t* dirty;         // [bh][c]  membership changed this iteration
  int32_t* iters_run;     // [bh]     iterations executed (internal copy of `iters`)
  int32_t* resid_nz;      // [bh]     the second bf16 piece of some centre is non-zero
  float* dmin;            // [bh][c]  distance from each centre to the nearest big mover (lloyd_step_kernel B2)
  bool carve(Carver& cv, int bh, int n, int c, int d);
};

// Arguments of the fused per-iteration kernel (lloyd_step.cu); all arrays are the [bh][...] ones above.
struct LloydStepArgs {
  const bf16* x;
  int n, c, cpad;
  int iter;           // -1: set up the state of iteration 0 (norms, pieces, all-active list)
  int max_iters;
  int use_tc;         // tensor-core assignment: pieces / bounds / active lists are maintained
  int bounded;        // bound-based skipping (use_tc and not FULL_EVAL)
  int bounded_state;  // ub / lb / dirty exist (== use_tc)
  int phases;         // bit 0: histograms .. permutation, bit 1: means + next iteration's inputs
  int wsort, scratch_bytes;  // filled by the launcher
  int32_t *assign, *prev, *perm, *sizes, *offsets, *iters;
  float *cent, *cnorm, *own, *ub, *lb, *move, *dmin, *cnorm_pad, *xnorm;
  uint8_t* dirty;
  bf16* pieces;
  int32_t *active, *nactive, *resid_nz, *done, *iters_run;
};
int launch_lloyd_step(const LloydStepArgs& args, int bh, int d, cudaStream_t st);

int launch_kmeans(int exec_mode, int bh, int n, int d, int c, const bf16* x, const float* init,
                  int max_iters, int32_t* assign, int32_t* perm, int32_t* sizes, int32_t* offsets,
                  float* centroids, int32_t* iters, double* inertia, KmeansScratch& sc,
                  cudaStream_t st);
// device-side k-means++ seeding (seed.cu): subsample size, and the two-kernel launch
int seed_subsample(int n, int c, int oversample);
int launch_seed(int bh, int n, int d, int c, int oversample, const bf16* x, uint32_t seed, int first_instance,
                float* cent, bf16* gram_ws, cudaStream_t st);
// the reference's numpy k-means++ draw on the device (seed_ref.cu)
size_t seed_reference_ws_bytes(int bh, int n);
int launch_seed_reference(int bh, int n, int d, int c, const bf16* x, const uint64_t* pcg_states, float* cent,
                          int32_t* picks, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_gather_rows(int bh, int n, int d, const bf16* x, const int32_t* perm, bf16* out,
                       cudaStream_t st);
int launch_segment_means(int bh, int n, int d, int c, const bf16* xp, const int32_t* sizes,
                         const int32_t* offsets, float* means, float* norms, cudaStream_t st);

struct ErrScratch {
  float* sbar;    // [bh][c_q][c_k] centroid logits
  bf16* kd_hi;    // [bh][n_k][d]   k - k̄ split into bf16 hi / lo (tensor-core path)
  bf16* kd_lo;
  float* kstat;   // [3][bh][n_k]   planes A, -2B, C of the per-key scalars
  bf16* qsplit;   // [bh][2][cqpad][d]
  bool carve(Carver& cv, const SvgEarShape& s);
};
int launch_error_table(const SvgEarShape& s, int exec_mode, int mode, const float* qc, const float* kc,
                       const float* vc, const bf16* kp, const bf16* vp, const int32_t* q_sizes,
                       const int32_t* k_sizes, const int32_t* k_offsets, double* err,
                       float* stabilizers, ErrScratch& sc, cudaStream_t st, bool key_stats_done = false);
int launch_error_table_keys(const SvgEarShape& s, int mode, const float* kc, const float* vc, const bf16* kp,
                            const bf16* vp, const int32_t* k_sizes, const int32_t* k_offsets, ErrScratch& sc,
                            cudaStream_t st);

int launch_route(int bh, int c_q, int c_k, const double* val, const int32_t* q_sizes,
                 const int32_t* k_sizes, int64_t capacity, int overshoot, int fallback,
                 int ratio_mode, uint8_t* mask, int64_t* entries, unsigned long long* keys,
                 cudaStream_t st);
int launch_score_mass(const SvgEarShape& s, const float* qc, const float* kc,
                      const int32_t* k_sizes, double* mass, cudaStream_t st);
int launch_route_top_p(const SvgEarShape& s, const double* err, const double* mass, const int32_t* q_sizes,
                       const int32_t* k_sizes, double p, int overshoot, int fallback, uint8_t* mask,
                       int64_t* entries, cudaStream_t st);

struct AttendScratch {
  int32_t* tile_list;   // [bh][max_tiles][4]  (q-cluster, first row, rows, pad)
  int32_t* tile_count;  // [bh]
  bf16* kbar_bf16;      // [bh][ckpad][d]
  bf16* vbar_bf16;      // [bh][ckpad][d]
  float* lnw;           // [bh][c_k]
  static int max_tiles(int n_q, int c_q, int rows) { return ceil_div(n_q, rows) + c_q; }
  static size_t bytes(const SvgEarShape& s);
  bool carve(Carver& cv, const SvgEarShape& s);
};
int launch_attend(const SvgEarShape& s, int exec_mode, const bf16* qp, const bf16* kp,
                  const bf16* vp, const int32_t* q_perm, const int32_t* q_sizes,
                  const int32_t* q_offsets, const int32_t* k_sizes, const int32_t* k_offsets,
                  const float* kc, const float* vc, const uint8_t* mask, void* out, float* lse,
                  AttendScratch& sc, cudaStream_t st);
// tcgen05 path (attend_tc.cu)
int attend_tc_rows_per_tile();
int launch_attend_tc(const SvgEarShape& s, const bf16* qp, const bf16* kp, const bf16* vp,
                     const int32_t* q_perm, const int32_t* k_sizes, const int32_t* k_offsets,
                     const uint8_t* mask, bf16* out, float* lse, AttendScratch& sc, int variant,
                     cudaStream_t st);

}  // namespace svg
