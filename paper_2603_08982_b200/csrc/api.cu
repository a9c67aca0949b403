// extern "C" entry points of libsvgear.so (declared in include/svgear.h).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <string.h>

#include "common.cuh"

using namespace svg;

namespace svg {
long long g_launches = 0;

void report_cuda_error(cudaError_t e, const char* file, int line) {
  static const bool on = getenv("SVGEAR_DEBUG") != nullptr;
  if (on) fprintf(stderr, "libsvgear: %s at %s:%d\n", cudaGetErrorString(e), file, line);
}

namespace {
// Helper streams are keyed by (lane, slot): a lane belongs to one caller stream, so that calls issued
// on different streams (head groups running concurrently) do not serialise on a shared helper.
constexpr int kHelperSlots = 3;  // 0: key side, 1: attention remainder tiles, 2: everything before attention ("front")
constexpr int kHelperLanes = 16;
std::mutex g_lane_mu;
cudaStream_t g_lane_owner[kHelperLanes];
int g_lanes_used = 0;
std::mutex g_helper_mu[kHelperLanes][kHelperSlots];
cudaStream_t g_helper_stream[kHelperLanes][kHelperSlots];
cudaEvent_t g_helper_fork[kHelperLanes][kHelperSlots], g_helper_join[kHelperLanes][kHelperSlots];

int lane_of(cudaStream_t main) {
  std::lock_guard<std::mutex> lk(g_lane_mu);
  for (int i = 0; i < g_lanes_used; ++i)
    if (g_lane_owner[i] == main) return i;
  if (g_lanes_used < kHelperLanes) {
    g_lane_owner[g_lanes_used] = main;
    return g_lanes_used++;
  }
  // more caller streams than lanes: share (correct, only less concurrent)
  return (int)(((uintptr_t)main >> 4) % kHelperLanes);
}
}  // namespace

HelperFork::HelperFork(cudaStream_t main, int slot, cudaStream_t from)
    : main_(from ? from : main), side_(nullptr), slot_(lane_of(main) * kHelperSlots + slot), ok_(false), joined_(false) {
  std::mutex& mu = (&g_helper_mu[0][0])[slot_];
  cudaStream_t& hs = (&g_helper_stream[0][0])[slot_];
  cudaEvent_t& ef = (&g_helper_fork[0][0])[slot_];
  cudaEvent_t& ej = (&g_helper_join[0][0])[slot_];
  mu.lock();
  (void)slot;
  if (!hs) {
    // The streams that carry the work BEFORE the attention kernel (slots 0 and 2) get the highest
    // priority: when two calls run side by side (head groups on two streams), one call's short
    // latency-bound kernels are then scheduled into SMs as the other call's attention CTAs retire,
    // instead of queueing behind its whole grid.  Slot 1 (attention remainder tiles) stays at the
    // default, lowest, priority, like the caller's stream that carries the main attention kernel.
    int prio_lo = 0, prio_hi = 0;
    (void)cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    const int prio = (slot % kHelperSlots) == 1 ? prio_lo : prio_hi;
    if (cudaStreamCreateWithPriority(&hs, cudaStreamNonBlocking, prio) != cudaSuccess ||
        cudaEventCreateWithFlags(&ef, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ej, cudaEventDisableTiming) != cudaSuccess) {
      hs = nullptr;
      (void)cudaGetLastError();
      return;
    }
  }
  side_ = hs;
  ok_ = cudaEventRecord(ef, main_) == cudaSuccess && cudaStreamWaitEvent(side_, ef, 0) == cudaSuccess;
}

int HelperFork::join() {
  if (joined_) return SVGEAR_OK;
  joined_ = true;
  int rc = SVGEAR_OK;
  cudaEvent_t ej = (&g_helper_join[0][0])[slot_];
  if (ok_ && (cudaEventRecord(ej, side_) != cudaSuccess || cudaStreamWaitEvent(main_, ej, 0) != cudaSuccess))
    rc = SVGEAR_ECUDA;
  (&g_helper_mu[0][0])[slot_].unlock();
  return rc;
}

HelperFork::~HelperFork() { (void)join(); }
}  // namespace svg

namespace {

constexpr int kSeedOversampleMax = 8;  // the workspace holds Gram matrices for oversample <= 8

bool shape_ok(const SvgEarShape* s) {
  if (!s) return false;
  if (s->bh < 1 || s->n_q < 1 || s->n_k < 1) return false;
  if (s->d != 64 && s->d != 128) return false;
  if (s->c_q < 1 || s->c_q > s->n_q || s->c_q > kMaxClusters) return false;
  if (s->c_k < 1 || s->c_k > s->n_k || s->c_k > kMaxClusters) return false;
  return true;
}

// Everything svgear_forward keeps in the workspace.  The same routine sizes (base == nullptr) and
// carves it, so the two can never disagree.
struct ForwardPlan {
  KmeansScratch km;   // query side (also what svgear_kmeans alone uses)
  KmeansScratch km2;  // key side: the two Lloyd loops run concurrently on two streams
  AttendScratch at;
  ErrScratch es;
  int32_t *q_assign, *k_assign, *q_perm, *k_perm, *q_sizes, *k_sizes, *q_offsets, *k_offsets;
  int32_t *q_iters, *k_iters;
  float *q_cent, *k_cent, *v_cent, *stab, *lse_tmp;
  double* err;
  unsigned long long* route_keys;
  int64_t* entries;
  bf16 *qp, *kp, *vp;
  bf16 *q_gram, *k_gram;  // Gram matrices of the seeding subsamples (svgear_forward_seeded)
};

bool plan_forward(const SvgEarShape& s, Carver& cv, ForwardPlan& p) {
  const int nmax = s.n_q > s.n_k ? s.n_q : s.n_k;
  const int cmax = s.c_q > s.c_k ? s.c_q : s.c_k;
  p.km.carve(cv, s.bh, nmax, cmax, s.d);
  p.km2.carve(cv, s.bh, s.n_k, s.c_k, s.d);
  p.at.carve(cv, s);
  p.q_assign = cv.take<int32_t>((size_t)s.bh * s.n_q);
  p.k_assign = cv.take<int32_t>((size_t)s.bh * s.n_k);
  p.q_perm = cv.take<int32_t>((size_t)s.bh * s.n_q);
  p.k_perm = cv.take<int32_t>((size_t)s.bh * s.n_k);
  p.q_sizes = cv.take<int32_t>((size_t)s.bh * s.c_q);
  p.k_sizes = cv.take<int32_t>((size_t)s.bh * s.c_k);
  p.q_offsets = cv.take<int32_t>((size_t)s.bh * s.c_q);
  p.k_offsets = cv.take<int32_t>((size_t)s.bh * s.c_k);
  p.q_iters = cv.take<int32_t>(s.bh);
  p.k_iters = cv.take<int32_t>(s.bh);
  p.q_cent = cv.take<float>((size_t)s.bh * s.c_q * s.d);
  p.k_cent = cv.take<float>((size_t)s.bh * s.c_k * s.d);
  p.v_cent = cv.take<float>((size_t)s.bh * s.c_k * s.d);
  p.es.carve(cv, s);
  p.stab = cv.take<float>((size_t)s.bh * s.c_q);
  p.lse_tmp = cv.take<float>((size_t)s.bh * s.n_q);
  p.err = cv.take<double>((size_t)s.bh * s.c_q * s.c_k);
  p.route_keys = cv.take<unsigned long long>((size_t)s.bh * s.c_q * s.c_k);
  p.entries = cv.take<int64_t>(s.bh);
  p.qp = cv.take<bf16>((size_t)s.bh * s.n_q * s.d);
  p.kp = cv.take<bf16>((size_t)s.bh * s.n_k * s.d);
  p.vp = cv.take<bf16>((size_t)s.bh * s.n_k * s.d);
  const size_t mq = (size_t)seed_subsample(s.n_q, s.c_q, kSeedOversampleMax);
  const size_t mk = (size_t)seed_subsample(s.n_k, s.c_k, kSeedOversampleMax);
  p.q_gram = cv.take<bf16>((size_t)s.bh * mq * mq);
  p.k_gram = cv.take<bf16>((size_t)s.bh * mk * mk);
  return cv.ok;
}

size_t forward_bytes(const SvgEarShape& s) {
  Carver cv(nullptr, (size_t)-1);
  ForwardPlan p;
  plan_forward(s, cv, p);
  return cv.off + 256;
}

bool device_present() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return n > 0;
}

}  // namespace

extern "C" {

const char* svgear_strerror(int status) {
  switch (status) {
    case SVGEAR_OK: return "ok";
    case SVGEAR_EINVAL: return "invalid argument";
    case SVGEAR_ESHAPE: return "unsupported or inconsistent shape";
    case SVGEAR_ECUDA: return "CUDA error (or no CUDA device)";
    case SVGEAR_EWORKSPACE: return "workspace too small";
    case SVGEAR_EUNSUPPORTED: return "not supported on this path";
    default: return "unknown status";
  }
}

int svgear_version(void) { return SVGEAR_VERSION; }

int64_t svgear_launch_count(void) { return (int64_t)svg::g_launches; }

int svgear_workspace_bytes(const SvgEarShape* shape, size_t* bytes) {
  if (!shape || !bytes) return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  *bytes = forward_bytes(*shape);
  return SVGEAR_OK;
}

int svgear_kmeans(int32_t exec_mode, int32_t bh, int32_t n, int32_t d, int32_t c, const void* x,
                  const float* init_centroids, int32_t max_iters, int32_t* assign, int32_t* perm,
                  int32_t* sizes, int32_t* offsets, float* centroids, int32_t* iters,
                  double* inertia, void* workspace, size_t workspace_bytes, void* stream) {
  if (!x || !init_centroids || !assign || !perm || !sizes || !offsets || !centroids || !workspace)
    return SVGEAR_EINVAL;
  if (max_iters < 1) return SVGEAR_EINVAL;
  const int32_t base_mode = exec_mode & ~SVGEAR_KMEANS_FULL_EVAL;
  if (base_mode != SVGEAR_EXEC_BF16_TENSOR && base_mode != SVGEAR_EXEC_FP32_CHECK) return SVGEAR_EINVAL;
  if (bh < 1 || n < 1 || (d != 64 && d != 128) || c < 1 || c > n || c > kMaxClusters)
    return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  KmeansScratch sc;
  if (!sc.carve(cv, bh, n, c, d)) return SVGEAR_EWORKSPACE;
  return launch_kmeans(exec_mode, bh, n, d, c, (const bf16*)x, init_centroids, max_iters, assign, perm, sizes,
                       offsets, centroids, iters, inertia, sc, (cudaStream_t)stream);
}

int svgear_kmeans_seed(int32_t bh, int32_t n, int32_t d, int32_t c, const void* x, int32_t oversample,
                       uint32_t seed, int32_t first_instance, float* centroids, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!x || !centroids || !workspace) return SVGEAR_EINVAL;
  if (oversample < 1 || first_instance < 0) return SVGEAR_EINVAL;
  if (bh < 1 || n < 1 || (d != 64 && d != 128) || c < 1 || c > n || c > kMaxClusters)
    return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  const size_t m = (size_t)seed_subsample(n, c, oversample);
  Carver cv(workspace, workspace_bytes);
  bf16* gram = cv.take<bf16>((size_t)bh * m * m);
  if (!cv.ok) return SVGEAR_EWORKSPACE;
  return launch_seed(bh, n, d, c, oversample, (const bf16*)x, seed, first_instance, centroids, gram,
                     (cudaStream_t)stream);
}

int svgear_kmeans_seed_reference(int32_t bh, int32_t n, int32_t d, int32_t c, const void* x,
                                 const uint64_t* pcg64_states, float* centroids, int32_t* picks, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (!x || !pcg64_states || !centroids || !workspace) return SVGEAR_EINVAL;
  if (bh < 1 || n < 1 || (d != 64 && d != 128) || c < 1 || c > n || c > kMaxClusters) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  if (workspace_bytes < seed_reference_ws_bytes(bh, n)) return SVGEAR_EWORKSPACE;
  return launch_seed_reference(bh, n, d, c, (const bf16*)x, pcg64_states, centroids, picks, workspace, workspace_bytes,
                               (cudaStream_t)stream);
}

int svgear_kmeans_seed_reference_workspace(int32_t bh, int32_t n, size_t* bytes) {
  if (!bytes || bh < 1 || n < 1) return SVGEAR_EINVAL;
  *bytes = seed_reference_ws_bytes(bh, n);
  return SVGEAR_OK;
}

int svgear_permute_rows(int32_t bh, int32_t n, int32_t d, const void* x, const int32_t* perm,
                        void* out, void* stream) {
  if (!x || !perm || !out) return SVGEAR_EINVAL;
  if (bh < 1 || n < 1 || (d != 64 && d != 128)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  return launch_gather_rows(bh, n, d, (const bf16*)x, perm, (bf16*)out, (cudaStream_t)stream);
}

int svgear_segment_means(int32_t bh, int32_t n, int32_t d, int32_t c, const void* x_permuted,
                         const int32_t* sizes, const int32_t* offsets, float* means, void* stream) {
  if (!x_permuted || !sizes || !offsets || !means) return SVGEAR_EINVAL;
  if (bh < 1 || n < 1 || (d != 64 && d != 128) || c < 1 || c > n) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  return launch_segment_means(bh, n, d, c, (const bf16*)x_permuted, sizes, offsets, means, nullptr,
                              (cudaStream_t)stream);
}

int svgear_error_table(const SvgEarShape* shape, int32_t exec_mode, int32_t mode, const float* q_centroids,
                       const float* k_centroids, const float* v_centroids, const void* k_permuted,
                       const void* v_permuted, const int32_t* q_sizes, const int32_t* k_sizes,
                       const int32_t* k_offsets, double* error_table, float* stabilizers,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape || !q_centroids || !k_centroids || !k_permuted || !q_sizes || !k_sizes || !k_offsets ||
      !error_table || !stabilizers || !workspace)
    return SVGEAR_EINVAL;
  if (mode != SVGEAR_EST_VALUE_AWARE && mode != SVGEAR_EST_PLAIN) return SVGEAR_EINVAL;
  if (mode == SVGEAR_EST_VALUE_AWARE && (!v_centroids || !v_permuted)) return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  ErrScratch es;
  if (!es.carve(cv, *shape)) return SVGEAR_EWORKSPACE;
  if (exec_mode != SVGEAR_EXEC_BF16_TENSOR && exec_mode != SVGEAR_EXEC_FP32_CHECK) return SVGEAR_EINVAL;
  return launch_error_table(*shape, exec_mode, mode, q_centroids, k_centroids, v_centroids,
                            (const bf16*)k_permuted, (const bf16*)v_permuted, q_sizes, k_sizes,
                            k_offsets, error_table, stabilizers, es, (cudaStream_t)stream);
}

int svgear_route_error_aware(int32_t bh, int32_t c_q, int32_t c_k, const double* error_table,
                             const int32_t* q_sizes, const int32_t* k_sizes,
                             int64_t capacity_entries, int32_t overshoot,
                             int32_t single_item_fallback, uint8_t* mask, int64_t* entries,
                             void* workspace, size_t workspace_bytes, void* stream) {
  if (!error_table || !q_sizes || !k_sizes || !mask || !workspace) return SVGEAR_EINVAL;
  if (capacity_entries < 0) return SVGEAR_EINVAL;
  if (overshoot != SVGEAR_FILL_REMAINDER && overshoot != SVGEAR_STOP_AT_FIRST_OVERFLOW)
    return SVGEAR_EINVAL;
  if (bh < 1 || c_q < 1 || c_k < 1 || c_k > kMaxClusters) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  unsigned long long* keys = cv.take<unsigned long long>((size_t)bh * c_q * c_k);
  if (!cv.ok) return SVGEAR_EWORKSPACE;
  return launch_route(bh, c_q, c_k, error_table, q_sizes, k_sizes, capacity_entries, overshoot,
                      single_item_fallback ? 1 : 0, 0, mask, entries, keys, (cudaStream_t)stream);
}

int svgear_route_score(const SvgEarShape* shape, const float* q_centroids,
                       const float* k_centroids, const int32_t* q_sizes, const int32_t* k_sizes,
                       int64_t capacity_entries, int32_t overshoot, uint8_t* mask,
                       int64_t* entries, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape || !q_centroids || !k_centroids || !q_sizes || !k_sizes || !mask || !workspace)
    return SVGEAR_EINVAL;
  if (capacity_entries < 0) return SVGEAR_EINVAL;
  if (overshoot != SVGEAR_FILL_REMAINDER && overshoot != SVGEAR_STOP_AT_FIRST_OVERFLOW)
    return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  double* mass = cv.take<double>((size_t)shape->bh * shape->c_q * shape->c_k);
  unsigned long long* keys = cv.take<unsigned long long>((size_t)shape->bh * shape->c_q * shape->c_k);
  if (!cv.ok) return SVGEAR_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_score_mass(*shape, q_centroids, k_centroids, k_sizes, mass, st);
  if (rc != SVGEAR_OK) return rc;
  return launch_route(shape->bh, shape->c_q, shape->c_k, mass, q_sizes, k_sizes, capacity_entries,
                      overshoot, 0, 1, mask, entries, keys, st);
}

int svgear_route_error_aware_top_p(const SvgEarShape* shape, const double* error_table,
                                   const float* q_centroids, const float* k_centroids,
                                   const int32_t* q_sizes, const int32_t* k_sizes, double p,
                                   int32_t overshoot, int32_t single_item_fallback, uint8_t* mask,
                                   int64_t* entries, void* workspace, size_t workspace_bytes,
                                   void* stream) {
  if (!shape || !error_table || !q_centroids || !k_centroids || !q_sizes || !k_sizes || !mask || !workspace)
    return SVGEAR_EINVAL;
  if (!(p > 0.0 && p <= 1.0)) return SVGEAR_EINVAL;
  if (overshoot != SVGEAR_FILL_REMAINDER && overshoot != SVGEAR_STOP_AT_FIRST_OVERFLOW)
    return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  double* mass = cv.take<double>((size_t)shape->bh * shape->c_q * shape->c_k);
  if (!cv.ok) return SVGEAR_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_score_mass(*shape, q_centroids, k_centroids, k_sizes, mass, st);
  if (rc != SVGEAR_OK) return rc;
  return launch_route_top_p(*shape, error_table, mass, q_sizes, k_sizes, p, overshoot,
                            single_item_fallback ? 1 : 0, mask, entries, st);
}

int svgear_route_score_top_p(const SvgEarShape* shape, const float* q_centroids, const float* k_centroids,
                             const int32_t* q_sizes, const int32_t* k_sizes, double p, uint8_t* mask,
                             int64_t* entries, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape || !q_centroids || !k_centroids || !q_sizes || !k_sizes || !mask || !workspace) return SVGEAR_EINVAL;
  if (!(p > 0.0 && p <= 1.0)) return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  double* mass = cv.take<double>((size_t)shape->bh * shape->c_q * shape->c_k);
  if (!cv.ok) return SVGEAR_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_score_mass(*shape, q_centroids, k_centroids, k_sizes, mass, st);
  if (rc != SVGEAR_OK) return rc;
  return launch_route_top_p(*shape, nullptr, mass, q_sizes, k_sizes, p, SVGEAR_FILL_REMAINDER, 0, mask, entries, st);
}

int svgear_sparse_attend(const SvgEarShape* shape, int32_t exec_mode, const void* q_permuted,
                         const void* k_permuted, const void* v_permuted, const int32_t* q_perm,
                         const int32_t* q_sizes, const int32_t* q_offsets, const int32_t* k_sizes,
                         const int32_t* k_offsets, const float* k_centroids,
                         const float* v_centroids, const uint8_t* mask, void* out, float* lse,
                         void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape || !q_permuted || !k_permuted || !v_permuted || !q_sizes || !q_offsets || !k_sizes ||
      !k_offsets || !k_centroids || !v_centroids || !mask || !out || !workspace)
    return SVGEAR_EINVAL;
  const int32_t variant = exec_mode & (SVGEAR_ATTEND_ONE_THREAD_PER_ROW | SVGEAR_ATTEND_TILE128);
  const int32_t base_mode = exec_mode & ~variant;
  if (base_mode != SVGEAR_EXEC_BF16_TENSOR && base_mode != SVGEAR_EXEC_FP32_CHECK) return SVGEAR_EINVAL;
  if (variant && base_mode != SVGEAR_EXEC_BF16_TENSOR) return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  Carver cv(workspace, workspace_bytes);
  AttendScratch sc;
  if (!sc.carve(cv, *shape)) return SVGEAR_EWORKSPACE;
  return launch_attend(*shape, exec_mode, (const bf16*)q_permuted, (const bf16*)k_permuted,
                       (const bf16*)v_permuted, q_perm, q_sizes, q_offsets, k_sizes, k_offsets,
                       k_centroids, v_centroids, mask, out, lse, sc, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
// Device-side k-means++ seeding folded into the forward pass: each side's seeding kernel runs on the
// stream of that side's Lloyd loop (svgear_forward_seeded), so the short query-side seeding does not
// wait for the long key-side one.
struct SeedPlan {
  int oversample;
  uint32_t seed;
  int first;  // index of this call's first instance in the caller's whole batch
};

int forward_impl(const SvgEarShape* shape, const void* q, const void* k, const void* v,
                 float* q_init, float* k_init, const SeedPlan* sp, int32_t kmeans_iters,
                 int32_t estimator_mode, int64_t capacity_entries, int32_t overshoot,
                 int32_t single_item_fallback, int32_t exec_mode, double top_p, void* out, uint8_t* mask,
                 const SvgEarAux* aux, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape || !q || !k || !v || !q_init || !k_init || !out || !mask || !workspace)
    return SVGEAR_EINVAL;
  if (kmeans_iters < 1 || capacity_entries < 0) return SVGEAR_EINVAL;
  if (!(top_p >= 0.0 && top_p <= 1.0)) return SVGEAR_EINVAL;
  if (estimator_mode != SVGEAR_EST_VALUE_AWARE && estimator_mode != SVGEAR_EST_PLAIN)
    return SVGEAR_EINVAL;
  if (overshoot != SVGEAR_FILL_REMAINDER && overshoot != SVGEAR_STOP_AT_FIRST_OVERFLOW)
    return SVGEAR_EINVAL;
  if (exec_mode != SVGEAR_EXEC_BF16_TENSOR && exec_mode != SVGEAR_EXEC_FP32_CHECK)
    return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (!device_present()) return SVGEAR_ECUDA;
  const SvgEarShape& s = *shape;
  Carver cv(workspace, workspace_bytes);
  ForwardPlan p;
  if (!plan_forward(s, cv, p)) return SVGEAR_EWORKSPACE;
  SvgEarAux a;
  memset(&a, 0, sizeof(a));
  if (aux) a = *aux;
  // aux outputs, when requested, are written in place instead of the workspace copies
  int32_t* q_assign = a.q_assign ? a.q_assign : p.q_assign;
  int32_t* k_assign = a.k_assign ? a.k_assign : p.k_assign;
  int32_t* q_perm = a.q_perm ? a.q_perm : p.q_perm;
  int32_t* k_perm = a.k_perm ? a.k_perm : p.k_perm;
  int32_t* q_sizes = a.q_sizes ? a.q_sizes : p.q_sizes;
  int32_t* k_sizes = a.k_sizes ? a.k_sizes : p.k_sizes;
  int32_t* q_offsets = a.q_offsets ? a.q_offsets : p.q_offsets;
  int32_t* k_offsets = a.k_offsets ? a.k_offsets : p.k_offsets;
  float* q_cent = a.q_centroids ? a.q_centroids : p.q_cent;
  float* k_cent = a.k_centroids ? a.k_centroids : p.k_cent;
  float* v_cent = a.v_centroids ? a.v_centroids : p.v_cent;
  int32_t* q_iters = a.q_iters ? a.q_iters : p.q_iters;
  int32_t* k_iters = a.k_iters ? a.k_iters : p.k_iters;
  double* err = a.error_table ? a.error_table : p.err;
  float* stab = a.stabilizers ? a.stabilizers : p.stab;
  int64_t* entries = a.mask_entries ? a.mask_entries : p.entries;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  // (1) cluster Q and K independently; V follows K (analysis.py:228-238).  The two sides share
  // nothing, and the late Lloyd iterations are short latency-bound launches, so the key side is
  // forked onto a helper stream (HelperFork, common.cuh); the join makes the caller's stream the
  // only one anything downstream depends on.
  int rc_k = SVGEAR_ECUDA;
  rc = SVGEAR_ECUDA;
  const bool keys_early = exec_mode == SVGEAR_EXEC_BF16_TENSOR;
  // everything before the attention kernel runs on high-priority helper streams ("front" for the query
  // side, estimator and routing; slot 0 for the key side), the attention kernel on the caller's stream
  HelperFork ff(st, 2);
  if (!ff.ok()) return SVGEAR_ECUDA;
  cudaStream_t front = ff.side();
  {
    HelperFork fk(st, 0, front);
    if (!fk.ok()) return SVGEAR_ECUDA;
    cudaStream_t side = fk.side();
    rc_k = sp ? launch_seed(s.bh, s.n_k, s.d, s.c_k, sp->oversample, (const bf16*)k, sp->seed + 0x9E37u, sp->first,
                            k_init, p.k_gram, side)
              : SVGEAR_OK;
    if (!rc_k)
      rc_k = launch_kmeans(exec_mode, s.bh, s.n_k, s.d, s.c_k, (const bf16*)k, k_init, kmeans_iters, k_assign,
                           k_perm, k_sizes, k_offsets, k_cent, k_iters, nullptr, p.km2, side);
    if (!rc_k) rc_k = launch_gather_rows(s.bh, s.n_k, s.d, (const bf16*)k, k_perm, p.kp, side);
    if (!rc_k) rc_k = launch_gather_rows(s.bh, s.n_k, s.d, (const bf16*)v, k_perm, p.vp, side);
    if (!rc_k)
      rc_k = launch_segment_means(s.bh, s.n_k, s.d, s.c_k, p.vp, k_sizes, k_offsets, v_cent, nullptr, side);
    // the key-side half of the estimator needs nothing from the query side: keep it on the helper
    // stream, under the (usually longer) query-side Lloyd loop
    if (!rc_k && keys_early)
      rc_k = launch_error_table_keys(s, estimator_mode, k_cent, v_cent, p.kp, p.vp, k_sizes, k_offsets, p.es, side);
    rc = sp ? launch_seed(s.bh, s.n_q, s.d, s.c_q, sp->oversample, (const bf16*)q, sp->seed, sp->first, q_init,
                          p.q_gram, front)
            : SVGEAR_OK;
    if (!rc)
      rc = launch_kmeans(exec_mode, s.bh, s.n_q, s.d, s.c_q, (const bf16*)q, q_init, kmeans_iters, q_assign,
                         q_perm, q_sizes, q_offsets, q_cent, q_iters, nullptr, p.km, front);
    if (!rc) rc = launch_gather_rows(s.bh, s.n_q, s.d, (const bf16*)q, q_perm, p.qp, front);
    // join unconditionally so that the helper stream never outlives the caller's ordering
    if (fk.join() != SVGEAR_OK) rc = SVGEAR_ECUDA;
  }
  if (rc) return rc;
  if (rc_k) return rc_k;
  if (a.kmeans_done_event) SVG_CUDA_OK(cudaEventRecord((cudaEvent_t)a.kmeans_done_event, front));
  // (2) error table + routing
  rc = launch_error_table(s, exec_mode, estimator_mode, q_cent, k_cent, v_cent, p.kp, p.vp, q_sizes,
                          k_sizes, k_offsets, err, stab, p.es, front, keys_early);
  if (rc) return rc;
  if (top_p > 0.0) {  // per-query-cluster top-p budget (router.py:172-190); the key buffer holds the masses
    double* mass = reinterpret_cast<double*>(p.route_keys);
    rc = launch_score_mass(s, q_cent, k_cent, k_sizes, mass, front);
    if (rc) return rc;
    rc = launch_route_top_p(s, err, mass, q_sizes, k_sizes, top_p, overshoot, single_item_fallback ? 1 : 0, mask,
                            entries, front);
  } else {
    rc = launch_route(s.bh, s.c_q, s.c_k, err, q_sizes, k_sizes, capacity_entries, overshoot,
                      single_item_fallback ? 1 : 0, 0, mask, entries, p.route_keys, front);
  }
  if (ff.join() != SVGEAR_OK && !rc) rc = SVGEAR_ECUDA;
  if (rc) return rc;
  // (3) fused executor, output scattered to original token order
  return launch_attend(s, exec_mode, p.qp, p.kp, p.vp, q_perm, q_sizes, q_offsets, k_sizes, k_offsets,
                       k_cent, v_cent, mask, out, a.lse, p.at, st);
}
}  // namespace

extern "C" {

int svgear_forward(const SvgEarShape* shape, const void* q, const void* k, const void* v,
                   const float* q_init, const float* k_init, int32_t kmeans_iters,
                   int32_t estimator_mode, int64_t capacity_entries, int32_t overshoot,
                   int32_t single_item_fallback, int32_t exec_mode, double top_p, void* out, uint8_t* mask,
                   const SvgEarAux* aux, void* workspace, size_t workspace_bytes, void* stream) {
  return forward_impl(shape, q, k, v, const_cast<float*>(q_init), const_cast<float*>(k_init), nullptr,
                      kmeans_iters, estimator_mode, capacity_entries, overshoot, single_item_fallback, exec_mode,
                      top_p, out, mask, aux, workspace, workspace_bytes, stream);
}

int svgear_forward_seeded(const SvgEarShape* shape, const void* q, const void* k, const void* v,
                          int32_t oversample, uint32_t seed, int32_t first_instance, float* q_init, float* k_init,
                          int32_t kmeans_iters, int32_t estimator_mode, int64_t capacity_entries, int32_t overshoot,
                          int32_t single_item_fallback, int32_t exec_mode, double top_p, void* out, uint8_t* mask,
                          const SvgEarAux* aux, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape || first_instance < 0 || oversample < 1 || oversample > kSeedOversampleMax) return SVGEAR_EINVAL;
  if (!shape_ok(shape)) return SVGEAR_ESHAPE;
  if (seed_subsample(shape->n_q, shape->c_q, oversample) < shape->c_q ||
      seed_subsample(shape->n_k, shape->c_k, oversample) < shape->c_k)
    return SVGEAR_ESHAPE;
  SeedPlan sp{oversample, seed, first_instance};
  return forward_impl(shape, q, k, v, q_init, k_init, &sp, kmeans_iters, estimator_mode, capacity_entries,
                      overshoot, single_item_fallback, exec_mode, top_p, out, mask, aux, workspace,
                      workspace_bytes, stream);
}

}  // extern "C"
