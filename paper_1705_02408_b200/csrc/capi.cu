// paper_1705_02408_b200/csrc/capi.cu -- the extern "C" boundary of
// libmpap.so (include/mpap.h): argument validation, status codes, device
// memory ownership.  All compute happens in build_kernels.cu / search_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "mpap_internal.cuh"

namespace mpap {
static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void note_launch(int k) { g_launches.fetch_add(k); }

static std::atomic<long long> g_team_launches[3];
void note_team(int team) { g_team_launches[team].fetch_add(1); }

void* workspace(cudaStream_t st, int tag, size_t bytes) {
  struct Key {
    int dev;
    cudaStream_t st;
    int tag;
    bool operator<(const Key& o) const {
      if (dev != o.dev) return dev < o.dev;
      if (st != o.st) return st < o.st;
      return tag < o.tag;
    }
  };
  static std::mutex mu;
  static std::map<Key, std::pair<void*, size_t>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto& e = cache[Key{dev, st, tag}];
  if (e.second >= bytes && e.first) return e.first;
  if (e.first) cudaFreeAsync(e.first, st);
  e.first = nullptr;
  e.second = 0;
  const size_t grow = bytes + bytes / 4;   // headroom against small size changes
  void* p = nullptr;
  if (cudaMallocAsync(&p, grow, st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  e.first = p;
  e.second = grow;
  return p;
}

namespace {
struct BufCache {
  std::mutex mu;
  std::map<int, std::multimap<size_t, void*>> free_by_dev;   // size -> buffer
  std::map<void*, std::pair<size_t, int>> owned;              // buffer -> (size, device)
  std::map<int, size_t> cached_bytes, cap_bytes;
};
BufCache& bufcache() {
  static BufCache* c = new BufCache();   // never destroyed: release may run at exit
  return *c;
}
size_t round_size(size_t b) {
  const size_t g = (b >= (size_t(2) << 20)) ? (size_t(2) << 20) : 256;
  return ((std::max<size_t>(b, 1) + g - 1) / g) * g;
}
}  // namespace

void* rm_alloc(size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t want = round_size(bytes);
  BufCache& c = bufcache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto& fl = c.free_by_dev[dev];
    auto it = fl.lower_bound(want);
    if (it != fl.end() && it->first <= want + want / 8) {
      void* p = it->second;
      c.cached_bytes[dev] -= it->first;
      fl.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, want, st) != cudaSuccess) {
    cudaGetLastError();
    // drop this device's cache and retry once
    std::vector<void*> drop;
    {
      std::lock_guard<std::mutex> lk(c.mu);
      for (auto& kv : c.free_by_dev[dev]) drop.push_back(kv.second);
      c.free_by_dev[dev].clear();
      c.cached_bytes[dev] = 0;
      for (void* q : drop) c.owned.erase(q);
    }
    if (drop.empty()) {
      set_error(MPAP_ERR_OUT_OF_MEMORY, "device allocation failed");
      return nullptr;
    }
    cudaStreamSynchronize(st);
    for (void* q : drop) cudaFreeAsync(q, st);
    cudaStreamSynchronize(st);
    if (cudaMallocAsync(&p, want, st) != cudaSuccess) {
      cudaGetLastError();
      set_error(MPAP_ERR_OUT_OF_MEMORY, "device allocation failed");
      return nullptr;
    }
  }
  std::lock_guard<std::mutex> lk(c.mu);
  c.owned[p] = {want, dev};
  return p;
}

void rm_release(void* p) {
  if (!p) return;
  BufCache& c = bufcache();
  std::unique_lock<std::mutex> lk(c.mu);
  auto it = c.owned.find(p);
  if (it == c.owned.end()) {   // not ours (cannot happen for roadmap arrays)
    lk.unlock();
    cudaFreeAsync(p, 0);
    return;
  }
  const size_t sz = it->second.first;
  const int dev = it->second.second;
  if (!c.cap_bytes.count(dev)) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    size_t cap = tot / 4;
    if (const char* e = getenv("MPAP_CACHE_MB")) cap = (size_t)atoll(e) << 20;
    c.cap_bytes[dev] = cap;
  }
  if (c.cached_bytes[dev] + sz > c.cap_bytes[dev]) {
    c.owned.erase(it);
    lk.unlock();
    cudaFreeAsync(p, 0);
    return;
  }
  c.free_by_dev[dev].emplace(sz, p);
  c.cached_bytes[dev] += sz;
}

void retain_pool_memory(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == device) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(device);
}

// ---- per-kernel event timing ------------------------------------------------
namespace {
struct PendingRec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<int> g_prof_on{0};
std::vector<PendingRec> g_pending;
std::map<std::string, std::pair<double, long long>> g_prof_acc;

void prof_drain_locked() {
  for (auto& p : g_pending) {
    float ms = 0.0f;
    if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      auto& acc = g_prof_acc[p.name];
      acc.first += ms;
      acc.second += 1;
    }
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  g_pending.clear();
}
}  // namespace

// NVTX: every kernel launch of the library is a named host range (visible to
// nsys / ncu --nvtx when a tool is attached; a no-op otherwise).
ProfScope::ProfScope(const char* kernel, cudaStream_t stream) : name(kernel), st(stream), rec(nullptr) {
  nvtxRangePushA(kernel);
  if (!g_prof_on.load()) return;
  PendingRec* r = new PendingRec{kernel, nullptr, nullptr};
  cudaEventCreate(&r->a);
  cudaEventCreate(&r->b);
  cudaEventRecord(r->a, st);
  rec = r;
}

ProfScope::~ProfScope() {
  nvtxRangePop();
  if (!rec) return;
  PendingRec* r = static_cast<PendingRec*>(rec);
  cudaEventRecord(r->b, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_pending.push_back(*r);
  delete r;
}

mpap_status set_error(mpap_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

mpap_status cuda_error(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) return MPAP_ERR_OUT_OF_MEMORY;
  return MPAP_ERR_CUDA;
}
}  // namespace mpap

using namespace mpap;

#define CKC(x)                                          \
  do {                                                  \
    cudaError_t _e = (x);                               \
    if (_e != cudaSuccess) {                            \
      mpap_status _s = cuda_error(_e, #x);              \
      mpap_roadmap_free(rm);                            \
      return _s;                                        \
    }                                                   \
  } while (0)

static bool is_fin(double x) { return std::isfinite(x); }

// Lazy roadmaps (NEXT-1 part i): calls other than the single-query search see
// a fully evaluated roadmap -- evaluate every remaining row first.
static mpap_status ensure_evaluated(const mpap_roadmap* rm, cudaStream_t st) {
  if (!rm->lazy) return MPAP_OK;
  return evaluate_rows_device(const_cast<mpap_roadmap*>(rm), nullptr, 0, st);
}

template <typename T>
static cudaError_t rm_alloc_into(T** out, size_t bytes, cudaStream_t st) {
  *out = static_cast<T*>(rm_alloc(bytes, st));
  return *out ? cudaSuccess : cudaErrorMemoryAllocation;
}

static mpap_status validate_params(const mpap_params* p, double r) {
  if (!p) return set_error(MPAP_ERR_INVALID_ARGUMENT, "params is NULL");
  if (p->pos_dim != 2 && p->pos_dim != 3) return set_error(MPAP_ERR_INVALID_ARGUMENT, "pos_dim must be 2 or 3");
  if (p->dynamics != MPAP_KINEMATIC && p->dynamics != MPAP_DOUBLE_INTEGRATOR)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "unknown dynamics");
  if (p->heuristic < MPAP_PH_OMNI_COUNT || p->heuristic > MPAP_PH_FOV_HEADING_MLP)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "unknown heuristic");
  if (p->heuristic >= MPAP_PH_FOV_HEADING_COUNT && !p->has_heading)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "heading heuristic needs has_heading");
  if (p->heuristic == MPAP_PH_FOV_HEADING_MLP && !p->mlp)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "MLP heuristic needs 122 weights");
  if (!(r > 0.0) || !is_fin(r)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "r must be finite and > 0");
  const double pos[] = {p->control_weight, p->nominal_speed, p->dt, p->collision_dt, p->n_f, p->max_range,
                        p->v_ref, p->w_ref};
  for (double x : pos)
    if (!(x > 0.0) || !is_fin(x)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "params: positive finite field");
  if (!(p->fov_cos_half > 0.0) || p->fov_cos_half > 1.0)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "fov_cos_half must be in (0, 1]");
  if (!is_fin(p->mlp_gain)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "mlp_gain not finite");
  if ((p->edge_peaks != 0 && p->edge_peaks != 1) || (p->lazy_edges != 0 && p->lazy_edges != 1))
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "edge_peaks and lazy_edges must be 0 or 1");
  for (int k = 0; k < p->pos_dim; ++k)
    if (!(p->ws_lo[k] < p->ws_hi[k])) return set_error(MPAP_ERR_INVALID_ARGUMENT, "workspace lo >= hi");
  return MPAP_OK;
}

// Per-environment size limits of the edge kernels: the per-step visible
// counts are uint16 (k_heuristic -> k_fold), and each warp stages the
// environment's features (D + 1 doubles each) and boxes (2D doubles) in shared
// memory (kEdgeWarps warps per block, <= 227 KB per block with the static
// arrays).  Larger environments are rejected, never wrapped or truncated.
static mpap_status check_env_sizes(int d, int64_t n_obstacles, int64_t n_features) {
  constexpr int64_t kEdgeWarps = 4, kStaticBytes = 8 * 1024, kSmemMax = 227 * 1024;
  if (n_features > 65535) return set_error(MPAP_ERR_INVALID_ARGUMENT, "more than 65535 features in one environment");
  // per warp at most fs (d + 3.5) + 3 d os doubles with fs, os = F, O rounded
  // up to a multiple of 4 (warp_scratch_doubles in build_kernels.cu: kept
  // features, masks, float feature copies and the edge's feature list make
  // fs (d + 3.5); boxes 2 d os, plus d os for the optional float box copies)
  const int64_t fs = (n_features + 3) & ~3, os = (n_obstacles + 3) & ~3;
  const int64_t bytes = 4 * kEdgeWarps * (fs * (2 * d + 7) + os * 6 * d) + kStaticBytes;
  if (bytes > kSmemMax)
    return set_error(MPAP_ERR_INVALID_ARGUMENT,
                     "environment too large for the edge kernels' shared-memory working set "
                     "(16 (F4 (2 d + 7) + 6 d O4) bytes + 8 KB, F4 / O4 = F / O rounded up to a multiple of 4, "
                     "must fit in 227 KB)");
  return MPAP_OK;
}

extern "C" {

const char* mpap_status_str(mpap_status s) {
  switch (s) {
    case MPAP_OK: return "MPAP_OK";
    case MPAP_ERR_INVALID_ARGUMENT: return "MPAP_ERR_INVALID_ARGUMENT";
    case MPAP_ERR_NO_GOAL_NODE: return "MPAP_ERR_NO_GOAL_NODE";
    case MPAP_ERR_NO_FEASIBLE_PLAN: return "MPAP_ERR_NO_FEASIBLE_PLAN";
    case MPAP_ERR_BUFFER_TOO_SMALL: return "MPAP_ERR_BUFFER_TOO_SMALL";
    case MPAP_ERR_OUT_OF_MEMORY: return "MPAP_ERR_OUT_OF_MEMORY";
    case MPAP_ERR_CUDA: return "MPAP_ERR_CUDA";
  }
  return "MPAP_ERR_UNKNOWN";
}

const char* mpap_last_error(void) { return g_last_error.c_str(); }

int64_t mpap_launch_count(void) { return (int64_t)g_launches.load(); }

int64_t mpap_search_launches(int32_t team) {
  return (team >= 0 && team < 3) ? (int64_t)g_team_launches[team].load() : -1;
}

void mpap_prof_enable(int32_t on) { g_prof_on.store(on ? 1 : 0); }

void mpap_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_drain_locked();
  g_prof_acc.clear();
}

int32_t mpap_prof_read(const char* kernel, double* total_ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  prof_drain_locked();
  auto it = g_prof_acc.find(kernel ? kernel : "");
  if (it == g_prof_acc.end()) {
    if (total_ms) *total_ms = 0.0;
    if (launches) *launches = 0;
    return 0;
  }
  if (total_ms) *total_ms = it->second.first;
  if (launches) *launches = it->second.second;
  return 1;
}

void mpap_roadmap_free(mpap_roadmap* rm) {
  if (!rm) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(rm->device);
  // every search of this roadmap may still be in flight on some stream:
  // wait for the device, then hand the memory back to the stream-ordered pool
  cudaDeviceSynchronize();
  void* ptrs[] = {rm->d_samples, rm->d_obst, rm->d_feat, rm->d_obst_base, rm->d_feat_base, rm->d_node_base,
                  rm->d_row_ptr, rm->d_edges, rm->d_peak, rm->d_tau, rm->d_esrc, rm->d_ready};
  for (void* p : ptrs) rm_release(p);   // device is idle: safe to reuse from any stream
  cudaSetDevice(cur);
  delete rm;
}

static mpap_status build_batch_impl(int32_t n_envs, const double* samples, const int32_t* n, int32_t row_stride,
                                    const double* obstacles, const int32_t* n_obstacles, const double* features,
                                    const int32_t* n_features, double r, const mpap_params* params, int32_t mem,
                                    void* cuda_stream, int64_t row_lo, int64_t row_hi, mpap_roadmap** out);

mpap_status mpap_build_roadmap_batch(int32_t n_envs, const double* samples, const int32_t* n, int32_t row_stride,
                                     const double* obstacles, const int32_t* n_obstacles, const double* features,
                                     const int32_t* n_features, double r, const mpap_params* params, int32_t mem,
                                     void* cuda_stream, mpap_roadmap** out) {
  return build_batch_impl(n_envs, samples, n, row_stride, obstacles, n_obstacles, features, n_features, r, params,
                          mem, cuda_stream, 0, INT64_MAX, out);
}

mpap_status mpap_build_roadmap_rows(const double* samples, int32_t n, int32_t row_stride, const double* obstacles,
                                    int32_t n_obstacles, const double* features, int32_t n_features, double r,
                                    const mpap_params* params, int32_t row_begin, int32_t row_end, int32_t mem,
                                    void* cuda_stream, mpap_roadmap** out) {
  if (row_begin < 0 || row_end < row_begin || row_end > n)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "row range must satisfy 0 <= begin <= end <= n");
  return build_batch_impl(1, samples, &n, row_stride, obstacles, &n_obstacles, features, &n_features, r, params, mem,
                          cuda_stream, row_begin, row_end, out);
}

static mpap_status build_batch_impl(int32_t n_envs, const double* samples, const int32_t* n, int32_t row_stride,
                                    const double* obstacles, const int32_t* n_obstacles, const double* features,
                                    const int32_t* n_features, double r, const mpap_params* params, int32_t mem,
                                    void* cuda_stream, int64_t row_lo, int64_t row_hi, mpap_roadmap** out) {
  if (!out) return set_error(MPAP_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n_envs < 1 || !n || !n_obstacles || !n_features || !samples)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "n_envs < 1 or NULL count/sample arrays");
  if (mem != MPAP_MEM_HOST && mem != MPAP_MEM_DEVICE) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad mem space");
  mpap_status s = validate_params(params, r);
  if (s != MPAP_OK) return s;
  const int d = params->pos_dim;
  const int need = d * (params->dynamics == MPAP_DOUBLE_INTEGRATOR ? 2 : 1) + (params->has_heading ? 2 : 0);
  if (row_stride < need || row_stride > 8)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "row_stride too small (or > 8)");
  int64_t N = 0, O = 0, F = 0;
  for (int b = 0; b < n_envs; ++b) {
    if (n[b] < 1) return set_error(MPAP_ERR_INVALID_ARGUMENT, "n < 1");
    if (n_obstacles[b] < 0 || n_features[b] < 0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "negative count");
    mpap_status se = check_env_sizes(params->pos_dim, n_obstacles[b], n_features[b]);
    if (se != MPAP_OK) return se;
    N += n[b];
    O += n_obstacles[b];
    F += n_features[b];
  }
  if (N > INT32_MAX / 2) return set_error(MPAP_ERR_INVALID_ARGUMENT, "too many nodes");
  if ((O > 0 && !obstacles) || (F > 0 && !features))
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL obstacle/feature array");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  // host copies of the inputs are needed for validation of host arrays only;
  // device arrays are validated by value-independent checks (sizes) here.
  if (mem == MPAP_MEM_HOST) {
    for (int64_t i = 0; i < N * row_stride; ++i)
      if (!is_fin(samples[i])) return set_error(MPAP_ERR_INVALID_ARGUMENT, "non-finite sample coordinate");
    for (int64_t o = 0; o < O; ++o)
      for (int k = 0; k < d; ++k)
        if (!(obstacles[o * 2 * d + k] < obstacles[o * 2 * d + d + k]))
          return set_error(MPAP_ERR_INVALID_ARGUMENT, "obstacle with lo >= hi");
  }
  HostTimer tall("mpap_build_roadmap_batch total");
  mpap_roadmap* rm = new (std::nothrow) mpap_roadmap();
  if (!rm) return set_error(MPAP_ERR_OUT_OF_MEMORY, "host allocation failed");
  CKC(cudaGetDevice(&rm->device));
  retain_pool_memory(rm->device);
  rm->B = n_envs;
  DevParams& P = rm->prm;
  std::memset(&P, 0, sizeof(P));
  P.pos_dim = d;
  P.dynamics = params->dynamics;
  P.has_heading = params->has_heading;
  P.heuristic = params->heuristic;
  P.stride = row_stride;
  P.edge_peaks = params->edge_peaks;
  rm->lazy = params->lazy_edges != 0;
  P.hoff = d * (params->dynamics == MPAP_DOUBLE_INTEGRATOR ? 2 : 1);
  for (int k = 0; k < 3; ++k) {
    P.ws_lo[k] = params->ws_lo[k];
    P.ws_hi[k] = params->ws_hi[k];
  }
  P.control_weight = params->control_weight;
  P.nominal_speed = params->nominal_speed;
  P.dt = params->dt;
  P.collision_dt = params->collision_dt;
  P.n_f = params->n_f;
  P.fov_cos_half = params->fov_cos_half;
  P.max_range = params->max_range;
  P.mlp_gain = params->mlp_gain;
  P.v_ref = params->v_ref;
  P.w_ref = params->w_ref;
  P.r = r;
  P.row_lo = row_lo;   // row-sharded build (mpap_build_roadmap_rows); all rows otherwise
  P.row_hi = row_hi;
  if (params->mlp) std::memcpy(P.mlp, params->mlp, sizeof(double) * kMlpSize);
  rm->n.assign(n, n + n_envs);
  rm->n_obst.assign(n_obstacles, n_obstacles + n_envs);
  rm->n_feat.assign(n_features, n_features + n_envs);
  rm->node_base.assign(n_envs + 1, 0);
  std::vector<int32_t> ob(n_envs + 1, 0), fb(n_envs + 1, 0);
  for (int b = 0; b < n_envs; ++b) {
    rm->node_base[b + 1] = rm->node_base[b] + n[b];
    ob[b + 1] = ob[b] + n_obstacles[b];
    fb[b + 1] = fb[b] + n_features[b];
    rm->n_max = std::max(rm->n_max, n[b]);
    rm->o_max = std::max(rm->o_max, n_obstacles[b]);
    rm->f_max = std::max(rm->f_max, n_features[b]);
  }
  const cudaMemcpyKind kind = (mem == MPAP_MEM_HOST) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CKC(rm_alloc_into(&rm->d_samples, sizeof(double) * N * row_stride, st));
  CKC(cudaMemcpyAsync(rm->d_samples, samples, sizeof(double) * N * row_stride, kind, st));
  CKC(rm_alloc_into(&rm->d_obst, sizeof(double) * std::max<int64_t>(O * 2 * d, 1), st));
  if (O) CKC(cudaMemcpyAsync(rm->d_obst, obstacles, sizeof(double) * O * 2 * d, kind, st));
  CKC(rm_alloc_into(&rm->d_feat, sizeof(double) * std::max<int64_t>(F * d, 1), st));
  if (F) CKC(cudaMemcpyAsync(rm->d_feat, features, sizeof(double) * F * d, kind, st));
  CKC(rm_alloc_into(&rm->d_obst_base, sizeof(int32_t) * (n_envs + 1), st));
  CKC(cudaMemcpyAsync(rm->d_obst_base, ob.data(), sizeof(int32_t) * (n_envs + 1), cudaMemcpyHostToDevice, st));
  CKC(rm_alloc_into(&rm->d_feat_base, sizeof(int32_t) * (n_envs + 1), st));
  CKC(cudaMemcpyAsync(rm->d_feat_base, fb.data(), sizeof(int32_t) * (n_envs + 1), cudaMemcpyHostToDevice, st));
  CKC(rm_alloc_into(&rm->d_node_base, sizeof(int64_t) * (n_envs + 1), st));
  CKC(cudaMemcpyAsync(rm->d_node_base, rm->node_base.data(), sizeof(int64_t) * (n_envs + 1),
                      cudaMemcpyHostToDevice, st));
  s = build_roadmap_device(rm, st);
  if (s != MPAP_OK) {
    mpap_roadmap_free(rm);
    return s;
  }
  // the stream-ordered allocation of row_ptr/edges must be visible to other
  // streams that later search this roadmap
  CKC(cudaStreamSynchronize(st));
  *out = rm;
  return MPAP_OK;
}

mpap_status mpap_build_roadmap(const double* samples, int32_t n, int32_t row_stride, const double* obstacles,
                               int32_t n_obstacles, const double* features, int32_t n_features, double r,
                               const mpap_params* params, int32_t mem, void* cuda_stream, mpap_roadmap** out) {
  return mpap_build_roadmap_batch(1, samples, &n, row_stride, obstacles, &n_obstacles, features, &n_features, r,
                                  params, mem, cuda_stream, out);
}

mpap_status mpap_roadmap_import(int32_t n, int32_t pos_dim, const double* positions, const int32_t* row_ptr,
                                const uint32_t* dst_coll, const float* w, const float* s, const float* c, double r,
                                void* cuda_stream, mpap_roadmap** out) {
  if (!out) return set_error(MPAP_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n < 1 || (pos_dim != 2 && pos_dim != 3) || !positions || !row_ptr)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad n/pos_dim/positions/row_ptr");
  if (!(r > 0.0) || !is_fin(r)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "r must be finite and > 0");
  if (row_ptr[0] != 0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "row_ptr[0] != 0");
  for (int32_t u = 0; u < n; ++u)
    if (row_ptr[u + 1] < row_ptr[u]) return set_error(MPAP_ERR_INVALID_ARGUMENT, "row_ptr decreasing");
  const int64_t nnz = row_ptr[n];
  if (nnz > 0 && (!dst_coll || !w || !s || !c)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL edge arrays");
  std::vector<EdgeRec> er((size_t)std::max<int64_t>(nnz, 1));
  for (int64_t k = 0; k < nnz; ++k) {
    if ((int64_t)(dst_coll[k] & 0x7fffffffu) >= n) return set_error(MPAP_ERR_INVALID_ARGUMENT, "dst out of range");
    if (!(w[k] >= 0.0f) || !(s[k] == s[k]) || !(c[k] >= 0.0f))
      return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad edge value");
    er[k].dst_coll = dst_coll[k];
    er[k].w = w[k];
    er[k].s = s[k];
    er[k].c = c[k];
  }
  for (int64_t k = 0; k < (int64_t)n * pos_dim; ++k)
    if (!is_fin(positions[k])) return set_error(MPAP_ERR_INVALID_ARGUMENT, "non-finite position");
  mpap_roadmap* rm = new (std::nothrow) mpap_roadmap();
  if (!rm) return set_error(MPAP_ERR_OUT_OF_MEMORY, "host allocation failed");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  CKC(cudaGetDevice(&rm->device));
  retain_pool_memory(rm->device);
  rm->B = 1;
  std::memset(&rm->prm, 0, sizeof(rm->prm));
  rm->prm.pos_dim = pos_dim;
  rm->prm.stride = pos_dim;
  rm->prm.r = r;
  rm->n.assign(1, n);
  rm->n_obst.assign(1, 0);
  rm->n_feat.assign(1, 0);
  rm->node_base = {0, n};
  rm->edge_base = {0, nnz};
  rm->n_max = n;
  int64_t nf = 0;
  for (int64_t k = 0; k < nnz; ++k) nf += (dst_coll[k] >> 31) == 0u;
  rm->nnz_free.assign(1, nf);
  rm->nnz_total = nnz;
  std::vector<int64_t> rp64(n + 1);
  for (int32_t u = 0; u <= n; ++u) rp64[u] = row_ptr[u];
  CKC(rm_alloc_into(&rm->d_samples, sizeof(double) * n * pos_dim, st));
  CKC(cudaMemcpyAsync(rm->d_samples, positions, sizeof(double) * n * pos_dim, cudaMemcpyHostToDevice, st));
  CKC(rm_alloc_into(&rm->d_node_base, sizeof(int64_t) * 2, st));
  CKC(cudaMemcpyAsync(rm->d_node_base, rm->node_base.data(), sizeof(int64_t) * 2, cudaMemcpyHostToDevice, st));
  CKC(rm_alloc_into(&rm->d_row_ptr, sizeof(int64_t) * (n + 1), st));
  CKC(cudaMemcpyAsync(rm->d_row_ptr, rp64.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
  CKC(rm_alloc_into(&rm->d_edges, sizeof(EdgeRec) * er.size(), st));
  CKC(cudaMemcpyAsync(rm->d_edges, er.data(), sizeof(EdgeRec) * er.size(), cudaMemcpyHostToDevice, st));
  CKC(cudaStreamSynchronize(st));
  *out = rm;
  return MPAP_OK;
}

int32_t mpap_roadmap_envs(const mpap_roadmap* rm) { return rm ? rm->B : 0; }

mpap_status mpap_roadmap_work(const mpap_roadmap* rm, uint64_t* counters, int32_t n) {
  if (!rm || !counters || n < 0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap/counters");
  for (int32_t i = 0; i < n; ++i) counters[i] = (i < kWorkCounters) ? (uint64_t)rm->work[i] : 0;
  return MPAP_OK;
}

mpap_status mpap_roadmap_info(const mpap_roadmap* rm, int32_t env, int32_t* n, int64_t* nnz, int64_t* nnz_free) {
  if (!rm || env < 0 || env >= rm->B) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap/env");
  if (n) *n = rm->n[env];
  if (nnz) *nnz = rm->edge_base[env + 1] - rm->edge_base[env];
  if (nnz_free) *nnz_free = rm->nnz_free[env];
  return MPAP_OK;
}

mpap_status mpap_roadmap_export(const mpap_roadmap* rm, int32_t env, int32_t* row_ptr, uint32_t* dst_coll, float* w,
                                float* s, float* c) {
  if (rm) {
    mpap_status se = ensure_evaluated(rm, nullptr);
    if (se != MPAP_OK) return se;
  }
  if (!rm || env < 0 || env >= rm->B || !row_ptr)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap/env/row_ptr");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  const int32_t ne = rm->n[env];
  std::vector<int64_t> rp(ne + 1);
  cudaError_t e = cudaMemcpy(rp.data(), rm->d_row_ptr + rm->node_base[env], sizeof(int64_t) * (ne + 1),
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_error(e, "export row_ptr");
  const int64_t e0 = rp[0], nnz = rp[ne] - rp[0];
  for (int32_t u = 0; u <= ne; ++u) row_ptr[u] = (int32_t)(rp[u] - e0);
  std::vector<EdgeRec> er((size_t)std::max<int64_t>(nnz, 1));
  if (nnz) {
    e = cudaMemcpy(er.data(), rm->d_edges + e0, sizeof(EdgeRec) * nnz, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_error(e, "export edges");
  }
  for (int64_t k = 0; k < nnz; ++k) {
    if (dst_coll) dst_coll[k] = er[k].dst_coll;
    if (w) w[k] = er[k].w;
    if (s) s[k] = er[k].s;
    if (c) c[k] = er[k].c;
  }
  return MPAP_OK;
}

// Multiset symmetric difference of two lists of k-double rows (exact compare).
static void sym_diff(const std::vector<double>& a, const std::vector<double>& b, int k, std::vector<double>& out) {
  auto rows = [k](const std::vector<double>& v) {
    std::vector<std::vector<double>> r(v.size() / k);
    for (size_t i = 0; i < r.size(); ++i) r[i].assign(v.begin() + i * k, v.begin() + (i + 1) * k);
    std::sort(r.begin(), r.end());
    return r;
  };
  const auto ra = rows(a), rb = rows(b);
  size_t i = 0, j = 0;
  while (i < ra.size() || j < rb.size()) {
    if (j == rb.size() || (i < ra.size() && ra[i] < rb[j])) {
      out.insert(out.end(), ra[i].begin(), ra[i].end());
      ++i;
    } else if (i == ra.size() || rb[j] < ra[i]) {
      out.insert(out.end(), rb[j].begin(), rb[j].end());
      ++j;
    } else {
      ++i;
      ++j;
    }
  }
}

// Replace env's segment of a concatenated per-env array (rows of k doubles).
static mpap_status splice_env(double** arr, int32_t** d_base, std::vector<int32_t>& counts, int env,
                              const std::vector<double>& seg, int k, cudaStream_t st) {
  const int B = (int)counts.size();
  std::vector<int32_t> base(B + 1, 0);
  for (int b = 0; b < B; ++b) base[b + 1] = base[b] + counts[b];
  const int32_t n_new = (int32_t)(seg.size() / k);
  const int64_t tot = (int64_t)base[B] - counts[env] + n_new;
  double* na = static_cast<double*>(rm_alloc(sizeof(double) * std::max<int64_t>(tot * k, 1), st));
  if (!na) return MPAP_ERR_OUT_OF_MEMORY;
  const int64_t head = (int64_t)base[env] * k, tail = ((int64_t)base[B] - base[env + 1]) * k;
  cudaError_t e = cudaSuccess;
  if (head) e = cudaMemcpyAsync(na, *arr, sizeof(double) * head, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && n_new)
    e = cudaMemcpyAsync(na + head, seg.data(), sizeof(double) * seg.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && tail)
    e = cudaMemcpyAsync(na + head + (int64_t)n_new * k, *arr + (int64_t)base[env + 1] * k, sizeof(double) * tail,
                        cudaMemcpyDeviceToDevice, st);
  counts[env] = n_new;
  for (int b = 0; b < B; ++b) base[b + 1] = base[b] + counts[b];
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(*d_base, base.data(), sizeof(int32_t) * (B + 1), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    rm_release(na);
    return cuda_error(e, "splice env arrays");
  }
  rm_release(*arr);
  *arr = na;
  return MPAP_OK;
}

mpap_status mpap_roadmap_update(mpap_roadmap* rm, int32_t env, const double* obstacles, int32_t n_obstacles,
                                const double* features, int32_t n_features, int32_t mem, void* cuda_stream,
                                int64_t* n_reevaluated) {
  if (n_reevaluated) *n_reevaluated = 0;
  if (!rm || env < 0 || env >= rm->B) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap/env");
  if (!rm->d_tau) return set_error(MPAP_ERR_INVALID_ARGUMENT, "imported roadmaps cannot be updated");
  if (mem != MPAP_MEM_HOST && mem != MPAP_MEM_DEVICE) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad mem space");
  if (n_obstacles < 0 || n_features < 0 || (n_obstacles > 0 && !obstacles) || (n_features > 0 && !features))
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad obstacle/feature arrays");
  {
    mpap_status se = check_env_sizes(rm->prm.pos_dim, n_obstacles, n_features);
    if (se != MPAP_OK) return se;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  {
    mpap_status se = ensure_evaluated(rm, st);
    if (se != MPAP_OK) return se;
  }
  const int d = rm->prm.pos_dim;
  std::vector<double> nbx((size_t)n_obstacles * 2 * d), nft((size_t)n_features * d);
  const cudaMemcpyKind kind = (mem == MPAP_MEM_HOST) ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost;
  cudaError_t e = cudaSuccess;
  if (n_obstacles) e = cudaMemcpy(nbx.data(), obstacles, sizeof(double) * nbx.size(), kind);
  if (e == cudaSuccess && n_features) e = cudaMemcpy(nft.data(), features, sizeof(double) * nft.size(), kind);
  if (e != cudaSuccess) return cuda_error(e, "update inputs");
  for (double x : nbx)
    if (!is_fin(x)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "non-finite obstacle");
  for (double x : nft)
    if (!is_fin(x)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "non-finite feature");
  for (int32_t o = 0; o < n_obstacles; ++o)
    for (int k = 0; k < d; ++k)
      if (!(nbx[(size_t)o * 2 * d + k] < nbx[(size_t)o * 2 * d + d + k]))
        return set_error(MPAP_ERR_INVALID_ARGUMENT, "obstacle with lo >= hi");
  // the old sets of this env
  cudaDeviceSynchronize();   // searches / builds reading the old arrays may be in flight
  int64_t ob = 0, fb = 0;
  for (int b = 0; b < env; ++b) {
    ob += rm->n_obst[b];
    fb += rm->n_feat[b];
  }
  std::vector<double> obx((size_t)rm->n_obst[env] * 2 * d), oft((size_t)rm->n_feat[env] * d);
  if (!obx.empty()) e = cudaMemcpy(obx.data(), rm->d_obst + ob * 2 * d, sizeof(double) * obx.size(),
                                   cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && !oft.empty())
    e = cudaMemcpy(oft.data(), rm->d_feat + fb * d, sizeof(double) * oft.size(), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_error(e, "update old sets");
  std::vector<double> cbox, cfeat;
  sym_diff(obx, nbx, 2 * d, cbox);
  sym_diff(oft, nft, d, cfeat);
  mpap_status s = MPAP_OK;
  if (!cbox.empty()) {
    s = splice_env(&rm->d_obst, &rm->d_obst_base, rm->n_obst, env, nbx, 2 * d, st);
    if (s != MPAP_OK) return s;
  }
  if (!cfeat.empty()) {
    s = splice_env(&rm->d_feat, &rm->d_feat_base, rm->n_feat, env, nft, d, st);
    if (s != MPAP_OK) return s;
  }
  rm->o_max = rm->f_max = 0;
  for (int b = 0; b < rm->B; ++b) {
    rm->o_max = std::max(rm->o_max, rm->n_obst[b]);
    rm->f_max = std::max(rm->f_max, rm->n_feat[b]);
  }
  return update_roadmap_device(rm, env, cbox, cfeat, n_reevaluated, st);
}

mpap_status mpap_roadmap_export_peaks(const mpap_roadmap* rm, int32_t env, float* S, float* C) {
  if (rm) {
    mpap_status se = ensure_evaluated(rm, nullptr);
    if (se != MPAP_OK) return se;
  }
  if (!rm || env < 0 || env >= rm->B) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap/env");
  if (!rm->d_peak) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap carries no peaks");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  const int64_t e0 = rm->edge_base[env], nnz = rm->edge_base[env + 1] - e0;
  if (nnz == 0) return MPAP_OK;
  std::vector<float2> pk((size_t)nnz);
  cudaError_t e = cudaMemcpy(pk.data(), rm->d_peak + e0, sizeof(float2) * nnz, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_error(e, "export peaks");
  for (int64_t k = 0; k < nnz; ++k) {
    if (S) S[k] = pk[k].x;
    if (C) C[k] = pk[k].y;
  }
  return MPAP_OK;
}

mpap_status mpap_roadmap_set_peaks(mpap_roadmap* rm, const float* S, const float* C) {
  if (!rm || rm->B != 1) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap (single env only)");
  const int64_t nnz = rm->nnz_total;
  if (nnz > 0 && (!S || !C)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL peak arrays");
  std::vector<float2> pk((size_t)std::max<int64_t>(nnz, 1));
  for (int64_t k = 0; k < nnz; ++k) {
    if (!(S[k] >= 0.0f) || !(C[k] >= 0.0f) || !std::isfinite(S[k]) || !std::isfinite(C[k]))
      return set_error(MPAP_ERR_INVALID_ARGUMENT, "peaks must be finite and >= 0");
    pk[k] = make_float2(S[k], C[k]);
  }
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  float2* d = nullptr;
  cudaDeviceSynchronize();   // searches of this roadmap may be in flight
  d = static_cast<float2*>(rm_alloc(sizeof(float2) * pk.size(), 0));
  if (!d) return MPAP_ERR_OUT_OF_MEMORY;
  cudaError_t e = cudaMemcpyAsync(d, pk.data(), sizeof(float2) * pk.size(), cudaMemcpyHostToDevice, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e != cudaSuccess) {
    rm_release(d);
    return cuda_error(e, "peak upload");
  }
  rm_release(rm->d_peak);
  rm->d_peak = d;
  return MPAP_OK;
}

static mpap_status check_query(const mpap_roadmap* rm, int32_t env, int32_t start, const mpap_goal* goal,
                               double beta) {
  if (env < 0 || env >= rm->B) return set_error(MPAP_ERR_INVALID_ARGUMENT, "env out of range");
  if (start < 0 || start >= rm->n[env]) return set_error(MPAP_ERR_INVALID_ARGUMENT, "start out of range");
  if (!goal) return set_error(MPAP_ERR_INVALID_ARGUMENT, "goal is NULL");
  if (std::isnan(beta) || beta < 0.0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "beta must be >= 0 (or +inf)");
  return MPAP_OK;
}

static void to_desc(QueryDesc& q, int32_t env, int32_t start, const mpap_goal* g, double beta, uint32_t flags) {
  q.flags = flags;
  q.pad = 0;
  q.env = env;
  q.start = start;
  q.beta = beta;
  for (int k = 0; k < 3; ++k) {
    q.goal_lo[k] = g->lo[k];
    q.goal_hi[k] = g->hi[k];
  }
}

static mpap_status check_flags(const mpap_roadmap* rm, uint32_t flags) {
  if (flags & ~MPAP_SEARCH_FORALL_T) return set_error(MPAP_ERR_INVALID_ARGUMENT, "unknown search flag");
  if ((flags & MPAP_SEARCH_FORALL_T) && !rm->d_peak)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "MPAP_SEARCH_FORALL_T needs edge peaks (mpap_roadmap_set_peaks)");
  return MPAP_OK;
}

mpap_status mpap_search(const mpap_roadmap* rm, int32_t env, int32_t start, const mpap_goal* goal,
                        double perception_bound, double lambda, int32_t* path, int32_t path_capacity,
                        mpap_result* result, mpap_wave* waves, int32_t waves_capacity, void* cuda_stream) {
  return mpap_search_ex(rm, env, start, goal, perception_bound, lambda, 0u, path, path_capacity, result, waves,
                        waves_capacity, cuda_stream);
}

mpap_status mpap_search_ex(const mpap_roadmap* rm, int32_t env, int32_t start, const mpap_goal* goal,
                           double perception_bound, double lambda, uint32_t flags, int32_t* path,
                           int32_t path_capacity, mpap_result* result, mpap_wave* waves, int32_t waves_capacity,
                           void* cuda_stream) {
  if (!rm || !result || (!path && path_capacity > 0) || path_capacity < 0)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL roadmap/result/path");
  if (!(lambda > 0.0) || lambda > 1.0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "lambda must be in (0, 1]");
  mpap_status s = check_query(rm, env, start, goal, perception_bound);
  if (s != MPAP_OK) return s;
  s = check_flags(rm, flags);
  if (s != MPAP_OK) return s;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  QueryDesc q;
  to_desc(q, env, start, goal, perception_bound, flags);
  std::vector<int32_t> pbuf((size_t)std::max(path_capacity, 1));
  mpap_result r{};
  s = search_batch_device(rm, 1, &q, lambda, pbuf.data(), std::max(path_capacity, 1), &r, waves, waves_capacity,
                          MPAP_MEM_HOST, static_cast<cudaStream_t>(cuda_stream));
  if (s != MPAP_OK) return s;
  *result = r;
  if (r.status == MPAP_OK) {
    if (r.path_len > path_capacity) {
      result->status = MPAP_ERR_BUFFER_TOO_SMALL;
      return set_error(MPAP_ERR_BUFFER_TOO_SMALL, "path_capacity too small");
    }
    std::memcpy(path, pbuf.data(), sizeof(int32_t) * r.path_len);
    return MPAP_OK;
  }
  if (r.status == MPAP_ERR_BUFFER_TOO_SMALL) return set_error(MPAP_ERR_BUFFER_TOO_SMALL, "path_capacity too small");
  if (r.status == MPAP_ERR_NO_FEASIBLE_PLAN) return set_error(MPAP_ERR_NO_FEASIBLE_PLAN, "no feasible plan");
  if (r.status == MPAP_ERR_NO_GOAL_NODE) return set_error(MPAP_ERR_NO_GOAL_NODE, "no node in the goal region");
  return set_error((mpap_status)r.status, "search failed");
}

mpap_status mpap_search_batch(const mpap_roadmap* rm, int32_t n_queries, const int32_t* envs, const int32_t* starts,
                              const mpap_goal* goals, const double* perception_bounds, double lambda, int32_t* paths,
                              int32_t path_capacity, mpap_result* results, int32_t mem, void* cuda_stream) {
  return mpap_search_batch_ex(rm, n_queries, envs, starts, goals, perception_bounds, lambda, 0u, paths,
                              path_capacity, results, mem, cuda_stream);
}

mpap_status mpap_search_batch_ex(const mpap_roadmap* rm, int32_t n_queries, const int32_t* envs,
                                 const int32_t* starts, const mpap_goal* goals, const double* perception_bounds,
                                 double lambda, uint32_t flags, int32_t* paths, int32_t path_capacity,
                                 mpap_result* results, int32_t mem, void* cuda_stream) {
  return mpap_search_batch_trace(rm, n_queries, envs, starts, goals, perception_bounds, lambda, flags, paths,
                                 path_capacity, results, mem, nullptr, 0, cuda_stream);
}

mpap_status mpap_search_batch_trace(const mpap_roadmap* rm, int32_t n_queries, const int32_t* envs,
                                    const int32_t* starts, const mpap_goal* goals, const double* perception_bounds,
                                    double lambda, uint32_t flags, int32_t* paths, int32_t path_capacity,
                                    mpap_result* results, int32_t mem, mpap_wave* waves, int32_t waves_capacity,
                                    void* cuda_stream) {
  if (waves_capacity < 0 || (waves_capacity > 0 && !waves))
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "waves is NULL or waves_capacity < 0");
  if (!rm || n_queries < 0 || (n_queries > 0 && (!envs || !starts || !goals || !perception_bounds || !paths ||
                                                  !results)) || path_capacity < 1)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL argument or path_capacity < 1");
  if (mem != MPAP_MEM_HOST && mem != MPAP_MEM_DEVICE) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad mem space");
  if (!(lambda > 0.0) || lambda > 1.0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "lambda must be in (0, 1]");
  mpap_status sf = check_flags(rm, flags);
  if (sf != MPAP_OK) return sf;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  std::vector<QueryDesc> qs(n_queries);
  for (int k = 0; k < n_queries; ++k) {
    mpap_status s = check_query(rm, envs[k], starts[k], &goals[k], perception_bounds[k]);
    if (s != MPAP_OK) return s;
    to_desc(qs[k], envs[k], starts[k], &goals[k], perception_bounds[k], flags);
  }
  return search_batch_device(rm, n_queries, qs.data(), lambda, paths, path_capacity, results,
                             waves_capacity > 0 ? waves : nullptr, waves_capacity, mem,
                             static_cast<cudaStream_t>(cuda_stream));
}


mpap_status mpap_mc_verify_batch(const mpap_roadmap* rm, int32_t n_plans, const int32_t* envs, const int32_t* paths,
                                 int32_t path_stride, const int32_t* path_lens, const mpap_mc_params* mc,
                                 uint64_t trial0, double* max_err, double* max_dev, mpap_mc_result* results,
                                 void* cuda_stream) {
  if (!rm || !mc || n_plans < 0 || (n_plans > 0 && (!envs || !paths || !path_lens || !results)) || path_stride < 1)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL argument, n_plans < 0 or path_stride < 1");
  if (!rm->d_samples || !rm->d_tau || rm->prm.dynamics != MPAP_DOUBLE_INTEGRATOR)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "Monte Carlo needs a double-integrator roadmap built with geometry");
  if (mc->trials < 1) return set_error(MPAP_ERR_INVALID_ARGUMENT, "trials must be >= 1");
  const double nonneg[] = {mc->sigma_imu, mc->sigma_vis, mc->p0_pos, mc->p0_vel, mc->delta};
  for (double x : nonneg)
    if (!is_fin(x) || x < 0.0) return set_error(MPAP_ERR_INVALID_ARGUMENT, "noise/covariance/delta must be finite >= 0");
  if (!is_fin(mc->u_max) || !(mc->u_max > 0.0) || !is_fin(mc->k_p) || !is_fin(mc->k_d))
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "u_max must be > 0 and gains finite");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  for (int32_t p = 0; p < n_plans; ++p) {
    if (envs[p] < 0 || envs[p] >= rm->B) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad env");
    if (path_lens[p] < 1 || path_lens[p] > path_stride) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad path_len");
    const int32_t* path = paths + (size_t)p * path_stride;
    for (int32_t j = 0; j < path_lens[p]; ++j)
      if (path[j] < 0 || path[j] >= rm->n[envs[p]]) return set_error(MPAP_ERR_INVALID_ARGUMENT, "node out of range");
  }
  mpap_status se = ensure_evaluated(rm, static_cast<cudaStream_t>(cuda_stream));
  if (se != MPAP_OK) return se;
  return mc_verify_device(rm, n_plans, envs, paths, path_stride, path_lens, mc, trial0, max_err, max_dev, results,
                          static_cast<cudaStream_t>(cuda_stream));
}

mpap_status mpap_roadmap_rows_evaluated(const mpap_roadmap* rm, int32_t env, int64_t* rows) {
  if (!rm || !rows || env < 0 || env >= rm->B) return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad roadmap/env/rows");
  if (!rm->lazy) {
    *rows = rm->n[env];
    return MPAP_OK;
  }
  std::vector<int32_t> r(rm->n[env]);
  cudaError_t e = cudaMemcpy(r.data(), rm->d_ready + rm->node_base[env], sizeof(int32_t) * r.size(),
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_error(e, "rows_evaluated");
  int64_t c = 0;
  for (int32_t x : r) c += (x == 1);
  *rows = c;
  return MPAP_OK;
}

mpap_status mpap_mc_verify(const mpap_roadmap* rm, int32_t env, const int32_t* path, int32_t path_len,
                           const mpap_mc_params* mc, uint64_t trial0, double* max_err, double* max_dev,
                           mpap_mc_result* result, void* cuda_stream) {
  if (!result || !path || path_len < 1) return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL result/path or path_len < 1");
  mpap_status s = mpap_mc_verify_batch(rm, 1, &env, path, path_len, &path_len, mc, trial0, max_err, max_dev, result,
                                       cuda_stream);
  if (s != MPAP_OK) return s;
  if (result->status != MPAP_OK) return set_error((mpap_status)result->status, "plan edge is not a collision-free roadmap edge");
  return MPAP_OK;
}

}  // extern "C"
