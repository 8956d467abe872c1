// paper_1705_02408_b200/csrc/mpap_internal.cuh -- internal declarations of
// libmpap.so (CUDA side only; the CPU oracle in oracle/ shares nothing with
// this file).  Public ABI: include/mpap.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "mpap.h"

namespace mpap {

constexpr int kMlpSize = 122;
constexpr int kWorkCounters = 16;

// Kernel-parameter copy of mpap_params plus derived constants; passed by value
// (lives in the constant bank, so every lane reads it as a broadcast).
struct DevParams {
  int pos_dim, dynamics, has_heading, heuristic;
  int stride;  // doubles per sample row
  int edge_peaks;  // compute per-edge (S, C) peaks (NEXT-3)
  int hoff;    // offset of (cos yaw, sin yaw) in a row
  double ws_lo[3], ws_hi[3];
  double control_weight, nominal_speed, dt, collision_dt, n_f, fov_cos_half, max_range;
  double mlp_gain, v_ref, w_ref;
  double r;
  int64_t row_lo, row_hi;  // global rows whose edges are built (row-sharded build); others get none
  double mlp[kMlpSize];
};

// One roadmap edge: 16 bytes, read with one LDG.128 by the search
// (SURVEY.md §8(a) a4).  x = dst | coll << 31, y = w (f32 bits), z = s, w = c.
struct __align__(16) EdgeRec {
  uint32_t dst_coll;
  float w, s, c;
};

// Output of the neighbour kernel: one r-disc entry before collision/heuristic.
struct __align__(16) NearRec {
  int32_t v;
  float w;      // (float)Cost(u,v)
  double tau;   // edge duration (kinematic: length/speed; DI: tau*)
};

}  // namespace mpap

struct mpap_roadmap {
  int device = 0;
  int B = 0;
  mpap::DevParams prm{};
  std::vector<int32_t> n;          // nodes per env
  std::vector<int64_t> node_base;  // first global row of each env (B+1)
  std::vector<int64_t> edge_base;  // first global edge of each env (B+1)
  std::vector<int32_t> n_obst, n_feat;
  std::vector<int64_t> nnz_free;   // collision-free edges per env
  int32_t n_max = 0, o_max = 0, f_max = 0;
  double* d_samples = nullptr;     // [sum n][stride]
  double* d_obst = nullptr;        // [sum O][2d]
  double* d_feat = nullptr;        // [sum F][d]
  int32_t* d_obst_base = nullptr;  // [B+1]
  int32_t* d_feat_base = nullptr;  // [B+1]
  int64_t* d_node_base = nullptr;  // [B+1]
  int64_t* d_row_ptr = nullptr;    // [sum n + 1] global edge offsets
  mpap::EdgeRec* d_edges = nullptr;
  double* d_tau = nullptr;         // [nnz_total] edge durations (NEXT-1 updates re-evaluate edges from it)
  int32_t* d_esrc = nullptr;       // [nnz_total] global source row of each edge (k_fold)
  float2* d_peak = nullptr;        // [nnz_total] (S, C) prefix maxima per edge (NEXT-3); may be null (import)
  int64_t nnz_total = 0;
  bool lazy = false;               // NEXT-1 part i: rows evaluated on first expansion (mpap_params.lazy_edges)
  int32_t* d_ready = nullptr;      // lazy: [sum n] 0 = not evaluated, 2 = requested, 1 = evaluated
  unsigned long long work[mpap::kWorkCounters] = {};  // build work counters (mpap_roadmap_work)
  cudaStream_t alloc_stream = nullptr;                 // stream the device arrays were allocated on
  // search capacities learned from earlier regrow-and-retry rounds on this
  // roadmap (staircase slots, labels, candidates); 0 = default
  mutable int hint_K = 0, hint_L = 0, hint_C = 0;
};

namespace mpap {
// MPAP_DEBUG_TIMING=1 prints host-side phase times to stderr (tuning aid).
struct HostTimer {
  const char* what;
  std::chrono::steady_clock::time_point t0;
  static bool on() {
    static int v = -1;
    if (v < 0) v = getenv("MPAP_DEBUG_TIMING") ? 1 : 0;
    return v == 1;
  }
  explicit HostTimer(const char* w) : what(w), t0(std::chrono::steady_clock::now()) {}
  ~HostTimer() {
    if (on())
      fprintf(stderr, "[mpap] %s %.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

// SM count of the current device
int device_sms();
// exclusive scan of int32 row counts -> int64 row offsets (k_scan)
cudaError_t scan_row_counts(const int32_t* cnt, int64_t n, int64_t* row_ptr, cudaStream_t st);

// launch bookkeeping shared by the translation units (host side)
void note_launch(int k = 1);
// search launches per team kind (mpap_search_launches): 0 grid, 1 cluster, 2 CTA
void note_team(int team);

// Optional per-kernel CUDA-event timing (mpap_prof_enable): a scope records
// an event pair on the launching stream around one kernel launch.
struct ProfScope {
  const char* name;
  cudaStream_t st;
  void* rec;
  ProfScope(const char* kernel, cudaStream_t stream);
  ~ProfScope();
};
mpap_status set_error(mpap_status s, const std::string& msg);
// keeps freed stream-ordered memory in the device pool (no OS round trip per call)
void retain_pool_memory(int device);
// Per-(device, stream, tag) scratch workspace that only grows: repeated calls
// on one stream reuse it (stream order serialises them); other streams get
// their own.  Returns nullptr on allocation failure.
void* workspace(cudaStream_t st, int tag, size_t bytes);
enum { WS_NEAR = 0, WS_SEARCH = 1, WS_KOFF = 2, WS_KV = 3, WS_FLIST = 4 };
// Device buffer cache for roadmap arrays (capi.cu).  Roadmaps are built and
// freed every step of a batched pipeline with the same sizes; growing the
// stream-ordered pool for them stalled the host for up to 0.5 s per call
// (measured), so released buffers are kept per device and reused
// best-fit (slack <= 1/8).  rm_alloc returns nullptr on failure (error set).
// rm_release requires that no device work still uses the buffer (callers
// synchronise first); beyond a cap (1/4 of device memory, MPAP_CACHE_MB) the
// buffer is returned to the driver.
void* rm_alloc(size_t bytes, cudaStream_t st);
void rm_release(void* p);
mpap_status cuda_error(cudaError_t e, const char* what);

// roadmap build (build_kernels.cu)
mpap_status build_roadmap_device(mpap_roadmap* rm, cudaStream_t st);
// NEXT-1: re-evaluate the edges of env affected by the changed boxes/features
// (host arrays); rm's obstacle/feature arrays already hold the new sets.
mpap_status update_roadmap_device(mpap_roadmap* rm, int env, const std::vector<double>& cbox,
                                  const std::vector<double>& cfeat, int64_t* n_reeval, cudaStream_t st);

// NEXT-1 part i: evaluate collision + heuristic of the listed global rows
// (device array d_rows[n_req]; d_rows == nullptr: every row not yet
// evaluated) of a lazy roadmap, marking them ready.
mpap_status evaluate_rows_device(mpap_roadmap* rm, const int32_t* d_rows, int64_t n_req, cudaStream_t st);

// search (search_kernels.cu)
struct QueryDesc {
  int32_t env, start;
  double beta;
  double goal_lo[3], goal_hi[3];
  uint32_t flags, pad;   // MPAP_SEARCH_* flags
};
mpap_status search_batch_device(const mpap_roadmap* rm, int32_t nq, const QueryDesc* h_queries,
                                double lambda, int32_t* paths, int32_t path_cap, mpap_result* results,
                                mpap_wave* h_waves, int32_t waves_cap, int32_t mem, cudaStream_t st);

// Monte Carlo verification (mc_kernels.cu; NEXT-4); arguments validated by capi.cu
mpap_status mc_verify_device(const mpap_roadmap* rm, int32_t n_plans, const int32_t* envs, const int32_t* paths,
                             int32_t path_stride, const int32_t* path_lens, const mpap_mc_params* mc,
                             uint64_t trial0, double* max_err, double* max_dev, mpap_mc_result* results,
                             cudaStream_t st);
}  // namespace mpap
