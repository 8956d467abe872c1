/*
 * include/mpap.h -- C ABI of libmpap.so, the B200 (sm_100a) hot path of MPAP
 * (Ichter, Landry, Schmerling, Pavone, "Perception-Aware Motion Planning via
 * Multiobjective Search on GPUs", arXiv 1705.02408; "P:n" = line n of the
 * paper source /root/reference/PAPER.md, cited for the reader -- nothing here
 * reads it at run time).
 *
 * Two calls carry the method (BASELINE.json north_star):
 *   mpap_build_roadmap*  -- Alg. 2 BuildGraph + Alg. 1 line 2,
 *                           the perception-heuristic precompute (P:178,
 *                           P:222-225): r_n-disc neighbour CSR with per-edge
 *                           cost, perception-heuristic summary and collision bit.
 *   mpap_search*         -- Alg. 3 Explore: group-marching
 *                           multiobjective (cost, h) search; returns the plan,
 *                           its cost and its perception value.
 * Numerics follow DESIGN.md §3 "Numeric contract" (bit-exact with the CPU
 * oracle in oracle/, which shares no code with this library).
 *
 * Conventions for every entry point:
 *   - returns mpap_status; never throws, never aborts the process;
 *   - on a non-OK status mpap_last_error() gives a thread-local detail string;
 *   - outputs are valid only on MPAP_OK, except where stated;
 *   - `cuda_stream` is a cudaStream_t (NULL = legacy default stream); all
 *     device work is ordered on it.  The device is the one current when
 *     mpap_build_roadmap* was called; the roadmap is bound to it.
 *   - pointer arguments documented as "mem space" are host pointers when
 *     mem == MPAP_MEM_HOST and device pointers when mem == MPAP_MEM_DEVICE;
 *     all other pointers are host pointers.  Inputs are borrowed (read during
 *     the call, never retained).
 */
#ifndef MPAP_H
#define MPAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MPAP_OK = 0,
  MPAP_ERR_INVALID_ARGUMENT = 1, /* a documented precondition failed            */
  MPAP_ERR_NO_GOAL_NODE = 2,     /* no node position in X_goal (R19)      */
  MPAP_ERR_NO_FEASIBLE_PLAN = 3, /* P_open emptied with no goal plan (A3.5) */
  MPAP_ERR_BUFFER_TOO_SMALL = 4, /* path_capacity too small; path_len = required */
  MPAP_ERR_OUT_OF_MEMORY = 5,    /* device allocation failed                     */
  MPAP_ERR_CUDA = 6              /* CUDA runtime error; see mpap_last_error()    */
} mpap_status;

enum { MPAP_MEM_HOST = 0, MPAP_MEM_DEVICE = 1 };

/* Cost(u,v) model (reading R7). */
enum { MPAP_KINEMATIC = 0, MPAP_DOUBLE_INTEGRATOR = 1 };

/* Perception heuristic (P:323-328 feature count; P:476-477 learned; R9-R12). */
enum {
  MPAP_PH_OMNI_COUNT = 0,         /* visible = in range and unobstructed           */
  MPAP_PH_FOV_VELOCITY_COUNT = 1, /* + in the FOV cone around the velocity         */
  MPAP_PH_FOV_HEADING_COUNT = 2,  /* + in the FOV cone around the interpolated yaw */
  MPAP_PH_FOV_HEADING_MLP = 3     /* heading count + learned-style 3-8-8-2 MLP      */
};

typedef struct {
  int32_t pos_dim;        /* d in {2, 3}                                            */
  int32_t dynamics;       /* MPAP_KINEMATIC or MPAP_DOUBLE_INTEGRATOR               */
  int32_t has_heading;    /* sample row ends with (cos yaw, sin yaw) (R21, N1)      */
  int32_t heuristic;      /* MPAP_PH_*                                             */
  double ws_lo[3], ws_hi[3]; /* workspace box; leaving it is a collision (R8)       */
  double control_weight;  /* r_u > 0 in J = int_0^tau (1 + r_u |u|^2) dt (R7)       */
  double nominal_speed;   /* > 0; kinematic edge duration = length / speed (R9)     */
  double dt;              /* > 0; heuristic timestep                        */
  double collision_dt;    /* > 0; polyline resolution of double-integrator edges    */
  double n_f;             /* > 0; features offsetting drift (P:325-327, 12 in paper) */
  double fov_cos_half;    /* in (0, 1]; cos of the FOV half angle           */
  double max_range;       /* > 0; feature range                         */
  const double *mlp;      /* MLP only: 122 doubles W1[8x3] b1[8] W2[8x8] b2[8]
                             W3[2x8] b3[2] (host memory); else may be NULL          */
  double mlp_gain;        /* gamma of R12                                           */
  double v_ref, w_ref;    /* > 0; MLP input scales (R12)                            */
  int32_t edge_peaks;     /* 0 or 1: also compute the per-edge peaks (S, C) that
                             MPAP_SEARCH_FORALL_T needs (NEXT-3; costs ~2.5% of the
                             build: two more running maxima per heuristic step)    */
  int32_t lazy_edges;     /* 0 or 1 (NEXT-1 part i): the build
                             computes Near + Cost only; collision bits and heuristic
                             summaries of a row are evaluated when a search
                             (mpap_search*, mpap_search_batch*) first expands a
                             plan at that node -- the search reads the same
                             (coll, s, c), so every plan is identical.  The search
                             suspends before a wave whose heads need rows, the
                             library evaluates the rows requested by all queries
                             of the call in one pass and resumes.  Export, update
                             and Monte Carlo first evaluate all remaining rows.   */
} mpap_params;

/* Opaque, device-resident, immutable after build: B >= 1 environments, each
 * with its own node set and CSR ("offline precomputation"). */
typedef struct mpap_roadmap mpap_roadmap;

/*
 * mpap_build_roadmap_batch -- Alg. 2 + heuristic precompute for B environments
 * sharing `r` and `params`.
 *   n_envs          B >= 1.
 *   samples         mem space; rows of env 0, then env 1, ...; row b,u has
 *                   row_stride doubles: p[d] (+ v[d] if double integrator)
 *                   (+ cos yaw, sin yaw if has_heading).  Row u = node u of its
 *                   env; x_init is whichever node the search names as start.
 *   n               host, [B]: node count of each env (>= 1).
 *   obstacles       mem space; [sum O_b][2d] closed boxes lo[d], hi[d].
 *   n_obstacles     host, [B] (>= 0).
 *   features        mem space; [sum F_b][d] feature positions.
 *   n_features      host, [B] (>= 0).
 *   r               r_n > 0, finite: Near(V,u,r) = {v: Cost(u,v) < r}.
 *   params          host; see mpap_params.
 *   mem             MPAP_MEM_HOST or MPAP_MEM_DEVICE for the three arrays.
 *   out             receives the roadmap handle; free with mpap_roadmap_free.
 * Errors: INVALID_ARGUMENT (null pointers, n < 1, pos_dim not 2/3, row_stride
 * too small, lo >= hi in a box, non-finite samples, r <= 0, params out of
 * range, an environment with more than 65535 features or whose features and
 * boxes exceed the edge kernels' per-warp shared-memory working set:
 * 16 (F4 (2 d + 7) + 6 d O4) + 8192 bytes <= 227 KB with F4, O4 = F, O rounded
 * up to a multiple of 4, e.g. F <= 796 at O = 200, d = 3), OUT_OF_MEMORY, CUDA.  Synchronises `cuda_stream` before
 * returning.
 */
mpap_status mpap_build_roadmap_batch(int32_t n_envs, const double *samples, const int32_t *n,
                                     int32_t row_stride, const double *obstacles,
                                     const int32_t *n_obstacles, const double *features,
                                     const int32_t *n_features, double r, const mpap_params *params,
                                     int32_t mem, void *cuda_stream, mpap_roadmap **out);

/* Single-environment form of the north_star call
 * mpap_build_roadmap(samples, obstacles, features, r): B = 1. */
mpap_status mpap_build_roadmap(const double *samples, int32_t n, int32_t row_stride,
                               const double *obstacles, int32_t n_obstacles,
                               const double *features, int32_t n_features, double r,
                               const mpap_params *params, int32_t mem, void *cuda_stream,
                               mpap_roadmap **out);

/*
 * mpap_build_roadmap_rows -- row-sharded build of one environment (SURVEY.md
 * §8(e); Alg. 2 is "embarrassingly parallel" over rows): the same
 * inputs as mpap_build_roadmap, but only rows [row_begin, row_end) get their
 * r-disc neighbours, collision bits and heuristic summaries (every sample is
 * still a candidate neighbour); the other rows have no edges.  Rank g of G
 * builds its block of rows; the blocks' CSRs (mpap_roadmap_export) are
 * all-gathered and concatenated in row order, which equals the single-GPU
 * build bit for bit, and the full CSR is wrapped with mpap_roadmap_import.
 * Errors: as mpap_build_roadmap, plus INVALID_ARGUMENT unless
 * 0 <= row_begin <= row_end <= n.
 */
mpap_status mpap_build_roadmap_rows(const double *samples, int32_t n, int32_t row_stride,
                                    const double *obstacles, int32_t n_obstacles,
                                    const double *features, int32_t n_features, double r,
                                    const mpap_params *params, int32_t row_begin, int32_t row_end,
                                    int32_t mem, void *cuda_stream, mpap_roadmap **out);

/* X_goal: closed box on position (reading R20). */
typedef struct { double lo[3], hi[3]; } mpap_goal;

typedef struct {
  int32_t status;     /* mpap_status of this query (OK or NO_FEASIBLE_PLAN ...)     */
  int32_t path_len;   /* nodes in the plan, start first (0 if no plan)              */
  int32_t waves;      /* non-empty groups expanded (reading R24)                    */
  int32_t retries;    /* capacity regrow-and-rerun rounds used (exact).  A search
                         starts at the capacities earlier searches on the same
                         roadmap needed, or, while its slot arena stays under 4
                         GB, earlier searches on the device (env
                         MPAP_SEARCH_NO_HINT=1 disables the latter); capacities
                         never change a result, only this count and the time  */
  float cost;         /* plan cost p.cost (f32 sum along the path, N5)               */
  float h;            /* plan perception value p.h (A3.21; R25)                      */
  float h_peak;       /* max node-prefix h along the plan (<= beta) (R25)            */
  float pad;
  int64_t relaxations;     /* (plan in G, collision-free edge) pairs (R23)           */
  int64_t labels_inserted; /* plans that survived RemoveDominated (A3.15)            */
} mpap_result;

/* Per-wave counters (DESIGN.md §3 "counters"), identical to the oracle's. */
typedef struct {
  int64_t i, group, relax, beta_pass, inserted, killed, touched, stair_sum;
} mpap_wave;

/*
 * mpap_search -- Alg. 3 Explore on environment `env` of `rm` (SURVEY.md §8(a)
 * rows a5-a10).
 *   start           x_init node index in [0, n_env).
 *   goal            host; X_goal box (only the first pos_dim axes are used).
 *   perception_bound beta in [0, +inf] (Eq. 2; A3.9 P:251); +inf = agnostic.
 *   lambda          group cost factor in (0, 1] (reading R1).
 *   path            host, [path_capacity]: node sequence start..goal.
 *   result          host; filled for OK and NO_FEASIBLE_PLAN (path_len = 0).
 *   waves, waves_capacity  optional host trace of per-wave counters (NULL/0 = off);
 *                   result->waves says how many were produced.
 * Returns OK, NO_FEASIBLE_PLAN, NO_GOAL_NODE, BUFFER_TOO_SMALL (result->path_len
 * = required length), INVALID_ARGUMENT, OUT_OF_MEMORY, CUDA.  Synchronises.
 */
mpap_status mpap_search(const mpap_roadmap *rm, int32_t env, int32_t start, const mpap_goal *goal,
                        double perception_bound, double lambda, int32_t *path, int32_t path_capacity,
                        mpap_result *result, mpap_wave *waves, int32_t waves_capacity,
                        void *cuda_stream);

/*
 * mpap_search_batch -- n_queries independent queries, one persistent CTA per
 * query at a time (dynamic scheduling), all on `cuda_stream`.
 *   envs, starts, goals, perception_bounds   host, [n_queries].
 *   paths           mem space, [n_queries][path_capacity] int32.
 *   results         mem space, [n_queries] mpap_result.
 *   mem             MPAP_MEM_HOST: synchronises, outputs on the host.
 *                   MPAP_MEM_DEVICE: asynchronous; outputs are written on the
 *                   device in stream order; the caller synchronises.
 * Returns OK if the batch executed; each query's outcome is results[q].status.
 * Row q of `paths` is defined for its first results[q].path_len entries (when
 * results[q].status is OK); entries past path_len are unspecified.  If a
 * query cannot run (OUT_OF_MEMORY at the capacity regrow limit, a CUDA
 * error), every other query's record is still written and the first such
 * status is returned.
 */
mpap_status mpap_search_batch(const mpap_roadmap *rm, int32_t n_queries, const int32_t *envs,
                              const int32_t *starts, const mpap_goal *goals,
                              const double *perception_bounds, double lambda, int32_t *paths,
                              int32_t path_capacity, mpap_result *results, int32_t mem,
                              void *cuda_stream);

/*
 * Search flags (mpap_search_ex / mpap_search_batch_ex).
 *   MPAP_SEARCH_FORALL_T  Eq. 2 bounds the perception heuristic for
 *       all t, not only at the roadmap nodes (reading R11, SURVEY.md §8(f)
 *       NEXT-3): an edge is relaxed only if, in addition to the A3.9 cutoff,
 *       every step of the clamp fold along it stays within the bound:
 *       max(C_e, h + S_e) <= beta (f32 sum and max, compared in f64), where
 *       (S_e, C_e) are the prefix maxima of the edge's summary (s, c)
 *       (mpap_roadmap_export_peaks).  The roadmap must carry peaks (built by
 *       mpap_build_roadmap*, or set by mpap_roadmap_set_peaks after import),
 *       else INVALID_ARGUMENT.
 */
#define MPAP_SEARCH_FORALL_T 1u

/* mpap_search with flags (0 = mpap_search). */
mpap_status mpap_search_ex(const mpap_roadmap *rm, int32_t env, int32_t start, const mpap_goal *goal,
                           double perception_bound, double lambda, uint32_t flags, int32_t *path,
                           int32_t path_capacity, mpap_result *result, mpap_wave *waves,
                           int32_t waves_capacity, void *cuda_stream);

/* mpap_search_batch with flags applied to every query (0 = mpap_search_batch). */
mpap_status mpap_search_batch_ex(const mpap_roadmap *rm, int32_t n_queries, const int32_t *envs,
                                 const int32_t *starts, const mpap_goal *goals,
                                 const double *perception_bounds, double lambda, uint32_t flags,
                                 int32_t *paths, int32_t path_capacity, mpap_result *results, int32_t mem,
                                 void *cuda_stream);

/*
 * mpap_search_batch_trace -- mpap_search_batch_ex that also records the
 * per-wave counters (SURVEY.md §8(c) counters; the mpap_wave of mpap_search)
 * of every query, in the same launch configuration as the untraced batch
 * (one cluster or one CTA per query; whole grid query by query for small
 * batches), with the counting template of the search kernels.
 *   waves           host, [n_queries][waves_capacity]; query q's waves k <
 *                   min(results[q].waves, waves_capacity) are written to
 *                   waves[q * waves_capacity + k]; the rest is unspecified.
 *   waves_capacity  >= 0 (0 = mpap_search_batch_ex).
 * Errors as mpap_search_batch_ex; INVALID_ARGUMENT for waves == NULL with a
 * positive capacity.  Synchronises before returning when waves_capacity > 0.
 */
mpap_status mpap_search_batch_trace(const mpap_roadmap *rm, int32_t n_queries, const int32_t *envs,
                                    const int32_t *starts, const mpap_goal *goals,
                                    const double *perception_bounds, double lambda, uint32_t flags,
                                    int32_t *paths, int32_t path_capacity, mpap_result *results, int32_t mem,
                                    mpap_wave *waves, int32_t waves_capacity, void *cuda_stream);

/*
 * Device-resident row blocks of a row-sharded build:
 * rank g builds rows [row_begin, row_end) with mpap_build_roadmap_rows, hands
 * its block to one NCCL all-gather as device arrays, and every rank assembles
 * the gathered blocks into a search roadmap on the device -- no host round
 * trip of the CSR.
 *
 * mpap_roadmap_block_device -- the block of `rm` (built by
 * mpap_build_roadmap_rows, one environment, not lazy):
 *   counts    device, [row_end - row_begin] int32: entries per row, in row order.
 *   edges     device, [capacity] 16-byte records {dst | coll << 31, f32 w, s, c}
 *             (the roadmap's own layout), the block's rows in order.
 *   capacity  records `edges` can hold (>= 0).
 *   nnz       out (host): the block's record count.
 * Errors: INVALID_ARGUMENT (NULL, not a one-environment eager build, another
 * device), BUFFER_TOO_SMALL (nnz > capacity: nothing written, *nnz set),
 * CUDA.  Synchronises `cuda_stream`.
 *
 * mpap_roadmap_assemble_device -- the device counterpart of
 * mpap_roadmap_import for n_blocks gathered blocks:
 *   n, pos_dim, positions  as mpap_roadmap_import (host positions).
 *   row_begin     host, [n_blocks + 1]: block b holds rows [row_begin[b],
 *                 row_begin[b + 1]); row_begin[0] = 0, row_begin[n_blocks] = n.
 *   counts        device, [n_blocks][counts_stride] int32 (block b's row
 *                 counts first in its slot; counts_stride >= every block's rows).
 *   edges         device, [n_blocks][edges_stride] 16-byte records (block b's
 *                 records first in its slot).
 *   r             r_n (> 0, finite).
 * The CSR is the concatenation of the blocks in row order (one scan of the
 * counts, one copy kernel).  Errors: INVALID_ARGUMENT (blocks not tiling [0,
 * n), a block wider than its slot, a dst out of range, bad positions / r),
 * OUT_OF_MEMORY, CUDA.  Synchronises `cuda_stream`; the inputs stay owned by
 * the caller. */
mpap_status mpap_roadmap_block_device(const mpap_roadmap *rm, int32_t *counts, void *edges, int64_t capacity,
                                      int64_t *nnz, void *cuda_stream);
mpap_status mpap_roadmap_assemble_device(int32_t n, int32_t pos_dim, const double *positions, int32_t n_blocks,
                                         const int32_t *row_begin, const int32_t *counts, int32_t counts_stride,
                                         const void *edges, int64_t edges_stride, double r, void *cuda_stream,
                                         mpap_roadmap **out);

/*
 * mpap_roadmap_import -- wrap a precomputed single-environment CSR (P:337:
 * neighbours and edge data "precomputed offline") so mpap_search can run on it.
 *   n, pos_dim      node count (>= 1) and position dimension (2 or 3).
 *   positions       host, [n][pos_dim] node positions (goal membership, R20).
 *   row_ptr         host, [n+1] non-decreasing, row_ptr[0] = 0.
 *   dst_coll, w, s, c  host, [row_ptr[n]]: dst | coll << 31 (dst < n), f32 w >= 0,
 *                   s, c >= 0 the tropical edge summary (R10).
 *   r               r_n used for the group threshold lambda r_n (> 0).
 * Errors: INVALID_ARGUMENT, OUT_OF_MEMORY, CUDA.  Synchronises.
 */
mpap_status mpap_roadmap_import(int32_t n, int32_t pos_dim, const double *positions, const int32_t *row_ptr,
                                const uint32_t *dst_coll, const float *w, const float *s, const float *c,
                                double r, void *cuda_stream, mpap_roadmap **out);

/* Environment count and per-env sizes: n nodes, nnz edges, nnz_free
 * collision-free edges. */
mpap_status mpap_roadmap_info(const mpap_roadmap *rm, int32_t env, int32_t *n, int64_t *nnz,
                              int64_t *nnz_free);
int32_t mpap_roadmap_envs(const mpap_roadmap *rm);

/* Work counters of the build that produced `rm` (summed over its envs),
 * counted by the kernels themselves; bench.py turns them into algorithmic
 * FP64 operation counts.  Index: 0 pairs scanned, 1 pairs
 * passing the double-integrator prefilter, 2 bisection iterations, 3 r-disc
 * edges, 4 collision segments, 5 collision slab tests, 6 heuristic steps,
 * 7 feature range tests, 8 FOV tests, 9 occlusion segments, 10 occlusion slab
 * tests, 11 MLP evaluations, 12 collision-free edges, 13 culling tests.
 * Writes min(n, 16) counters, zero-fills the rest. */
mpap_status mpap_roadmap_work(const mpap_roadmap *rm, uint64_t *counters, int32_t n);

/* Copy env's CSR to host buffers (parity/debug): row_ptr[n+1] (local edge
 * offsets), dst_coll[nnz] = dst | coll << 31, w, s, c [nnz] (f32). */
mpap_status mpap_roadmap_export(const mpap_roadmap *rm, int32_t env, int32_t *row_ptr,
                                uint32_t *dst_coll, float *w, float *s, float *c);

/*
 * mpap_roadmap_update -- online replanning:
 * replace environment `env`'s obstacle and feature sets and re-evaluate only
 * the edges whose collision bit or heuristic summary (and peaks) can change:
 * those whose trajectory bounding box, grown by max_range + 1e-3, overlaps a
 * changed box or feature (the multiset symmetric differences of the old and
 * new sets; exact value comparison).  Afterwards `rm` equals
 * mpap_build_roadmap* of the new environment bit for bit (the neighbour
 * structure and costs depend on the samples only).
 *   obstacles [n_obstacles][2d], features [n_features][d]: in `mem` space
 *                   (validated as in the build).
 *   n_reevaluated   out (may be NULL): number of edges re-evaluated.
 * Synchronises the device.  Errors: INVALID_ARGUMENT (bad env, arrays, an
 * imported roadmap, the size limits of mpap_build_roadmap_batch), OUT_OF_MEMORY,
 * CUDA.
 */
mpap_status mpap_roadmap_update(mpap_roadmap *rm, int32_t env, const double *obstacles, int32_t n_obstacles,
                                const double *features, int32_t n_features, int32_t mem, void *cuda_stream,
                                int64_t *n_reevaluated);

/* Copy env's per-edge peaks (S, C) to host [nnz] f32 each (NULL skips one):
 * S_e = max over prefixes of the increment sum (>= 0), C_e = max over steps of
 * the clamped fold from 0 (>= 0); zero for colliding edges.  INVALID_ARGUMENT
 * if the roadmap carries no peaks (imported without mpap_roadmap_set_peaks). */
mpap_status mpap_roadmap_export_peaks(const mpap_roadmap *rm, int32_t env, float *S, float *C);

/* Attach peaks to a single-env imported roadmap: host S, C [nnz] f32, finite,
 * >= 0.  Replaces any previous peaks.  Synchronises. */
mpap_status mpap_roadmap_set_peaks(mpap_roadmap *rm, const float *S, const float *C);

/*
 * Monte Carlo verification (Alg. 1 step 4; §3: "an
 * asymptotically exact probability of motion plan p satisfying a
 * localization error bound through MC sampling").
 * One trial simulates the double-integrator vehicle tracking the
 * plan's nominal trajectory (the edges' cubic trajectories, reading R7) with
 * feedback on its ESTIMATED state, an inertial estimate from a noisy
 * accelerometer and a translation-only 3D-to-3D position fix from
 * the features in view from the TRUE state, fused by a per-axis
 * Kalman filter.  Exact model, operation order and the counter-based
 * noise generator: DESIGN.md §4 readings R31-R36.
 */
typedef struct {
  int32_t trials;     /* trials per plan, >= 1                                  */
  int32_t pad;
  uint64_t seed;      /* noise stream key; trial t of every plan uses stream (seed, trial0 + t) */
  double sigma_imu;   /* accelerometer noise per axis (m/s^2), >= 0             */
  double sigma_vis;   /* feature relative-position noise per axis (m), >= 0     */
  double u_max;       /* per-axis control limit, > 0                            */
  double k_p, k_d;    /* tracking gains per axis (e.g. LQR), finite             */
  double p0_pos, p0_vel;  /* initial filter covariance diagonal, >= 0           */
  double delta;       /* localisation error bound delta_x_hat of Eq. 1   */
} mpap_mc_params;

typedef struct {
  int32_t status;     /* OK, or INVALID_ARGUMENT if a plan edge is not a
                         collision-free edge of the roadmap                      */
  int32_t trials;
  int64_t exceed;     /* trials with max_t |x_hat - x| >= delta                  */
  int64_t steps;      /* simulation steps per trial                             */
  int64_t fixes;      /* steps with >= 1 feature in view, summed over trials    */
  double p_hat;       /* exceed / trials                                */
} mpap_mc_result;

/*
 * mpap_mc_verify_batch -- MC verification of n_plans plans, all trials of
 * all plans in one launch (warp per trial).
 *   rm              a double-integrator roadmap built by mpap_build_roadmap*
 *                   (imported roadmaps carry no geometry: INVALID_ARGUMENT).
 *   envs            host, [n_plans] environment of each plan.
 *   paths           host, [n_plans][path_stride] node sequences (start first),
 *                   as returned by mpap_search_batch.
 *   path_lens       host, [n_plans], 1 <= len <= path_stride (len 1 = start in
 *                   goal: zero steps, zero errors).
 *   mc              host; trials, noise, gains, delta (validated).
 *   trial0          first trial id (trials are independent streams).
 *   max_err, max_dev  host, [n_plans][mc->trials] f64 each (NULL skips):
 *                   max over steps of |x_hat - x| and |x_nom - x|.
 *   results         host, [n_plans].
 * Returns OK if the batch executed (each plan's outcome in results[p].status),
 * INVALID_ARGUMENT for bad arguments, OUT_OF_MEMORY, CUDA.  Synchronises.
 */
mpap_status mpap_mc_verify_batch(const mpap_roadmap *rm, int32_t n_plans, const int32_t *envs,
                                 const int32_t *paths, int32_t path_stride, const int32_t *path_lens,
                                 const mpap_mc_params *mc, uint64_t trial0, double *max_err,
                                 double *max_dev, mpap_mc_result *results, void *cuda_stream);

/* Single-plan form: returns results->status (OK or INVALID_ARGUMENT for an
 * invalid plan) unless the call itself failed. */
mpap_status mpap_mc_verify(const mpap_roadmap *rm, int32_t env, const int32_t *path, int32_t path_len,
                           const mpap_mc_params *mc, uint64_t trial0, double *max_err, double *max_dev,
                           mpap_mc_result *result, void *cuda_stream);

/* Lazy roadmaps (mpap_params.lazy_edges): rows of env whose collision bits and
 * heuristic summaries have been evaluated so far (n for an eager roadmap). */
mpap_status mpap_roadmap_rows_evaluated(const mpap_roadmap *rm, int32_t env, int64_t *rows);

/* Releases the roadmap's device memory (NULL is a no-op).  Waits for the
 * device to be idle first (searches of this roadmap may be in flight). */
void mpap_roadmap_free(mpap_roadmap *rm);

const char *mpap_status_str(mpap_status s);
const char *mpap_last_error(void);

/* Number of kernel launches issued by this thread's calls so far (bench
 * evidence: "gpu_launches"). */
int64_t mpap_launch_count(void);

/* Search launches so far (all threads) per team kind -- evidence of which
 * launch configuration ran: team 0 = the whole grid on one query
 * (cooperative launch), 1 = one thread-block cluster per query, 2 = one CTA
 * per query.  Returns -1 for another team value. */
int64_t mpap_search_launches(int32_t team);

/* Per-kernel CUDA-event timing for measurement (bench.py): when enabled,
 * every kernel launch of this library is bracketed by an event pair recorded
 * on its launching stream.  mpap_prof_read synchronises those events and
 * returns the accumulated milliseconds and launch count of `kernel`
 * ("k_near", "k_scan", "k_collide", "k_heuristic", "k_fold",
 * "k_search", "k_mc"); returns 1 if it was seen. */
void mpap_prof_enable(int32_t on);
void mpap_prof_reset(void);
int32_t mpap_prof_read(const char *kernel, double *total_ms, int64_t *launches);

/* FP64 issue-rate microbenchmark on the current device (measurement only; the
 * roofline denominator of the FP64-bound build kernels):
 * kind 0 = DFMA, 1 = DADD, 2 = DMUL.  Writes the best of 5 timed launches as
 * instructions per second (one instruction = one op, the convention of
 * mpap_roadmap_work's counters) and that launch's milliseconds (ms may be
 * NULL).  INVALID_ARGUMENT for a NULL ops_per_s or an unknown kind; CUDA
 * errors as MPAP_ERR_CUDA. */
mpap_status mpap_prof_fp64_peak(int32_t kind, double *ops_per_s, double *ms);

#ifdef __cplusplus
}
#endif
#endif /* MPAP_H */
