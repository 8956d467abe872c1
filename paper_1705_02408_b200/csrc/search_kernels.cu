// paper_1705_02408_b200/csrc/search_kernels.cu -- Alg. 3 Explore on sm_100a.
//
// The group-marching multiobjective search of PAPER.md P:237-265 (text
// P:227-235).  A "team" runs one query: for a batch, one persistent CTA per
// query at a time (queries are pulled from an atomic work counter, so
// independent queries load-balance across the 148 SMs); for a single
// latency-bound query, the whole grid of a cooperative launch (grid.sync
// between phases).  Per wave (one non-empty group G_i):
//
//   expand   warp per plan p of G_i; the head's CSR row is streamed 32 edges
//            at a time with one 16-byte load per lane (A3.6-A3.8):
//              cost' = p.cost + w,  h' = max(c, p.h + s)       (PH; R10)
//            cutoff h' <= beta (A3.9); a candidate already dominated by the
//            node's current non-dominated staircase is dropped on the spot
//            (it cannot survive RemoveDominated); survivors are
//            appended with warp-aggregated atomics (ballot + popc).
//   group    per-destination counts -> atomic range allocation -> scatter,
//            so each touched node's candidates are contiguous.
//   merge    RemoveDominated (A3.15) as a set operation per touched
//            node -- old staircase entries dominated by a candidate die (open
//            ones are removed from P_open), candidates dominated by another
//            candidate are dropped, survivors get label ids and enter the
//            staircase and the pending open list.  Small nodes (<= 48
//            candidates and entries): one warp each, all-pairs in shared
//            memory, pulled from a work counter.  Large nodes: one whole CTA
//            each, O(k log k): bitonic sort, prefix-min scan for the
//            survivors, binary searches for the kills and the merged order.
//   advance  G_i is retired (A3.16), i <- i+1 (A3.17), and the pending list
//            is partitioned into G_{i+1} = {cost <= (i+1) lambda r_n} (A3.18)
//            with ballot compaction; empty groups are skipped exactly (R24).
// The loop stops when G holds a goal plan (A3.5) or nothing is open; the
// result is the minimum (cost, h, node sequence) plan over the goal nodes'
// staircases (A3.20-A3.21; R16).  Every per-wave decision depends only on
// sets, never on thread order (R14), so plans are bit-identical to the oracle.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "mpap_internal.cuh"

#ifndef MPAP_EXPAND_BATCH_META
#define MPAP_EXPAND_BATCH_META 1   // expand: plan metadata loaded 32 plans per warp at a time
#endif
#ifndef MPAP_MERGE_MONO
#define MPAP_MERGE_MONO 1   // CTA merge: per-thread bounds advance over consecutive old entries
#endif
#ifndef MPAP_MERGE_RANKSORT
#define MPAP_MERGE_RANKSORT 1   // CTA merge: warp sorts + rank merge (else one bitonic network)
#endif

namespace mpap {
namespace cg = cooperative_groups;

#define FULLM 0xffffffffu
constexpr int kST = 512;              // threads per search CTA
constexpr int kCluster = 8;           // largest CTAs per query in cluster mode (portable cluster size)
constexpr int kSeqQueries = 8;       // batches up to this size run query by query on the whole grid
constexpr int kSeqLargeN = 8000;     // ... and so do batches on one environment of at least this many nodes
constexpr int kSeqLargeMaxQ = 32;    //     of at most this many queries (C4 refinement rounds of 32 bounds,
                                     //     measured; larger batches fill the SMs with clusters / CTAs)
constexpr int kMaxTies = 32;           // (cost, h) ties listed for the R16 tie-break; more -> leader scan
constexpr int kMrgCap = 48;           // merge: a node's candidates / staircase staged in shared memory up to this size
constexpr int kBigC = 2048;           // CTA merge of a large node: candidates (power of two, 4 per thread)
constexpr int kBigM = 4096;           // ... and staircase entries (8 per thread); larger nodes take the warp path
enum : uint8_t { L_OPEN = 0, L_CLOSED = 1, L_DEAD = 2 };
enum { OVF_LABELS = 1, OVF_CAND = 2, OVF_STAIR = 4, OVF_RING = 8 };
constexpr int kRingMax = 8;           // bucket ring of ceil(1/lambda) + 3 lists; more -> pending-list scan
constexpr int kRetryBase = 100;       // result.status = kRetryBase + OVF_* mask

struct SlotCaps {
  int n;     // nodes per slot (max over envs)
  int K;     // staircase slots per node
  int L;     // label pool capacity
  int C;     // candidates per wave
  int R;     // bucket ring size (0: one pending list re-partitioned every wave)
};

struct SearchArgs {
  // roadmap
  const double* samples;
  const int64_t* node_base;
  const int32_t* n_env;
  const int64_t* row_ptr;
  const EdgeRec* edges;
  const float2* peak;   // per-edge (S, C) prefix maxima (NEXT-3); null if the roadmap has none
  int stride, pos_dim;
  double T;           // lambda * r_n (f64)
  // queries
  const QueryDesc* queries;
  const int32_t* qidx;   // query index list (retries run a subset)
  int nq;
  int* work;
  // slots
  SlotCaps caps;
  int4* labels;
  uint8_t* lstate;
  float2* stair_ch;    // two buffers per node (double-buffered merge)
  int32_t* stair_id;
  int32_t* stair_n;    // count | buffer parity << 30
  int32_t* cand_cnt;
  int32_t* cand_off;
  int4* cand;
  int4* cand_sorted;
  int32_t* touched;
  int32_t* tsmall;     // touched nodes merged by one warp each
  int32_t* tbig;       // touched nodes merged by one CTA each
  int32_t* tmid;       // touched nodes with <= 32 candidates but a large staircase: one warp each
  int32_t* G;
  int32_t* pend;
  int32_t* pend2;
  int32_t* ring;       // [R][L] open labels by cost bucket (caps.R > 0)
  int32_t* stamp;
  uint8_t* goal;
  // outputs
  int32_t* paths;
  int path_cap;
  mpap_result* results;
  mpap_wave* waves;
  int waves_cap;
  // NEXT-1 part i (lazy roadmap, whole-grid single query): rows are evaluated
  // on first expansion; the kernel suspends before a wave whose heads have
  // unevaluated rows and resumes after the host evaluated them
  int32_t* ready;   // [sum n] 1 = evaluated (null: eager roadmap)
  int32_t* req;     // requested global rows
  int* nreq;
  int resume;
};

struct Ctl {
  int q, psize, nsize, ncand, ntouched, nlabels, overflow, any_goal, calloc;
  int gs[2], gig[2];                // |G| and goal-in-G of the group of wave w: index w & 1
  int nsmall, nbig, snext, bnext;   // merge work lists (small: warp per node, pulled from snext; big: CTA per
                                    // node, pulled from bnext)
  int nmid, mnext;                  // mid: warp per node (binary searches), pulled from mnext
  int rcount[kRingMax];             // bucket ring list lengths
  long long i, minb;
  unsigned long long relax, bpass, tcount, ssum, inserted, killed;
  unsigned long long relax_total, inserted_total;
  int waves;
  int suspended, pswap;   // lazy: suspended before a wave; pending lists swapped at suspension
  int need;               // lazy: some head of G_i has an unevaluated row
  unsigned long long best_key;
  int nties;
  int ties[kMaxTies];
};

// A team runs one query: a CTA (batched queries, __syncthreads) or the whole
// grid of a cooperative launch (a single latency-bound query, grid.sync).
struct CtaTeam {
  __device__ __forceinline__ int cta() const { return 0; }
  __device__ __forceinline__ int ncta() const { return 1; }
  __device__ __forceinline__ int rank() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ int warp() const { return threadIdx.x >> 5; }
  __device__ __forceinline__ int nwarps() const { return blockDim.x >> 5; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct GridTeam {
  __device__ __forceinline__ int cta() const { return blockIdx.x; }
  __device__ __forceinline__ int ncta() const { return gridDim.x; }
  __device__ __forceinline__ int rank() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int size() const { return gridDim.x * blockDim.x; }
  __device__ __forceinline__ int warp() const { return rank() >> 5; }
  __device__ __forceinline__ int nwarps() const { return size() >> 5; }
  __device__ __forceinline__ void sync() const { cg::this_grid().sync(); }
};

// A thread-block cluster (hardware barrier across its CTAs, which run on
// different SMs); used for batches with fewer queries than resident CTAs.
struct ClusterTeam {
  __device__ __forceinline__ int cta() const { return (int)cg::this_cluster().block_rank(); }
  __device__ __forceinline__ int ncta() const { return (int)cg::this_cluster().num_blocks(); }
  __device__ __forceinline__ int rank() const {
    return (int)cg::this_cluster().block_rank() * blockDim.x + threadIdx.x;
  }
  __device__ __forceinline__ int size() const { return (int)cg::this_cluster().num_blocks() * blockDim.x; }
  __device__ __forceinline__ int warp() const { return rank() >> 5; }
  __device__ __forceinline__ int nwarps() const { return size() >> 5; }
  __device__ __forceinline__ void sync() const { cg::this_cluster().sync(); }
};

// Debug bounds checks (compute-sanitizer is closed on this pool): a build with
// -DMPAP_DEBUG_CHECKS=1 counts every out-of-range store index of the search
// kernels in g_dcheck_fail (read back after each search; a non-zero count is
// reported as MPAP_ERR_CUDA).  Compiled out otherwise.
#ifndef MPAP_DEBUG_CHECKS
#define MPAP_DEBUG_CHECKS 0
#endif
__device__ unsigned long long g_dcheck_fail = 0;
#define DCHECK(cond) do { if (MPAP_DEBUG_CHECKS && !(cond)) atomicAdd(&g_dcheck_fail, 1ull); } while (0)
// Per-wave phase timestamps of a single (whole-grid) query, debug builds
// only (printed by the host when MPAP_PHASE_LOG is set): globaltimer after
// each phase barrier, and the merge work split.
constexpr int kPhaseWaves = 256;
__device__ unsigned long long g_phase[kPhaseWaves][8];
// debug builds: cycles of cta_merge's steps summed over large nodes (thread 0's
// clock: load+sort, survivors, kills, merged order + labels, tail), and count
__device__ unsigned long long g_merge_cyc[6];
#define MERGE_MARK(i) do { if (MPAP_DEBUG_CHECKS && tid == 0) { const unsigned long long c_ = clock64(); \
    atomicAdd(&g_merge_cyc[i], c_ - mk_); mk_ = c_; } } while (0)
__device__ int g_phase_stat[kPhaseWaves][4];   // nbig, nsmall, max candidates, max staircase of a big node
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PHASE_MARK(k) do { if (MPAP_DEBUG_CHECKS && leader && A.nq == 1 && wave < kPhaseWaves) g_phase[wave][k] = gtimer(); } while (0)

// control words are re-read after every team barrier
template <typename T>
__device__ __forceinline__ T vld(const T& x) { return *(const volatile T*)&x; }

__device__ __forceinline__ unsigned lane_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ long long bucket_of(float cost, double T) {
  const double c = (double)cost;
  long long b = (long long)ceil(c / T);
  if (b < 0) b = 0;
  while (b > 0 && c <= (double)(b - 1) * T) --b;
  while (c > (double)b * T) ++b;
  return b;
}

// Partition src -> (G if cost <= inext*T else dst).  Tracks the goal flag of
// G and the minimum bucket of dst.  Dead labels are dropped (lazy deletion).
template <typename Team>
__device__ void partition(const Team& team, const SearchArgs& A, Ctl* S, const int32_t* src, int nsrc, int32_t* G,
                          int32_t* dst, long long inext, const int4* labels, const uint8_t* lstate,
                          const uint8_t* goal, int tp) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lane_lt();
  const double thr = (double)inext * A.T;
  long long myminb = LLONG_MAX;
  bool mygoal = false;
  for (int k0 = team.warp() * 32; k0 < nsrc; k0 += team.nwarps() * 32) {
    const int k = k0 + lane;
    bool toG = false, toD = false;
    int id = -1;
    if (k < nsrc) {
      id = src[k];
      if (lstate[id] == L_OPEN) {
        const int4 lb = labels[id];
        const float cost = __int_as_float(lb.z);
        if ((double)cost <= thr) {
          toG = true;
          if (goal[lb.x]) mygoal = true;
        } else {
          toD = true;
          myminb = min(myminb, bucket_of(cost, A.T));
        }
      }
    }
    const unsigned mg = __ballot_sync(FULLM, toG);
    const unsigned md = __ballot_sync(FULLM, toD);
    int bg = 0, bd = 0;
    if (lane == 0) {
      if (mg) bg = atomicAdd(&S->gs[tp], __popc(mg));
      if (md) bd = atomicAdd(&S->nsize, __popc(md));
    }
    bg = __shfl_sync(FULLM, bg, 0);
    bd = __shfl_sync(FULLM, bd, 0);
    if (toG) { DCHECK(bg + __popc(mg & lt) < A.caps.L); G[bg + __popc(mg & lt)] = id; }
    if (toD) { DCHECK(bd + __popc(md & lt) < A.caps.L); dst[bd + __popc(md & lt)] = id; }
  }
  if (mygoal) S->gig[tp] = 1;
  if (myminb != LLONG_MAX) atomicMin(&S->minb, myminb);
}

// Staircase of node x: count and buffer from sn[x]; entries sorted by
// (cost ascending, h descending).  In a non-dominated set the h values of
// successive cost groups strictly decrease, so min{h : cost < c} is the h of
// the last entry with cost < c.
constexpr int kStairCountMask = (1 << 30) - 1;
__device__ __forceinline__ size_t stair_base(int snx, int x, int n, int K) {
  return ((size_t)(snx >> 30) * n + x) * (size_t)K;
}
__device__ __forceinline__ bool key_less(float ac, float ah, float bc, float bh) {
  return ac < bc || (ac == bc && ah > bh);
}

// Where a new open plan goes (A3.11 "P_open <- P_open + q"): the pending list
// re-partitioned every wave, or -- the paper's cost-thresholded buckets
// -- the ring list of its group index b = max(b(cost), i + 1), so the
// next group is one list (A3.18, reading R3).  b <= i + ceil(1/lambda) + 1
// since an edge costs less than r_n (f32 rounding included); a plan beyond
// the ring (not expected) flags OVF_RING and the query reruns on the list.
struct Pusher {
  int32_t* pend;
  int32_t* ring;
  int R, L;
  double T;
  long long i;
};

// Full warp; the lanes with v push plan `id` of cost c.
__device__ void push_open(Ctl* S, const Pusher& P, bool v, int id, float c) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lane_lt();
  if (P.R == 0) {
    const unsigned m = __ballot_sync(FULLM, v);
    if (!m) return;
    const int lead = __ffs(m) - 1;
    int base = 0;
    if (lane == lead) base = atomicAdd(&S->psize, __popc(m));
    base = __shfl_sync(FULLM, base, lead);
    if (v) P.pend[base + __popc(m & lt)] = id;
    return;
  }
  int slot = -1;
  if (v) {
    long long b = bucket_of(c, P.T);
    if (b < P.i + 1) b = P.i + 1;
    if (b > P.i + P.R) {
      atomicOr(&S->overflow, OVF_RING);
      v = false;
    } else {
      slot = (int)(b % P.R);
    }
  }
  unsigned pending = __ballot_sync(FULLM, v);
  while (pending) {   // warp-aggregated append per ring list
    const int lead = __ffs(pending) - 1;
    const int ls = __shfl_sync(FULLM, slot, lead);
    const bool mine = v && slot == ls;
    const unsigned m = __ballot_sync(FULLM, mine);
    int base = 0;
    if (lane == lead) base = atomicAdd(&S->rcount[ls], __popc(m));
    base = __shfl_sync(FULLM, base, lead);
    if (mine) P.ring[(size_t)ls * P.L + base + __popc(m & lt)] = id;
    pending &= ~m;
  }
}

// ---------------------------------------------------------------------------
// CTA-cooperative merge of one large node (RemoveDominated + insert, A3.15,
// P:193) -- the same set result as the warp path, in O(k log k):
//   1. the node's candidates are bitonic-sorted by (cost asc, h desc, parent);
//   2. candidate q survives iff min{h_r : cost_r < cost_q} > h_q (prefix-min
//      scan of h, read at the start of q's equal-cost group);
//   3. survivors form a staircase, so the cheapest-h survivor of cost < c is
//      the last one of cost < c: an old entry o dies iff that survivor has
//      h <= o.h (binary search);
//   4. merged order: old alive entry j goes to (alive entries before j) +
//      (survivors with key < o); survivor q to q + (alive entries with key <=
//      q) -- both by binary search, alive counts from a prefix sum.
// ---------------------------------------------------------------------------
struct BigSmem {
  int4 c[kBigC];          // candidates (x, cost, h, parent); survivors compacted in place
  float pm[kBigC];        // inclusive prefix minimum of h over the sorted candidates
  int gs[kBigC];          // start index of each candidate's equal-cost group
  int ap[kBigM + 1];      // alive old entries before j (the old staircase itself is read from global memory)
  float fscr[32];
  int iscr[32];
  int bc[2];
};
constexpr size_t kBigSmem = sizeof(BigSmem);

__device__ __forceinline__ bool cand_less(const int4& a, const int4& b) {
  const float ac = __int_as_float(a.y), bc = __int_as_float(b.y);
  const float ah = __int_as_float(a.z), bh = __int_as_float(b.z);
  return ac < bc || (ac == bc && (ah > bh || (ah == bh && a.w < b.w)));
}

// Block-wide exclusive scans (blockDim.x threads, a multiple of 32).
__device__ __forceinline__ int block_excl_sum(int v, int* scr, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULLM, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scr[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < nwb ? scr[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULLM, t, o);
      if (lane >= o) t += y;
    }
    scr[lane] = t;
  }
  __syncthreads();
  const int r = (w > 0 ? scr[w - 1] : 0) + x - v;
  *total = scr[nwb - 1];
  __syncthreads();
  return r;
}
__device__ __forceinline__ int4 shfl_xor4(const int4& v, int j) {
  return make_int4(__shfl_xor_sync(FULLM, v.x, j), __shfl_xor_sync(FULLM, v.y, j), __shfl_xor_sync(FULLM, v.z, j),
                   __shfl_xor_sync(FULLM, v.w, j));
}

// Block-wide exclusive prefix minimum (float) and maximum (int) in one pass.
__device__ __forceinline__ void block_excl_min_max(float vmin, int vmax, float* fscr, int* iscr, float& rmin,
                                                   int& rmax) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  float x = vmin;
  int y = vmax;
  for (int o = 1; o < 32; o <<= 1) {
    const float a = __shfl_up_sync(FULLM, x, o);
    const int b = __shfl_up_sync(FULLM, y, o);
    if (lane >= o) { x = fminf(x, a); y = max(y, b); }
  }
  const float ex = __shfl_up_sync(FULLM, x, 1);
  const int ey = __shfl_up_sync(FULLM, y, 1);
  if (lane == 31) { fscr[w] = x; iscr[w] = y; }
  __syncthreads();
  if (w == 0) {
    float t = lane < nwb ? fscr[lane] : __int_as_float(0x7f800000);
    int u = lane < nwb ? iscr[lane] : INT_MIN;
    for (int o = 1; o < 32; o <<= 1) {
      const float a = __shfl_up_sync(FULLM, t, o);
      const int b = __shfl_up_sync(FULLM, u, o);
      if (lane >= o) { t = fminf(t, a); u = max(u, b); }
    }
    fscr[lane] = t;
    iscr[lane] = u;
  }
  __syncthreads();
  float r = (lane > 0) ? ex : __int_as_float(0x7f800000);
  int q = (lane > 0) ? ey : INT_MIN;
  if (w > 0) { r = fminf(r, fscr[w - 1]); q = max(q, iscr[w - 1]); }
  __syncthreads();
  rmin = r;
  rmax = q;
}

__device__ void cta_merge(Ctl* S, const SlotCaps& C, int x, int n, const int4* cs, const int32_t* coff,
                          const int32_t* ccnt, float2* sch, int32_t* sid, int32_t* sn, int4* labels,
                          uint8_t* lstate, const Pusher& PU, unsigned long long& my_ins,
                          unsigned long long& my_kill) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  BigSmem& B = *reinterpret_cast<BigSmem*>(s_dyn);
  const int tid = threadIdx.x, bd = blockDim.x;
  constexpr int EC = kBigC / kST, EM = kBigM / kST;   // elements per thread
  unsigned long long mk_ = MPAP_DEBUG_CHECKS ? clock64() : 0ull;
  const int kc = ccnt[x];
  const int beg = coff[x] - kc;
  const int snx = sn[x];
  const int m = snx & kStairCountMask;
  const int par = snx >> 30;
  const float2* st = sch + stair_base(snx, x, n, C.K);
  const int32_t* si = sid + stair_base(snx, x, n, C.K);
  float2* nst = sch + ((size_t)(par ^ 1) * n + x) * (size_t)C.K;
  int32_t* nsi = sid + ((size_t)(par ^ 1) * n + x) * (size_t)C.K;
  int p2 = 2;
  while (p2 < kc) p2 <<= 1;
  const int4 pad = make_int4(x, 0x7f800000, (int)0xff800000, INT_MAX);   // +inf cost: sorts last
  // 1. bitonic sort ascending by (cost, -h, parent)
#if MPAP_MERGE_RANKSORT
  if (p2 <= bd) {
    // one element per thread: each warp sorts its 32 by shuffles (bitonic),
    // then every element's rank = its place in its run + how many elements
    // of each other run precede it (binary searches in shared memory; the
    // order is strict on candidates, pads sort last and rank >= kc)
    int4 v = (tid < kc) ? cs[beg + tid] : pad;
    const int lane = tid & 31, w = tid >> 5, nr = (p2 + 31) >> 5;
    for (int k = 2; k <= 32; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        // every candidate of the node has the same .x (the node): 3 shuffles
        const int4 o = make_int4(v.x, __shfl_xor_sync(FULLM, v.y, j), __shfl_xor_sync(FULLM, v.z, j),
                                 __shfl_xor_sync(FULLM, v.w, j));
        const bool up = (lane & k) == 0;
        const bool sw = ((lane & j) == 0) ? (cand_less(o, v) == up) : (cand_less(v, o) == up);
        if (sw) v = o;
      }
    }
    int4* runs = B.c + bd;
    runs[tid] = v;
    __syncthreads();
    if (w < nr) {
      int rank = lane;
      for (int r = 0; r < nr; ++r) {
        if (r == w) continue;
        const int4* rr = runs + r * 32;
        int lo = 0, hi = 32;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (cand_less(rr[mid], v)) lo = mid + 1; else hi = mid;
        }
        rank += lo;
      }
      if (rank < kc) B.c[rank] = v;
    }
    __syncthreads();
#else
  if (p2 <= bd) {
    // one element per thread in registers: partners closer than 32 by
    // shuffles, farther ones through two alternating shared-memory buffers
    // (one barrier per such step); the same compare-exchange network
    int4 v = (tid < kc) ? cs[beg + tid] : pad;
    int boff = 0;   // alternating halves B.c[0, bd) and B.c[bd, 2 bd)
    for (int k = 2; k <= p2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        int4 o;
        if (j >= 32) {
          B.c[boff + tid] = v;
          __syncthreads();
          o = B.c[boff + (tid ^ j)];
          boff ^= bd;
        } else {
          o = shfl_xor4(v, j);
        }
        // pair (i, i ^ j), i the lower index: swap iff cand_less(c[i ^ j], c[i]) == ((i & k) == 0)
        const bool up = (tid & k) == 0;
        const bool sw = ((tid & j) == 0) ? (cand_less(o, v) == up) : (cand_less(v, o) == up);
        if (sw) v = o;
      }
    }
    __syncthreads();   // the last exchange buffer's reads are done
    if (tid < p2) B.c[tid] = v;
    __syncthreads();
#endif
  } else {
  for (int i = tid; i < p2; i += bd) B.c[i] = (i < kc) ? cs[beg + i] : pad;
  __syncthreads();
  for (int k = 2; k <= p2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < p2; i += bd) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int4 a = B.c[i], b = B.c[ixj];
          if (cand_less(b, a) == ((i & k) == 0)) {
            B.c[i] = b;
            B.c[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  }
  MERGE_MARK(0);
  // 2. survivors: prefix min of h and equal-cost group starts
  int4 cq[EC];
  float lmin = __int_as_float(0x7f800000);
  int lmax = 0;
#pragma unroll
  for (int r = 0; r < EC; ++r) {
    const int i = tid * EC + r;
    cq[r] = B.c[i];
    if (i < kc) {
      lmin = fminf(lmin, __int_as_float(cq[r].z));
      if (i == 0 || __int_as_float(B.c[i - 1].y) != __int_as_float(cq[r].y)) lmax = i;
    }
  }
  float run;
  int gstart;
  block_excl_min_max(lmin, lmax, B.fscr, B.iscr, run, gstart);
  if (gstart < 0) gstart = 0;
#pragma unroll
  for (int r = 0; r < EC; ++r) {
    const int i = tid * EC + r;
    if (i < kc) {
      run = fminf(run, __int_as_float(cq[r].z));
      if (i == 0 || __int_as_float(B.c[i - 1].y) != __int_as_float(cq[r].y)) gstart = i;
      B.pm[i] = run;
      B.gs[i] = gstart;
    }
  }
  __syncthreads();
  bool surv[EC];
  int nloc = 0;
#pragma unroll
  for (int r = 0; r < EC; ++r) {
    const int i = tid * EC + r;
    surv[r] = false;
    if (i < kc) {
      const int g = B.gs[i];
      surv[r] = (g == 0) || (B.pm[g - 1] > __int_as_float(cq[r].z));
      nloc += surv[r] ? 1 : 0;
    }
  }
  int ns = 0;
  int spos = block_excl_sum(nloc, B.iscr, &ns);   // (its barriers also order the reads of B.c above)
#pragma unroll
  for (int r = 0; r < EC; ++r)
    if (surv[r]) B.c[spos++] = cq[r];
  __syncthreads();
  MERGE_MARK(1);
  // 3. kills of old entries
  bool alive[EM];
  int aloc = 0;
#if MPAP_MERGE_MONO
  int lo3 = -1;   // this thread's entries are consecutive and sorted: the bound only moves forward
#endif
#pragma unroll
  for (int r = 0; r < EM; ++r) {
    const int j = tid * EM + r;
    alive[r] = false;
    if (j < m) {
      const float2 o = st[j];
#if MPAP_MERGE_MONO
      int lo = lo3;   // first survivor with cost >= o.x
      if (lo < 0) {
        int hi = ns;
        lo = 0;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__int_as_float(B.c[mid].y) < o.x) lo = mid + 1; else hi = mid;
        }
      } else {
        while (lo < ns && __int_as_float(B.c[lo].y) < o.x) ++lo;
      }
      lo3 = lo;
#else
      int lo = 0, hi = ns;   // first survivor with cost >= o.x
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__int_as_float(B.c[mid].y) < o.x) lo = mid + 1; else hi = mid;
      }
#endif
      const bool dead = lo > 0 && __int_as_float(B.c[lo - 1].z) <= o.y;
      alive[r] = !dead;
      aloc += alive[r] ? 1 : 0;
      if (dead) {
        const int oid = si[j];
        if (lstate[oid] == L_OPEN) {
          lstate[oid] = L_DEAD;
          ++my_kill;
        }
      }
    }
  }
  int na = 0;
  int apos = block_excl_sum(aloc, B.iscr, &na);
#pragma unroll
  for (int r = 0; r < EM; ++r) {
    const int j = tid * EM + r;
    if (j < m) {
      B.ap[j] = apos;
      apos += alive[r] ? 1 : 0;
    }
  }
  if (tid == 0) {
    B.ap[m] = na;
    B.bc[0] = atomicAdd(&S->nlabels, ns);
  }
  __syncthreads();
  MERGE_MARK(2);
  // 4. merged staircase in the other buffer; survivors get labels
#if MPAP_MERGE_MONO
  int lo4 = -1;
#endif
#pragma unroll
  for (int r = 0; r < EM; ++r) {
    const int j = tid * EM + r;
    if (j < m && alive[r]) {
      const float2 o = st[j];
#if MPAP_MERGE_MONO
      int lo = lo4;   // survivors with key < o (non-decreasing over the thread's entries)
      if (lo < 0) {
        int hi = ns;
        lo = 0;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (key_less(__int_as_float(B.c[mid].y), __int_as_float(B.c[mid].z), o.x, o.y)) lo = mid + 1; else hi = mid;
        }
      } else {
        while (lo < ns && key_less(__int_as_float(B.c[lo].y), __int_as_float(B.c[lo].z), o.x, o.y)) ++lo;
      }
      lo4 = lo;
#else
      int lo = 0, hi = ns;   // survivors with key < o
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_less(__int_as_float(B.c[mid].y), __int_as_float(B.c[mid].z), o.x, o.y)) lo = mid + 1; else hi = mid;
      }
#endif
      const int pos = B.ap[j] + lo;
      if (pos < C.K) {
        nst[pos] = o;
        nsi[pos] = si[j];
      }
    }
  }
  const int lbase = B.bc[0];
  if (lbase + ns > C.L) {
    if (tid == 0) atomicOr(&S->overflow, OVF_LABELS);
  } else {
    for (int q0 = 0; q0 < ns; q0 += bd) {   // whole warps (push_open is warp-collective)
      const int q = q0 + tid;
      const bool v = q < ns;
      const int4 c = v ? B.c[q] : make_int4(0, 0, 0, 0);
      const float qc = __int_as_float(c.y), qh = __int_as_float(c.z);
      const int id = lbase + q;
      push_open(S, PU, v, id, qc);
      if (!v) continue;
      DCHECK(id < C.L && c.w >= 0 && c.w < C.L);
      labels[id] = make_int4(x, c.w, c.y, c.z);
      lstate[id] = L_OPEN;
      int lo = 0, hi = m;   // first old entry with key > q
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const float2 om = st[mid];
        if (key_less(qc, qh, om.x, om.y)) hi = mid; else lo = mid + 1;
      }
      const int pos = q + B.ap[lo];
      if (pos < C.K) {
        nst[pos] = make_float2(qc, qh);
        nsi[pos] = id;
      }
    }
  }
  MERGE_MARK(3);
  if (tid == 0) {
    const int newm = na + ns;
    if (newm > C.K) atomicOr(&S->overflow, OVF_STAIR);
    sn[x] = min(newm, C.K) | ((par ^ 1) << 30);
    my_ins += (unsigned long long)ns;
  }
  __syncthreads();   // B is reused by the CTA's next large node
  MERGE_MARK(4);
  if (MPAP_DEBUG_CHECKS && tid == 0) atomicAdd(&g_merge_cyc[5], 1ull);
}

// Warp merge of a node with <= 32 candidates and a staircase of up to kBigM
// entries (left in global memory): the set semantics of cta_merge with one
// candidate per lane -- a shuffle bitonic sort, shuffle scans for the
// survivors, a binary search over the survivors per old entry, and a binary
// search over the old staircase per survivor, with the alive counts kept per
// 32-entry chunk in the warp's slice of the dynamic shared memory.
struct MidSmem {
  int4 sv[32];
  int pre[kBigM / 32 + 1];
  unsigned mask[kBigM / 32];
};
static_assert(sizeof(MidSmem) * (kST / 32) <= sizeof(BigSmem), "mid-merge slices must fit the CTA merge buffer");


__device__ void warp_mid_merge(Ctl* S, const SlotCaps& C, int x, int n, const int4* cs, const int32_t* coff,
                               const int32_t* ccnt, float2* sch, int32_t* sid, int32_t* sn, int4* labels,
                               uint8_t* lstate, const Pusher& PU, unsigned long long& my_ins,
                               unsigned long long& my_kill) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  MidSmem& W = reinterpret_cast<MidSmem*>(s_dyn)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = lane_lt();
  const int kc = ccnt[x];
  const int beg = coff[x] - kc;
  const int snx = sn[x];
  const int m = snx & kStairCountMask;
  const int par = snx >> 30;
  const float2* st = sch + stair_base(snx, x, n, C.K);
  const int32_t* si = sid + stair_base(snx, x, n, C.K);
  float2* nst = sch + ((size_t)(par ^ 1) * n + x) * (size_t)C.K;
  int32_t* nsi = sid + ((size_t)(par ^ 1) * n + x) * (size_t)C.K;
  int4 c = lane < kc ? cs[beg + lane] : make_int4(x, 0x7f800000, (int)0xff800000, INT_MAX);
  // 1. bitonic sort across the warp, ascending by (cost, -h, parent)
  for (int k = 2; k <= 32; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int4 o = shfl_xor4(c, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      if (lower ? (cand_less(o, c) == up) : (cand_less(c, o) == up)) c = o;
    }
  }
  // 2. survivors: min h over strictly cheaper candidates > own h
  const bool valid = lane < kc;
  const float cost = __int_as_float(c.y), h = __int_as_float(c.z);
  float pm = valid ? h : __int_as_float(0x7f800000);
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(FULLM, pm, o);
    if (lane >= o) pm = fminf(pm, y);
  }
  const float pc = __shfl_up_sync(FULLM, cost, 1);
  int g = (lane == 0 || pc != cost) ? lane : 0;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULLM, g, o);
    if (lane >= o) g = max(g, y);
  }
  const float pmg = __shfl_sync(FULLM, pm, g > 0 ? g - 1 : 0);
  const bool surv = valid && (g == 0 || pmg > h);
  const unsigned sm = __ballot_sync(FULLM, surv);
  const int ns = __popc(sm);
  if (surv) W.sv[__popc(sm & lt)] = c;
  __syncwarp();
  // 3. old entries: killed by a survivor? old alive ones to their merged slot
  int na = 0;
  for (int j0 = 0; j0 < m; j0 += 32) {
    const int j = j0 + lane;
    bool alive = false;
    float2 o = make_float2(0.0f, 0.0f);
    if (j < m) {
      o = st[j];
      int lo = 0, hi = ns;   // first survivor with cost >= o.x
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__int_as_float(W.sv[mid].y) < o.x) lo = mid + 1; else hi = mid;
      }
      const bool dead = lo > 0 && __int_as_float(W.sv[lo - 1].z) <= o.y;
      alive = !dead;
      if (dead) {
        const int oid = si[j];
        if (lstate[oid] == L_OPEN) {
          lstate[oid] = L_DEAD;
          ++my_kill;
        }
      }
    }
    const unsigned am = __ballot_sync(FULLM, alive);
    if (lane == 0) {
      W.pre[j0 >> 5] = na;
      W.mask[j0 >> 5] = am;
    }
    if (alive) {
      int lo = 0, hi = ns;   // survivors with key < o
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_less(__int_as_float(W.sv[mid].y), __int_as_float(W.sv[mid].z), o.x, o.y)) lo = mid + 1; else hi = mid;
      }
      const int pos = na + __popc(am & lt) + lo;
      if (pos < C.K) {
        nst[pos] = o;
        nsi[pos] = si[j];
      }
    }
    na += __popc(am);
  }
  __syncwarp();
  // 4. survivors: labels, pending list, merged slot
  int lbase = 0;
  if (lane == 0 && ns > 0) lbase = atomicAdd(&S->nlabels, ns);
  lbase = __shfl_sync(FULLM, lbase, 0);
  if (lbase + ns > C.L) {
    if (lane == 0) atomicOr(&S->overflow, OVF_LABELS);
  } else {
    const int4 q = W.sv[lane];
    const float qc = __int_as_float(q.y), qh = __int_as_float(q.z);
    const int id = lbase + lane;
    push_open(S, PU, lane < ns, id, qc);
  }
  if (lbase + ns <= C.L && lane < ns) {
    const int4 q = W.sv[lane];
    const float qc = __int_as_float(q.y), qh = __int_as_float(q.z);
    const int id = lbase + lane;
    DCHECK(id < C.L && q.w >= 0 && q.w < C.L);
    labels[id] = make_int4(x, q.w, q.y, q.z);
    lstate[id] = L_OPEN;
    int lo = 0, hi = m;   // first old entry with key > q
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const float2 om = st[mid];
      if (key_less(qc, qh, om.x, om.y)) hi = mid; else lo = mid + 1;
    }
    const int before = (lo == m) ? na : W.pre[lo >> 5] + __popc(W.mask[lo >> 5] & ((1u << (lo & 31)) - 1u));
    const int pos = lane + before;
    if (pos < C.K) {
      nst[pos] = make_float2(qc, qh);
      nsi[pos] = id;
    }
  }
  if (lane == 0) {
    const int newm = na + ns;
    if (newm > C.K) atomicOr(&S->overflow, OVF_STAIR);
    sn[x] = min(newm, C.K) | ((par ^ 1) << 30);
    my_ins += (unsigned long long)ns;
  }
  __syncwarp();
}

// Per-wave counters and work-queue heads, zeroed by the leader once per wave.
__device__ __forceinline__ void reset_wave_counters(Ctl* S) {
  S->relax = 0; S->bpass = 0; S->tcount = 0; S->ssum = 0; S->inserted = 0; S->killed = 0;
  S->ncand = 0; S->ntouched = 0; S->calloc = 0; S->nsmall = 0; S->nbig = 0; S->snext = 0; S->bnext = 0;
  S->nmid = 0; S->mnext = 0;
}

template <bool TRACE, typename Team>
__device__ void run_query(const Team& team, const SearchArgs& A, Ctl* S, int slot, int qpos) {
  const int q = A.qidx[qpos];
  const QueryDesc Q = A.queries[q];
  const int tid = team.rank(), lane = threadIdx.x & 31;
  const int nthr = team.size(), warp = team.warp(), nw = team.nwarps();
  const bool leader = (tid == 0);
  const unsigned lt = lane_lt();
  const SlotCaps C = A.caps;
  const int env = Q.env;
  const int n = A.n_env[env];
  const int64_t nbase = A.node_base[env];
  const int64_t* rp = A.row_ptr + nbase;
  // slot views
  int4* labels = A.labels + (size_t)slot * C.L;
  uint8_t* lstate = A.lstate + (size_t)slot * C.L;
  float2* sch = A.stair_ch + (size_t)slot * 2 * C.n * C.K;    // buffer b of node x at (b * n + x) * K
  int32_t* sid = A.stair_id + (size_t)slot * 2 * C.n * C.K;
  int32_t* sn = A.stair_n + (size_t)slot * C.n;
  int32_t* ccnt = A.cand_cnt + (size_t)slot * C.n;
  int32_t* coff = A.cand_off + (size_t)slot * C.n;
  int4* cand = A.cand + (size_t)slot * C.C;
  int4* cs = A.cand_sorted + (size_t)slot * C.C;
  int32_t* touched = A.touched + (size_t)slot * C.n;
  int32_t* tsmall = A.tsmall + (size_t)slot * C.n;
  int32_t* tbig = A.tbig + (size_t)slot * C.n;
  int32_t* tmid = A.tmid + (size_t)slot * C.n;
  int32_t* G = A.G + (size_t)slot * C.L;
  int32_t* pend = A.pend + (size_t)slot * C.L;
  int32_t* pend2 = A.pend2 + (size_t)slot * C.L;
  int32_t* const Galt = A.pend2 + (size_t)slot * C.L;   // ring mode: the second group list (pend2 is unused there)
  int32_t* ring = C.R ? A.ring + (size_t)slot * C.R * C.L : nullptr;
  int32_t* stamp = A.stamp + (size_t)slot * C.n;
  uint8_t* goal = A.goal + (size_t)slot * C.n;
  const double beta = Q.beta;
  const bool forall_t = (Q.flags & MPAP_SEARCH_FORALL_T) != 0u;   // Eq. 2 for every step (NEXT-3)
  const int d = A.pos_dim;
  mpap_result* R = A.results + q;

  // ---- a5: init (A3.1-A3.4) ----
  if (!A.resume) {
    if (leader) {
      S->gs[0] = 1; S->gs[1] = 0; S->psize = 0; S->nsize = 0; S->nlabels = 1;
      S->gig[0] = 0; S->gig[1] = 0; S->overflow = 0; S->any_goal = 0; S->i = 0; S->minb = LLONG_MAX;
      S->relax_total = 0; S->inserted_total = 0; S->waves = 0; S->suspended = 0; S->pswap = 0; S->need = 0;
      for (int r = 0; r < kRingMax; ++r) S->rcount[r] = 0;
      reset_wave_counters(S);
    }
    team.sync();
    bool mygoal = false;
    for (int x = tid; x < n; x += nthr) {
      sn[x] = 0;
      ccnt[x] = 0;
      if (TRACE) stamp[x] = -1;
      const double* p = A.samples + (nbase + x) * A.stride;
      bool in = true;
      for (int k = 0; k < d; ++k)
        if (p[k] < Q.goal_lo[k] || p[k] > Q.goal_hi[k]) in = false;
      goal[x] = in ? 1 : 0;
      mygoal |= in;
    }
    if (__any_sync(FULLM, mygoal) && lane == 0) S->any_goal = 1;
    team.sync();
    if (leader) {
      labels[0] = make_int4(Q.start, -1, __float_as_int(0.0f), __float_as_int(0.0f));
      lstate[0] = L_OPEN;
      sch[(size_t)Q.start * C.K] = make_float2(0.0f, 0.0f);   // buffer 0
      sid[(size_t)Q.start * C.K] = 0;
      sn[Q.start] = 1;
      G[0] = 0;
      S->gig[0] = goal[Q.start];
    }
    team.sync();
    if (!vld(S->any_goal)) {
      if (leader) {
        mpap_result r{};
        r.status = MPAP_ERR_NO_GOAL_NODE;
        *R = r;
      }
      return;
    }
  }
  // ---- wave loop (A3.5-A3.19) ----
  int wave = A.resume ? vld(S->waves) : 0;
  int pswap = A.resume ? vld(S->pswap) : 0;
  if (pswap) { int32_t* tmp = pend; pend = pend2; pend2 = tmp; }
  if (A.resume) {
    team.sync();
    if (leader) { S->suspended = 0; S->need = 0; }
    team.sync();
  }
  // the group index i, kept by every thread (each computes the same value;
  // S->i is its copy for a resumed launch and the host)
  long long i_loc = vld(S->i);
  while (true) {
    const int par = wave & 1;
    if (vld(S->gig[par]) || vld(S->gs[par]) == 0) break;     // A3.5 (G = {} <=> P_open = {} here)
    const int gsize = vld(S->gs[par]);
    const long long i_cur = i_loc;
    // ring mode: G_i and G_{i+1} in alternate lists, so retiring G_i and
    // forming G_{i+1} share one phase; the next group's counters were last
    // read at the top of the previous wave
    int32_t* const Gc = (C.R && par) ? Galt : G;
    int32_t* const Gn = (C.R && !par) ? Galt : G;
    if (leader) { S->gs[par ^ 1] = 0; S->gig[par ^ 1] = 0; }
    if (A.ready) {   // lazy roadmap: every head of G_i must have its row evaluated
      bool my_need = false;
      for (int k = tid; k < gsize; k += nthr) {
        const int64_t row = nbase + labels[Gc[k]].x;
        if (vld(A.ready[row]) != 1) {
          my_need = true;
          if (atomicCAS(&A.ready[row], 0, 2) == 0) A.req[atomicAdd(A.nreq, 1)] = (int32_t)row;
        }
      }
      if (my_need) atomicOr(&S->need, 1);
      team.sync();
      if (vld(S->need)) {   // suspend; the host evaluates the requested rows and resumes
        if (leader) { S->suspended = 1; S->pswap = pswap; }
        return;
      }
    }
    // the per-wave counters were reset by the previous wave's retire step
    // (or the init), two team barriers ago
    PHASE_MARK(0);
    // ---- a7 expand (A3.6-A3.11): warp per plan of G_i, 32 edges per step ----
    {
      unsigned long long my_relax = 0, my_bpass = 0, my_t = 0, my_ss = 0;
#if MPAP_EXPAND_BATCH_META
      // the warp's plans k = warp, warp + nw, ... (the same sequence), their
      // labels and CSR row bounds loaded 32 plans at a time (lane i: plan i of
      // the batch) so the label -> row-pointer load chain is paid once per 32
      for (int kb = warp; kb < gsize; kb += 32 * nw) {
        const int kk = kb + lane * nw;
        int p_l = 0;
        int4 lb_l = make_int4(0, 0, 0, 0);
        int64_t e0_l = 0, e1_l = 0;
        if (kk < gsize) {
          p_l = Gc[kk];
          lb_l = labels[p_l];
          e0_l = rp[lb_l.x];
          e1_l = rp[lb_l.x + 1];
        }
        const int nbat = min(32, (gsize - kb + nw - 1) / nw);
        for (int ib = 0; ib < nbat; ++ib) {
          const int p = __shfl_sync(FULLM, p_l, ib);
          const float pc = __int_as_float(__shfl_sync(FULLM, lb_l.z, ib));
          const float ph = __int_as_float(__shfl_sync(FULLM, lb_l.w, ib));
          const int64_t e0 = __shfl_sync(FULLM, e0_l, ib), e1 = __shfl_sync(FULLM, e1_l, ib);
          for (int64_t eb = e0; eb < e1; eb += 32) {
            const int64_t e = eb + lane;
            bool fr = false, emit = false;
            int x = 0;
            float qc = 0.f, qh = 0.f;
            if (e < e1) {
              const uint4 raw = __ldg(reinterpret_cast<const uint4*>(A.edges) + e);
              fr = (raw.x >> 31) == 0u;
              if (fr) {
                x = (int)(raw.x & 0x7fffffffu);
                qc = pc + __uint_as_float(raw.y);
                const float t = ph + __uint_as_float(raw.z);
                const float cc = __uint_as_float(raw.w);
                qh = (t > cc) ? t : cc;
                bool ok = (double)qh <= beta;                      // A3.9 cutoff
                if (forall_t && ok) {                              // every step of the edge
                  const float2 pk = __ldg(A.peak + e);
                  const float t2 = ph + pk.x;
                  ok = (double)((t2 > pk.y) ? t2 : pk.y) <= beta;
                }
                if (ok) {
                  ++my_bpass;
                  const int snx = sn[x];
                  const int m = snx & kStairCountMask;
                  if (TRACE) {
                    if (atomicExch(&stamp[x], wave) != wave) { ++my_t; my_ss += (unsigned long long)m; }
                  }
                  // dominated by the node's non-dominated staircase?  Such a
                  // candidate cannot survive RemoveDominated (transitivity).  With
                  // the staircase sorted, only the last entry of cost < qc matters.
                  const float2* st = sch + stair_base(snx, x, n, C.K);
                  // first index with cost >= qc; the wavefront's candidates are
                  // usually costlier than the whole staircase, so its last entry
                  // is checked first (one load instead of a log2(m)-deep search)
                  int lo = 0, hi = m;
                  float2 prev = make_float2(0.0f, __int_as_float(0x7f800000));
                  if (m > 0) {
                    const float2 last = st[m - 1];
                    if (last.x < qc) {
                      lo = m;
                      prev = last;
                    } else {
                      hi = m - 1;
                    }
                  }
                  while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (st[mid].x < qc) lo = mid + 1; else hi = mid;
                  }
                  if (lo > 0 && lo < m) prev = st[lo - 1];
                  const bool dom = lo > 0 && prev.y <= qh;
                  emit = !dom;
                }
              }
            }
            my_relax += __popc(__ballot_sync(FULLM, fr)) * (lane == 0 ? 1u : 0u);
            const unsigned em = __ballot_sync(FULLM, emit);
            if (em) {
              int base = 0;
              if (lane == 0) base = atomicAdd(&S->ncand, __popc(em));
              base = __shfl_sync(FULLM, base, 0);
              if (emit) {
                const int idx = base + __popc(em & lt);
                if (idx < C.C) {
                  DCHECK(x >= 0 && x < n);
                  cand[idx] = make_int4(x, __float_as_int(qc), __float_as_int(qh), p);
                  if (atomicAdd(&ccnt[x], 1) == 0) {
                    const int tpos = atomicAdd(&S->ntouched, 1);
                    DCHECK(tpos < n);
                    touched[tpos] = x;
                  }
                } else {
                  atomicOr(&S->overflow, OVF_CAND);
                }
              }
            }
          }

        }
      }
#else
      for (int k = warp; k < gsize; k += nw) {
        const int p = Gc[k];
        const int4 lb = labels[p];
        const int u = lb.x;
        const float pc = __int_as_float(lb.z), ph = __int_as_float(lb.w);
        const int64_t e0 = rp[u], e1 = rp[u + 1];
        for (int64_t eb = e0; eb < e1; eb += 32) {
          const int64_t e = eb + lane;
          bool fr = false, emit = false;
          int x = 0;
          float qc = 0.f, qh = 0.f;
          if (e < e1) {
            const uint4 raw = __ldg(reinterpret_cast<const uint4*>(A.edges) + e);
            fr = (raw.x >> 31) == 0u;
            if (fr) {
              x = (int)(raw.x & 0x7fffffffu);
              qc = pc + __uint_as_float(raw.y);
              const float t = ph + __uint_as_float(raw.z);
              const float cc = __uint_as_float(raw.w);
              qh = (t > cc) ? t : cc;
              bool ok = (double)qh <= beta;                      // A3.9 cutoff
              if (forall_t && ok) {                              // every step of the edge
                const float2 pk = __ldg(A.peak + e);
                const float t2 = ph + pk.x;
                ok = (double)((t2 > pk.y) ? t2 : pk.y) <= beta;
              }
              if (ok) {
                ++my_bpass;
                const int snx = sn[x];
                const int m = snx & kStairCountMask;
                if (TRACE) {
                  if (atomicExch(&stamp[x], wave) != wave) { ++my_t; my_ss += (unsigned long long)m; }
                }
                // dominated by the node's non-dominated staircase?  Such a
                // candidate cannot survive RemoveDominated (transitivity).  With
                // the staircase sorted, only the last entry of cost < qc matters.
                const float2* st = sch + stair_base(snx, x, n, C.K);
                // first index with cost >= qc; the wavefront's candidates are
                // usually costlier than the whole staircase, so its last entry
                // is checked first (one load instead of a log2(m)-deep search)
                int lo = 0, hi = m;
                float2 prev = make_float2(0.0f, __int_as_float(0x7f800000));
                if (m > 0) {
                  const float2 last = st[m - 1];
                  if (last.x < qc) {
                    lo = m;
                    prev = last;
                  } else {
                    hi = m - 1;
                  }
                }
                while (lo < hi) {
                  const int mid = (lo + hi) >> 1;
                  if (st[mid].x < qc) lo = mid + 1; else hi = mid;
                }
                if (lo > 0 && lo < m) prev = st[lo - 1];
                const bool dom = lo > 0 && prev.y <= qh;
                emit = !dom;
              }
            }
          }
          my_relax += __popc(__ballot_sync(FULLM, fr)) * (lane == 0 ? 1u : 0u);
          const unsigned em = __ballot_sync(FULLM, emit);
          if (em) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&S->ncand, __popc(em));
            base = __shfl_sync(FULLM, base, 0);
            if (emit) {
              const int idx = base + __popc(em & lt);
              if (idx < C.C) {
                DCHECK(x >= 0 && x < n);
                cand[idx] = make_int4(x, __float_as_int(qc), __float_as_int(qh), p);
                if (atomicAdd(&ccnt[x], 1) == 0) {
                  const int tpos = atomicAdd(&S->ntouched, 1);
                  DCHECK(tpos < n);
                  touched[tpos] = x;
                }
              } else {
                atomicOr(&S->overflow, OVF_CAND);
              }
            }
          }
        }
      }
#endif
      if (my_relax) atomicAdd(&S->relax, my_relax);
      if (my_bpass) atomicAdd(&S->bpass, my_bpass);
      if (TRACE) {
        if (my_t) atomicAdd(&S->tcount, my_t);
        if (my_ss) atomicAdd(&S->ssum, my_ss);
      }
    }
    team.sync();
    if (vld(S->overflow)) break;
    const int nt = vld(S->ntouched);
    PHASE_MARK(1);
    const int ncand = vld(S->ncand);
    // ---- group candidates by destination: contiguous range per touched node ----
    for (int t = tid; t < nt; t += nthr) {
      const int x = touched[t];
      const int kc = ccnt[x];
      coff[x] = atomicAdd(&S->calloc, kc);
      const int m = sn[x] & kStairCountMask;
      if ((kc > kMrgCap || m > kMrgCap) && kc <= 32 && m <= kBigM) tmid[atomicAdd(&S->nmid, 1)] = x;
      else if ((kc > kMrgCap || m > kMrgCap) && kc <= kBigC && m <= kBigM) tbig[atomicAdd(&S->nbig, 1)] = x;
      else tsmall[atomicAdd(&S->nsmall, 1)] = x;
      if (MPAP_DEBUG_CHECKS && A.nq == 1 && wave < kPhaseWaves) {
        atomicMax(&g_phase_stat[wave][2], kc);
        atomicMax(&g_phase_stat[wave][3], m);
      }
    }
    team.sync();
    PHASE_MARK(2);
    for (int k = tid; k < ncand; k += nthr) {
      const int4 cq = cand[k];
      const int pos = atomicAdd(&coff[cq.x], 1);
      DCHECK(pos >= 0 && pos < C.C);
      cs[pos] = cq;
    }
    team.sync();
    PHASE_MARK(3);
    if (MPAP_DEBUG_CHECKS && leader && A.nq == 1 && wave < kPhaseWaves) {
      g_phase_stat[wave][0] = vld(S->nbig);
      g_phase_stat[wave][1] = vld(S->nsmall);
    }
    // ---- a8 RemoveDominated + insert (A3.10-A3.15): warp per touched node ----
    {
      // per-warp shared-memory staging of the node's candidates (sorted copy,
      // then survivors) and of its non-dominated staircase: the all-pairs
      // dominance loops read them from shared memory (global fallback above
      // kMrgCap entries)
      __shared__ int4 s_cand[kST / 32][2][kMrgCap];
      __shared__ float2 s_sch[kST / 32][kMrgCap];
      __shared__ int32_t s_sid[kST / 32][kMrgCap];
      const int wl = threadIdx.x >> 5;
      unsigned long long my_ins = 0, my_kill = 0;
      const Pusher PU{pend, ring, C.R, C.L, A.T, i_cur};
      // large nodes: one CTA each (uniform per CTA: __syncthreads inside)
      const int nbig = vld(S->nbig), nsmall = vld(S->nsmall);
      if (nbig > 0) {   // pulled from a counter by whole CTAs (large nodes vary a lot in size)
        __shared__ int s_big;
        for (;;) {
          if (threadIdx.x == 0) s_big = atomicAdd(&S->bnext, 1);
          __syncthreads();
          const int b = s_big;
          __syncthreads();
          if (b >= nbig) break;
          cta_merge(S, C, tbig[b], n, cs, coff, ccnt, sch, sid, sn, labels, lstate, PU, my_ins, my_kill);
        }
      }
      // mid nodes (<= 32 candidates, large staircase): one warp each, with a
      // slice of the CTA's (now free) dynamic shared memory
      {
        const int nmid = vld(S->nmid);
        for (;;) {
          int t = 0;
          if (lane == 0) t = atomicAdd(&S->mnext, 1);
          t = __shfl_sync(FULLM, t, 0);
          if (t >= nmid) break;
          warp_mid_merge(S, C, tmid[t], n, cs, coff, ccnt, sch, sid, sn, labels, lstate, PU, my_ins, my_kill);
        }
      }
      // small nodes: one warp each, pulled from a counter (warps of CTAs busy
      // with large nodes join late)
      for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&S->snext, 1);
        t = __shfl_sync(FULLM, t, 0);
        if (t >= nsmall) break;
        const int x = tsmall[t];
        const int kc = ccnt[x];
        const int beg = coff[x] - kc;
        const int snx = sn[x];
        const int m = snx & kStairCountMask;
        const int par = snx >> 30;
        float2* st = sch + stair_base(snx, x, n, C.K);
        int32_t* si = sid + stair_base(snx, x, n, C.K);
        float2* nst = sch + ((size_t)(par ^ 1) * n + x) * (size_t)C.K;
        int32_t* nsi = sid + ((size_t)(par ^ 1) * n + x) * (size_t)C.K;
        int4* srt = cand + beg;   // candidate buffer is free after grouping: sorted copy
        int4* sv = cs + beg;      // then the grouped range holds the sorted survivors
        const int4* cin = cs + beg;
        if (kc <= kMrgCap) {      // stage the candidates; sort into / survivors in shared memory
          for (int q = lane; q < kc; q += 32) s_cand[wl][0][q] = cs[beg + q];
          cin = s_cand[wl][0];
          srt = s_cand[wl][1];
          sv = s_cand[wl][0];     // written after the sort has read every staged candidate
        }
        if (m <= kMrgCap) {       // stage the staircase (its dead marks stay in the copy)
          for (int j = lane; j < m; j += 32) {
            s_sch[wl][j] = st[j];
            s_sid[wl][j] = si[j];
          }
          st = s_sch[wl];
          si = s_sid[wl];
        }
        __syncwarp();
        // 1. sort the node's candidates by (cost asc, h desc), ties by index
        for (int q0 = 0; q0 < kc; q0 += 32) {
          const int qq = q0 + lane;
          if (qq < kc) {
            const int4 cq = cin[qq];
            const float qc = __int_as_float(cq.y), qh = __int_as_float(cq.z);
            int rank = 0;
            for (int r2 = 0; r2 < kc; ++r2) {
              const int4 cr = cin[r2];
              const float rc = __int_as_float(cr.y), rh = __int_as_float(cr.z);
              if (key_less(rc, rh, qc, qh) || (rc == qc && rh == qh && r2 < qq)) ++rank;
            }
            srt[rank] = cq;
          }
        }
        __syncwarp();
        // 2. candidate survivors: not dominated by a cheaper candidate (the
        //    staircase cannot dominate them: filtered at expansion)
        int ns = 0;
        for (int q0 = 0; q0 < kc; q0 += 32) {
          const int qq = q0 + lane;
          bool surv = false;
          int4 cq = make_int4(0, 0, 0, 0);
          if (qq < kc) {
            cq = srt[qq];
            surv = true;
            const float qc = __int_as_float(cq.y), qh = __int_as_float(cq.z);
            for (int r2 = 0; r2 < qq; ++r2) {
              const int4 cr = srt[r2];
              if (!(__int_as_float(cr.y) < qc)) break;   // sorted: no cheaper candidate left
              if (__int_as_float(cr.z) <= qh) { surv = false; break; }
            }
          }
          const unsigned sm = __ballot_sync(FULLM, surv);
          // survivors, in key order, go to the (now free) grouped range
          if (surv) sv[ns + __popc(sm & lt)] = cq;
          ns += __popc(sm);
        }
        __syncwarp();
        // 3. old entries killed by a candidate (checking the surviving
        //    candidates suffices: a dominated candidate's dominator dominates
        //    too); dead ids marked in place
        int na = 0;
        for (int j0 = 0; j0 < m; j0 += 32) {
          const int j = j0 + lane;
          bool alive = false;
          if (j < m) {
            const float2 o = st[j];
            alive = true;
            for (int r2 = 0; r2 < ns; ++r2) {
              const int4 cr = sv[r2];
              if (!(__int_as_float(cr.y) < o.x)) break;
              if (__int_as_float(cr.z) <= o.y) { alive = false; break; }
            }
            if (!alive) {
              const int oid = si[j];
              if (lstate[oid] == L_OPEN) {
                lstate[oid] = L_DEAD;
                ++my_kill;
              }
            }
          }
          const unsigned am = __ballot_sync(FULLM, alive);
          // 4a. old survivor -> rank among old survivors + new survivors before it
          if (alive) {
            const float2 o = st[j];
            int before = 0;
            for (int r2 = 0; r2 < ns; ++r2) {
              const int4 cr = sv[r2];
              if (key_less(__int_as_float(cr.y), __int_as_float(cr.z), o.x, o.y)) ++before; else break;
            }
            const int pos = na + __popc(am & lt) + before;
            if (pos < C.K) {
              nst[pos] = o;
              nsi[pos] = si[j];
            }
          }
          na += __popc(am);
          if (!alive && j < m) si[j] = -1;
        }
        __syncwarp();
        // 4b. new survivors: labels, pending list, position = own rank + old survivors before it
        for (int q0 = 0; q0 < ns; q0 += 32) {
          const int qq = q0 + lane;
          const bool v = qq < ns;
          const unsigned vm = __ballot_sync(FULLM, v);
          int lbase = 0;
          if (lane == 0) lbase = atomicAdd(&S->nlabels, __popc(vm));
          lbase = __shfl_sync(FULLM, lbase, 0);
          if (lbase + __popc(vm) > C.L) {
            if (lane == 0) atomicOr(&S->overflow, OVF_LABELS);
          } else {
            push_open(S, PU, v, lbase + lane, v ? __int_as_float(sv[qq].y) : 0.0f);
          }
          if (lbase + __popc(vm) <= C.L && v) {
            const int4 cq = sv[qq];
            const float qc = __int_as_float(cq.y), qh = __int_as_float(cq.z);
            const int id = lbase + lane;
            DCHECK(id < C.L && cq.w >= 0 && cq.w < C.L);
            labels[id] = make_int4(x, cq.w, cq.y, cq.z);
            lstate[id] = L_OPEN;
            int before = 0;   // alive old entries with key <= (qc, qh)
            for (int j = 0; j < m; ++j) {
              const float2 o = st[j];
              if (key_less(qc, qh, o.x, o.y)) break;
              if (si[j] >= 0) ++before;
            }
            const int pos = qq + before;
            if (pos < C.K) {
              nst[pos] = make_float2(qc, qh);
              nsi[pos] = id;
            }
          }
          if (lane == 0) my_ins += __popc(vm);
        }
        if (lane == 0) {
          const int newm = na + ns;
          if (newm > C.K) atomicOr(&S->overflow, OVF_STAIR);
          sn[x] = min(newm, C.K) | ((par ^ 1) << 30);
        }
      }
      if (my_kill) atomicAdd(&S->killed, my_kill);
      if (my_ins) atomicAdd(&S->inserted, my_ins);
    }
    team.sync();
    PHASE_MARK(4);
    if (vld(S->overflow)) break;
    // reset per-node candidate counters of touched nodes
    for (int t = tid; t < nt; t += nthr) ccnt[touched[t]] = 0;
    // ---- a9 retire G_i (A3.16), i <- i+1 (A3.17) ----
    for (int k = tid; k < gsize; k += nthr) {
      const int p = Gc[k];
      if (lstate[p] == L_OPEN) lstate[p] = L_CLOSED;
    }
    if (leader) {
      if (TRACE && wave < A.waves_cap) {
        mpap_wave wv;
        wv.i = i_cur; wv.group = gsize; wv.relax = (long long)vld(S->relax);
        wv.beta_pass = (long long)vld(S->bpass); wv.inserted = (long long)vld(S->inserted);
        wv.killed = (long long)vld(S->killed); wv.touched = (long long)vld(S->tcount);
        wv.stair_sum = (long long)vld(S->ssum);
        A.waves[(size_t)q * A.waves_cap + wave] = wv;
      }
      S->relax_total += vld(S->relax);
      S->inserted_total += vld(S->inserted);
      S->waves = wave + 1;
      S->nsize = 0; S->minb = LLONG_MAX;
      reset_wave_counters(S);   // nothing reads them between the merge barrier and the next expand
    }
    // ring mode: no barrier -- the partition below reads other plans' states
    // (a plan is in exactly one ring list) and writes the other group list
    if (!C.R) team.sync();
    PHASE_MARK(5);
    // ---- a6 G_{i+1} (A3.18), with the exact empty-group skip (R24) ----
    if (C.R) {
      // bucket ring: G_j = the live plans of list j (every plan of list j has
      // cost <= j T, every later plan more); empty lists are skipped
      long long j = i_cur + 1;
      for (;;) {
        const int r = (int)(j % C.R);
        const int cnt = vld(S->rcount[r]);
        partition(team, A, S, ring + (size_t)r * C.L, cnt, Gn, Gn, LLONG_MAX / 4, labels, lstate, goal, par ^ 1);
        team.sync();
        const bool done = vld(S->gs[par ^ 1]) > 0 || j >= i_cur + C.R;   // the same for every thread
        if (done) {
          // list r is next written R - 1 groups later (new plans go to lists
          // i + 1 .. i + R - 1), many barriers after this store
          if (leader) { S->rcount[r] = 0; S->i = j; }
          break;
        }
        team.sync();   // every thread has read gsize before the next list's partition adds to it
        if (leader) S->rcount[r] = 0;
        ++j;
      }
      i_loc = j;
      PHASE_MARK(6);
      ++wave;
      continue;
    }
    const int np = vld(S->psize);
    long long inext = i_cur + 1;
    partition(team, A, S, pend, np, G, pend2, inext, labels, lstate, goal, par ^ 1);
    team.sync();
    PHASE_MARK(6);
    if (vld(S->gs[par ^ 1]) == 0 && vld(S->nsize) > 0) {
      inext = vld(S->minb);
      const int n2 = vld(S->nsize);
      team.sync();
      if (leader) { S->nsize = 0; S->minb = LLONG_MAX; }
      team.sync();
      partition(team, A, S, pend2, n2, G, pend, inext, labels, lstate, goal, par ^ 1);
      team.sync();
      if (leader) { S->psize = vld(S->nsize); S->i = inext; }
    } else {
      // swap pending lists
      if (leader) { S->psize = vld(S->nsize); S->i = inext; }
      int32_t* tmp = pend; pend = pend2; pend2 = tmp;
      pswap ^= 1;
    }
    team.sync();
    i_loc = inext;
    ++wave;
  }

  // ---- a10 goal extraction (A3.20-A3.21) ----
  if (vld(S->overflow)) {
    if (leader) {
      mpap_result r{};
      r.status = kRetryBase + vld(S->overflow);
      *R = r;
    }
    return;
  }
  if (!vld(S->gig[wave & 1])) {   // P_open emptied: no feasible plan
    if (leader) {
      mpap_result r{};
      r.status = MPAP_ERR_NO_FEASIBLE_PLAN;
      r.waves = vld(S->waves);
      r.relaxations = (int64_t)vld(S->relax_total);
      r.labels_inserted = (int64_t)vld(S->inserted_total);
      *R = r;
    }
    return;
  }
  team.sync();
  if (leader) { S->best_key = ~0ull; S->nties = 0; }
  team.sync();
  for (int x = tid; x < n; x += nthr) {
    if (!goal[x]) continue;
    const int snx = sn[x];
    const int m = snx & kStairCountMask;
    const float2* st = sch + stair_base(snx, x, n, C.K);
    for (int j = 0; j < m; ++j) {
      const float2 ch = st[j];
      const unsigned long long key = ((unsigned long long)__float_as_uint(ch.x) << 32) | __float_as_uint(ch.y);
      atomicMin(&S->best_key, key);
    }
  }
  team.sync();
  const unsigned long long best_key = vld(S->best_key);
  for (int x = tid; x < n; x += nthr) {
    if (!goal[x]) continue;
    const int snx = sn[x];
    const int m = snx & kStairCountMask;
    const float2* st = sch + stair_base(snx, x, n, C.K);
    const int32_t* si = sid + stair_base(snx, x, n, C.K);
    for (int j = 0; j < m; ++j) {
      const float2 ch = st[j];
      const unsigned long long key = ((unsigned long long)__float_as_uint(ch.x) << 32) | __float_as_uint(ch.y);
      if (key == best_key) {
        const int slot_t = atomicAdd(&S->nties, 1);
        if (slot_t < kMaxTies) S->ties[slot_t] = si[j];
      }
    }
  }
  team.sync();
  if (leader) {
    // lexicographic tie-break on node sequences (R16); chains reversed into
    // the (now unused) G / pend2 arrays
    const int nties = vld(S->nties);
    int best = -1;
    auto consider = [&](int cand_id) {
      if (best < 0) { best = cand_id; return; }
      int la = 0, lb = 0;
      for (int x = cand_id; x >= 0; x = labels[x].y) G[la++] = labels[x].x;
      for (int x = best; x >= 0; x = labels[x].y) pend2[lb++] = labels[x].x;
      bool less = false, decided = false;
      for (int s = 0; s < min(la, lb); ++s) {
        const int a = G[la - 1 - s], b = pend2[lb - 1 - s];
        if (a != b) { less = a < b; decided = true; break; }
      }
      if (!decided) less = la < lb;
      if (less) best = cand_id;
    };
    if (nties <= kMaxTies) {
      for (int k = 0; k < nties; ++k) consider(vld(S->ties[k]));
    } else {
      // more (cost, h) ties than the shared list holds (rare): the leader
      // scans every goal node's staircase itself -- all ties are compared
      for (int x = 0; x < n; ++x) {
        if (!goal[x]) continue;
        const int snx = sn[x];
        const int m = snx & kStairCountMask;
        const float2* st = sch + stair_base(snx, x, n, C.K);
        const int32_t* si = sid + stair_base(snx, x, n, C.K);
        for (int j = 0; j < m; ++j) {
          const float2 ch = st[j];
          const unsigned long long key = ((unsigned long long)__float_as_uint(ch.x) << 32) | __float_as_uint(ch.y);
          if (key == best_key) consider(si[j]);
        }
      }
    }
    int len = 0;
    float hp = 0.0f;
    for (int x = best; x >= 0; x = labels[x].y) {
      ++len;
      const float hx = __int_as_float(labels[x].w);
      if (hx > hp) hp = hx;
    }
    mpap_result r{};
    r.waves = vld(S->waves);
    r.relaxations = (int64_t)vld(S->relax_total);
    r.labels_inserted = (int64_t)vld(S->inserted_total);
    r.cost = __int_as_float(labels[best].z);
    r.h = __int_as_float(labels[best].w);
    r.h_peak = hp;
    r.path_len = len;
    if (len <= A.path_cap) {
      int32_t* out = A.paths + (size_t)q * A.path_cap;
      int k = len - 1;
      for (int x = best; x >= 0; x = labels[x].y) out[k--] = labels[x].x;
      r.status = MPAP_OK;
    } else {
      r.status = MPAP_ERR_BUFFER_TOO_SMALL;
    }
    *R = r;
  }
}

// Batched queries: one CTA per query at a time, queries pulled from a counter.
template <bool TRACE>
__global__ void __launch_bounds__(kST, 2) k_search(SearchArgs A) {   // two CTAs (queries) per SM
  __shared__ Ctl S;
  __shared__ int s_q;
  const CtaTeam team;
  while (true) {
    if (threadIdx.x == 0) s_q = atomicAdd(A.work, 1);
    __syncthreads();
    const int qpos = s_q;
    __syncthreads();
    if (qpos >= A.nq) break;
    run_query<TRACE>(team, A, &S, blockIdx.x, qpos);
    __syncthreads();
  }
}

// Batched queries with one thread-block cluster per query at a time (queries
// pulled from a counter by the cluster's leader).  Control words live in
// global memory, one Ctl per cluster slot.
template <bool TRACE>
__global__ void __launch_bounds__(kST) k_search_cluster(SearchArgs A, Ctl* S_all) {
  const ClusterTeam team;
  const int slot = blockIdx.x / cg::this_cluster().num_blocks();
  Ctl* S = S_all + slot;
  if (A.ready) {   // lazy roadmap: query = slot (static), so a suspended query resumes in its slot
    if (slot < A.nq && (!A.resume || vld(S->suspended))) run_query<TRACE>(team, A, S, slot, slot);
    return;
  }
  while (true) {
    if (team.rank() == 0) S->q = atomicAdd(A.work, 1);
    team.sync();
    const int qpos = vld(S->q);
    team.sync();
    if (qpos >= A.nq) break;
    run_query<TRACE>(team, A, S, slot, qpos);
    team.sync();
  }
}

// A single query over the whole grid (cooperative launch; grid.sync between
// the phases of each wave).  Control words live in global memory.  One block
// per SM is pinned in the launch bounds: left free, ptxas may squeeze the
// kernel to 64 registers (two blocks per SM) with local-memory spills, which
// measured 3x slower single queries (C1 8.1 -> 27.0 ms, C4 1.02 beta_min
// 48 -> 136 ms; profiles/r02/search_regression_ab.jsonl).
template <bool TRACE>
__global__ void __launch_bounds__(kST, 1) k_search_grid(SearchArgs A, Ctl* S) {
  const GridTeam team;
  run_query<TRACE>(team, A, S, 0, 0);
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
#define CKS(x)                                         \
  do {                                                 \
    cudaError_t _e = (x);                              \
    if (_e != cudaSuccess) return cuda_error(_e, #x);  \
  } while (0)

namespace {
// Carves the per-launch slot arena: every array holds nslots consecutive
// per-slot views (slot s at element offset s * cap), each array 256-B aligned.
// With base == nullptr it only returns the byte count.
// Process-wide capacity hints per device: the staircase / label / candidate
// capacities earlier searches needed.  A fresh roadmap starts there when the
// slot arena stays within kHintArenaBytes (fewer overflow reruns, the same
// results: capacities never change what a search computes).
struct CapHint {
  int K = 0, L = 0, C = 0;
};
constexpr int kMaxDevices = 64;
constexpr size_t kHintArenaBytes = size_t(4) << 30;
constexpr int kHintMaxSlots = 64;
constexpr int64_t kGridHalfNnz = 256 * 1024;
CapHint g_cap_hint[kMaxDevices];
std::mutex g_cap_mu;

// Stream access-policy window (persisting hits) over [base, base + bytes),
// clamped to the device's window and persisting-L2 limits; removed (and the
// persisting lines released) when the object goes out of scope.
struct L2Window {
  cudaStream_t st;
  bool on = false;
  L2Window(cudaStream_t s, int dev, const void* base, size_t bytes, bool enable) : st(s) {
    if (!enable || !base || bytes == 0) return;
    int max_win = 0, max_persist = 0;
    if (cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
        max_win <= 0 || max_persist <= 0) {
      cudaGetLastError();
      return;
    }
    const size_t win = std::min(bytes, (size_t)max_win);
    const size_t persist = std::min(win, (size_t)max_persist);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = win;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)persist / (double)win);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    on = cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
    if (!on) cudaGetLastError();
  }
  ~L2Window() {
    if (!on) return;
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
  }
};

size_t carve(SearchArgs* A, const SlotCaps& c, int nslots, char* base) {
  size_t off = 0;
  auto take = [&](size_t per_slot) -> void* {
    void* r = base ? base + off : nullptr;
    off += ((per_slot * (size_t)nslots) + 255) & ~size_t(255);
    return r;
  };
  void* p;
  p = take(sizeof(int4) * (size_t)c.L);                 if (A) A->labels = (int4*)p;
  p = take((size_t)c.L);                                if (A) A->lstate = (uint8_t*)p;
  p = take(sizeof(float2) * 2 * (size_t)c.n * c.K);     if (A) A->stair_ch = (float2*)p;
  p = take(sizeof(int32_t) * 2 * (size_t)c.n * c.K);    if (A) A->stair_id = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->stair_n = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->cand_cnt = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->cand_off = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->touched = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->tsmall = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->tbig = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->tmid = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.n);              if (A) A->stamp = (int32_t*)p;
  p = take((size_t)c.n);                                if (A) A->goal = (uint8_t*)p;
  p = take(sizeof(int4) * (size_t)c.C);                 if (A) A->cand = (int4*)p;
  p = take(sizeof(int4) * (size_t)c.C);                 if (A) A->cand_sorted = (int4*)p;
  p = take(sizeof(int32_t) * (size_t)c.L);              if (A) A->G = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.L);              if (A) A->pend = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.L);              if (A) A->pend2 = (int32_t*)p;
  p = take(sizeof(int32_t) * (size_t)c.L * c.R);        if (A) A->ring = (int32_t*)p;
  return off;
}
}  // namespace


// The CTA merge of large nodes uses kBigSmem bytes of dynamic shared memory
// (above the 48 KB default): opt every search kernel in, once per device.
cudaError_t set_search_smem() {
  static int done_dev = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev == done_dev) return e;
  const void* fns[] = {(const void*)k_search<false>, (const void*)k_search<true>, (const void*)k_search_cluster<false>,
                       (const void*)k_search_cluster<true>, (const void*)k_search_grid<false>,
                       (const void*)k_search_grid<true>};
  for (const void* f : fns) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBigSmem);
    if (e != cudaSuccess) return e;
  }
  done_dev = dev;
  return cudaSuccess;
}

mpap_status search_batch_device(const mpap_roadmap* rm, int32_t nq, const QueryDesc* h_queries, double lambda,
                                int32_t* paths, int32_t path_cap, mpap_result* results, mpap_wave* h_waves,
                                int32_t waves_cap, int32_t mem, cudaStream_t st) {
  if (nq <= 0) return MPAP_OK;
  HostTimer total("search_batch_device total");
  int dev = 0, nsm = 0;
  CKS(cudaGetDevice(&dev));
  CKS(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const bool trace = (h_waves != nullptr && waves_cap > 0);
  int occ = 1;
  CKS(set_search_smem());
  if (trace) CKS(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_search<true>, kST, kBigSmem));
  else CKS(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_search<false>, kST, kBigSmem));
  occ = std::max(occ, 1);
  int occ_grid = 1, coop = 0;
  CKS(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (trace) CKS(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_grid, k_search_grid<true>, kST, kBigSmem));
  else CKS(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_grid, k_search_grid<false>, kST, kBigSmem));
  const bool use_grid = coop && occ_grid > 0 && getenv("MPAP_SEARCH_CTA") == nullptr && getenv("MPAP_SEARCH_NO_GRID") == nullptr;
  const bool use_cluster = getenv("MPAP_SEARCH_CTA") == nullptr && getenv("MPAP_SEARCH_NO_CLUSTER") == nullptr;
  // A handful of queries (a perception-bound sweep) runs one after the other
  // on the whole grid: 8-CTA clusters would leave most SMs idle (C4 sweep of 6
  // bounds: 370 ms batched vs 158 ms in sequence).  So does any
  // batch on one large environment (bound sweeps / refinement of a big
  // roadmap: each query is heavy enough to fill the grid).
  bool one_large_env = nq > 1 && nq <= kSeqLargeMaxQ;
  for (int32_t k = 0; k < nq && one_large_env; ++k)
    one_large_env = h_queries[k].env == h_queries[0].env && rm->n[h_queries[0].env] >= kSeqLargeN;
  if (nq > 1 && (nq <= kSeqQueries || one_large_env) && use_grid && !rm->lazy) {
    // every query runs and writes its record; the first failing status is
    // returned after all of them (as the batched path does)
    mpap_status first = MPAP_OK;
    for (int32_t k = 0; k < nq; ++k) {
      mpap_status s = search_batch_device(rm, 1, h_queries + k, lambda, paths + (size_t)k * path_cap, path_cap,
                                          results + k, trace ? h_waves + (size_t)k * waves_cap : nullptr,
                                          waves_cap, mem, st);
      if (s != MPAP_OK && first == MPAP_OK) first = s;
    }
    return first;
  }
  SlotCaps caps;
  caps.n = rm->n_max;
  caps.K = std::max(64, rm->hint_K);
  caps.L = std::max(std::max(1 << 17, 64 * rm->n_max), rm->hint_L);
  caps.C = std::max(caps.L, rm->hint_C);
  {  // bucket ring: ceil(1/lambda) + 3 lists cover every new plan's group index
    const double inv = std::ceil(1.0 / lambda);
    caps.R = (!rm->lazy && inv + 3.0 <= (double)kRingMax && getenv("MPAP_SEARCH_NO_RING") == nullptr)
                 ? (int)inv + 3 : 0;
  }

  // device copies of the queries and outputs
  QueryDesc* d_q = nullptr;
  int32_t* d_qidx = nullptr;
  int* d_work = nullptr;
  mpap_result* d_res = nullptr;
  int32_t* d_paths = nullptr;
  mpap_wave* d_waves = nullptr;
  CKS(cudaMallocAsync(&d_q, sizeof(QueryDesc) * nq, st));
  CKS(cudaMemcpyAsync(d_q, h_queries, sizeof(QueryDesc) * nq, cudaMemcpyHostToDevice, st));
  CKS(cudaMallocAsync(&d_qidx, sizeof(int32_t) * nq, st));
  CKS(cudaMallocAsync(&d_work, sizeof(int), st));
  if (mem == MPAP_MEM_DEVICE) {
    d_res = results;
    d_paths = paths;
  } else {
    CKS(cudaMallocAsync(&d_res, sizeof(mpap_result) * nq, st));
    CKS(cudaMallocAsync(&d_paths, sizeof(int32_t) * (size_t)nq * std::max(path_cap, 1), st));
  }
  if (trace) CKS(cudaMallocAsync(&d_waves, sizeof(mpap_wave) * (size_t)nq * waves_cap, st));

  std::vector<int32_t> todo(nq);
  for (int k = 0; k < nq; ++k) todo[k] = k;
  std::vector<int32_t> retries(nq, 0);
  std::vector<mpap_result> hres(nq);
  mpap_status status = MPAP_OK;
  // L2 persistence for the CSR edge records (read by every expansion, the
  // search's streamed data): an access-policy window on the stream for the
  // duration of this call (MPAP_SEARCH_L2_PERSIST=1; measured)
  L2Window l2w(st, dev, rm->d_edges, (size_t)rm->nnz_total * sizeof(EdgeRec),
               getenv("MPAP_SEARCH_L2_PERSIST") != nullptr);
  for (int round = 0; round < 12 && !todo.empty(); ++round) {
    const int nrun = (int)todo.size();
    // one query: the whole grid works on it (cooperative launch); otherwise one
    // CTA per query and as many slots as resident CTAs
    const bool grid_mode = (nrun == 1) && use_grid;
    // few queries: one cluster per query of 8, 4 or 2 CTAs -- the largest
    // with nrun x size <= SMs x (one-CTA-kernel occupancy); for the bench's
    // 64 queries that is 4 (measured: 2.0 ms vs 2.2 / 3.6 ms for 2 / 8 CTAs,
    // 3.5 ms for one CTA per query); many: one CTA each.  (A lazy roadmap
    // runs batches in cluster mode, one static slot per query, so suspended
    // queries resume in place.)
    int csize = kCluster;
    if (const char* cs = getenv("MPAP_SEARCH_CLUSTER")) {   // tuning: largest cluster size (2, 4 or 8)
      const int c = atoi(cs);
      if (c == 2 || c == 4 || c == 8) csize = c;
    }
    while (csize > 2 && nrun * csize > nsm * occ) csize >>= 1;
    const bool cluster_mode = !grid_mode && use_cluster && (nrun * csize <= nsm * occ || rm->lazy);
    const int nslots = grid_mode ? 1 : cluster_mode ? nrun : std::min(nrun, nsm * occ);
    // whole-grid team: one block per SM; half the SMs for a roadmap of at
    // most kGridHalfNnz edges, whose waves are too small to pay for the
    // wider barriers (measured: C1-C3 single queries 10-20 % faster on 74
    // blocks, C4 1.5x slower)
    int grid_ctas = nsm * occ_grid;
    if (grid_mode) {
      const int env0 = h_queries[todo[0]].env;
      if (rm->edge_base[env0 + 1] - rm->edge_base[env0] <= kGridHalfNnz) grid_ctas = std::max(1, grid_ctas / 2);
    }
    if (const char* gc = getenv("MPAP_SEARCH_GRID_CTAS")) grid_ctas = std::max(1, std::min(nsm * occ_grid, atoi(gc)));
    // (only for up to kHintMaxSlots slots: a many-slot arena seeded from a
    // smaller batch's maxima kept growing the workspace step after step)
    if (round == 0 && nslots <= kHintMaxSlots && dev >= 0 && dev < kMaxDevices &&
        getenv("MPAP_SEARCH_NO_HINT") == nullptr) {
      CapHint h;
      {
        std::lock_guard<std::mutex> lk(g_cap_mu);
        h = g_cap_hint[dev];
      }
      SlotCaps t = caps;
      t.L = std::max(t.L, h.L);
      t.C = std::max(t.C, h.C);
      t.K = std::max(t.K, h.K);
      while (t.K > caps.K && carve(nullptr, t, nslots, nullptr) > kHintArenaBytes) t.K = std::max(caps.K, t.K / 2);
      if (carve(nullptr, t, nslots, nullptr) <= kHintArenaBytes) caps = t;
    }
    const size_t sb_slots = carve(nullptr, caps, nslots, nullptr);
    const size_t sb = sb_slots + sizeof(Ctl) * (size_t)nslots + 256;
    HostTimer ta("slot arena");
    void* base = workspace(st, WS_SEARCH, sb);
    if (!base) {
      status = set_error(MPAP_ERR_OUT_OF_MEMORY, "search slot allocation failed");
      break;
    }
    SearchArgs A{};
    A.samples = rm->d_samples;
    A.node_base = rm->d_node_base;
    A.n_env = nullptr;
    A.row_ptr = rm->d_row_ptr;
    A.edges = rm->d_edges;
    A.peak = rm->d_peak;
    A.stride = rm->prm.stride;
    A.pos_dim = rm->prm.pos_dim;
    A.T = lambda * rm->prm.r;
    A.queries = d_q;
    A.qidx = d_qidx;
    A.nq = nrun;
    A.work = d_work;
    A.caps = caps;
    carve(&A, caps, nslots, static_cast<char*>(base));
    A.paths = d_paths;
    A.path_cap = path_cap;
    A.results = d_res;
    A.waves = d_waves;
    A.waves_cap = trace ? waves_cap : 0;
    // n_env lives with the roadmap's node bases: n_env[b] = node_base[b+1]-node_base[b]
    int32_t* d_nenv = nullptr;
    CKS(cudaMallocAsync(&d_nenv, sizeof(int32_t) * rm->B, st));
    CKS(cudaMemcpyAsync(d_nenv, rm->n.data(), sizeof(int32_t) * rm->B, cudaMemcpyHostToDevice, st));
    A.n_env = d_nenv;
    CKS(cudaMemcpyAsync(d_qidx, todo.data(), sizeof(int32_t) * nrun, cudaMemcpyHostToDevice, st));
    CKS(cudaMemsetAsync(d_work, 0, sizeof(int), st));
    // lazy roadmap (NEXT-1 part i): the whole-grid search suspends before a
    // wave whose heads have unevaluated rows; evaluate them and resume
    if (rm->lazy && !grid_mode && !cluster_mode) {
      mpap_status se = evaluate_rows_device(const_cast<mpap_roadmap*>(rm), nullptr, 0, st);
      if (se != MPAP_OK) return se;
    }
    const bool lazy_grid = rm->lazy && (grid_mode || cluster_mode);
    int32_t* d_req = nullptr;
    int* d_nreq = nullptr;
    if (lazy_grid) {
      CKS(cudaMallocAsync(&d_req, sizeof(int32_t) * std::max<int64_t>(rm->node_base[rm->B], 1), st));
      CKS(cudaMallocAsync(&d_nreq, sizeof(int), st));
      A.ready = rm->d_ready;
      A.req = d_req;
      A.nreq = d_nreq;
    }
    A.resume = 0;
    if (lazy_grid) {
      Ctl* d_ctl = reinterpret_cast<Ctl*>(static_cast<char*>(base) + ((sb_slots + 255) & ~size_t(255)));
      for (;;) {
        CKS(cudaMemsetAsync(d_nreq, 0, sizeof(int), st));
        {
          ProfScope ps("k_search", st);
          if (grid_mode) {
            void* args[] = {&A, &d_ctl};
            const void* fn = trace ? (const void*)k_search_grid<true> : (const void*)k_search_grid<false>;
            CKS(cudaLaunchCooperativeKernel(fn, dim3(grid_ctas), dim3(kST), args, kBigSmem, st));
          } else {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(nslots * csize);
            cfg.blockDim = dim3(kST);
            cfg.dynamicSmemBytes = kBigSmem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = csize;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (trace) CKS(cudaLaunchKernelEx(&cfg, k_search_cluster<true>, A, d_ctl));
            else CKS(cudaLaunchKernelEx(&cfg, k_search_cluster<false>, A, d_ctl));
          }
        }
        note_launch();
        note_team(grid_mode ? 0 : 1);
        int nreq = 0;
        CKS(cudaMemcpyAsync(&nreq, d_nreq, sizeof(int), cudaMemcpyDeviceToHost, st));
        CKS(cudaStreamSynchronize(st));
        if (nreq == 0) break;
        mpap_status se = evaluate_rows_device(const_cast<mpap_roadmap*>(rm), d_req, nreq, st);
        if (se != MPAP_OK) return se;
        A.resume = 1;
      }
      CKS(cudaFreeAsync(d_req, st));
      CKS(cudaFreeAsync(d_nreq, st));
    } else {
      ProfScope ps("k_search", st);
      Ctl* d_ctl = reinterpret_cast<Ctl*>(static_cast<char*>(base) + ((sb_slots + 255) & ~size_t(255)));
      if (grid_mode) {
        void* args[] = {&A, &d_ctl};
        const void* fn = trace ? (const void*)k_search_grid<true> : (const void*)k_search_grid<false>;
        CKS(cudaLaunchCooperativeKernel(fn, dim3(grid_ctas), dim3(kST), args, kBigSmem, st));
      } else if (cluster_mode) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nslots * csize);
        cfg.blockDim = dim3(kST);
        cfg.dynamicSmemBytes = kBigSmem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (trace) CKS(cudaLaunchKernelEx(&cfg, k_search_cluster<true>, A, d_ctl));
        else CKS(cudaLaunchKernelEx(&cfg, k_search_cluster<false>, A, d_ctl));
      } else if (trace) {
        k_search<true><<<nslots, kST, kBigSmem, st>>>(A);
      } else {
        k_search<false><<<nslots, kST, kBigSmem, st>>>(A);
      }
      note_launch();
      note_team(grid_mode ? 0 : cluster_mode ? 1 : 2);
    }
    CKS(cudaGetLastError());
    CKS(cudaFreeAsync(d_nenv, st));
    CKS(cudaMemcpyAsync(hres.data(), d_res, sizeof(mpap_result) * nq, cudaMemcpyDeviceToHost, st));
    {
      HostTimer tsync("search sync");
      CKS(cudaStreamSynchronize(st));
    }
    std::vector<int32_t> again;
    int mask = 0;
    for (int k : todo) {
      if (hres[k].status >= kRetryBase) {
        again.push_back(k);
        mask |= hres[k].status - kRetryBase;
        retries[k]++;
      }
    }
    if (mask & OVF_STAIR) caps.K *= 2;
    if (mask & OVF_RING) caps.R = 0;   // a plan beyond the ring: rerun on the pending list
    if (mask & OVF_LABELS) caps.L *= 2;
    if (mask & OVF_CAND) caps.C *= 2;
    rm->hint_K = std::max(rm->hint_K, caps.K);   // later searches on this roadmap start there
    rm->hint_L = std::max(rm->hint_L, caps.L);
    rm->hint_C = std::max(rm->hint_C, caps.C);
    if (dev >= 0 && dev < kMaxDevices) {   // ... and, within the arena budget, later roadmaps
      std::lock_guard<std::mutex> lk(g_cap_mu);
      CapHint& h = g_cap_hint[dev];
      h.K = std::max(h.K, caps.K);
      h.L = std::max(h.L, caps.L);
      h.C = std::max(h.C, caps.C);
    }
    todo.swap(again);
  }
  if (status == MPAP_OK && !todo.empty()) status = set_error(MPAP_ERR_OUT_OF_MEMORY, "search capacity regrow limit");
  for (int k : todo) {   // queries that could not complete carry the error, never a stale record
    hres[k] = mpap_result{};
    hres[k].status = status;
  }
  // write retry counts into the results
  for (int k = 0; k < nq; ++k) hres[k].retries = retries[k];
  if (mem == MPAP_MEM_DEVICE) {
    CKS(cudaMemcpyAsync(d_res, hres.data(), sizeof(mpap_result) * nq, cudaMemcpyHostToDevice, st));
  } else {
    std::memcpy(results, hres.data(), sizeof(mpap_result) * nq);
    CKS(cudaMemcpyAsync(paths, d_paths, sizeof(int32_t) * (size_t)nq * path_cap, cudaMemcpyDeviceToHost, st));
  }
  if (trace)
    CKS(cudaMemcpyAsync(h_waves, d_waves, sizeof(mpap_wave) * (size_t)nq * waves_cap, cudaMemcpyDeviceToHost, st));
  CKS(cudaStreamSynchronize(st));
  CKS(cudaFreeAsync(d_q, st));
  CKS(cudaFreeAsync(d_qidx, st));
  CKS(cudaFreeAsync(d_work, st));
  if (mem != MPAP_MEM_DEVICE) {
    CKS(cudaFreeAsync(d_res, st));
    CKS(cudaFreeAsync(d_paths, st));
  }
  if (d_waves) CKS(cudaFreeAsync(d_waves, st));
  if (mem == MPAP_MEM_DEVICE) CKS(cudaStreamSynchronize(st));
  if (MPAP_DEBUG_CHECKS && nq == 1 && getenv("MPAP_PHASE_LOG")) {
    static unsigned long long ph[kPhaseWaves][8];
    static int pst[kPhaseWaves][4];
    CKS(cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph)));
    CKS(cudaMemcpyFromSymbol(pst, g_phase_stat, sizeof(pst)));
    const int nw = std::min(kPhaseWaves, (int)results[0].waves);
    for (int w = 0; w < nw; ++w)
      fprintf(stderr, "[phase] wave %d us expand %.1f group %.1f scatter %.1f merge %.1f retire %.1f partition %.1f "
              "| nbig %d nsmall %d max_kc %d max_m %d\n", w, (ph[w][1] - ph[w][0]) * 1e-3, (ph[w][2] - ph[w][1]) * 1e-3,
              (ph[w][3] - ph[w][2]) * 1e-3, (ph[w][4] - ph[w][3]) * 1e-3, (ph[w][5] - ph[w][4]) * 1e-3,
              (ph[w][6] - ph[w][5]) * 1e-3, pst[w][0], pst[w][1], pst[w][2], pst[w][3]);
    std::memset(pst, 0, sizeof(pst));
    CKS(cudaMemcpyToSymbol(g_phase_stat, pst, sizeof(pst)));
    unsigned long long mc[6];
    CKS(cudaMemcpyFromSymbol(mc, g_merge_cyc, sizeof(mc)));
    const double nn = (double)std::max(mc[5], 1ull);
    fprintf(stderr, "[merge] large nodes %llu, cycles per node: load+sort %.0f survivors %.0f kills %.0f "
            "order+labels %.0f tail %.0f\n", mc[5], mc[0] / nn, mc[1] / nn, mc[2] / nn, mc[3] / nn, mc[4] / nn);
    std::memset(mc, 0, sizeof(mc));
    CKS(cudaMemcpyToSymbol(g_merge_cyc, mc, sizeof(mc)));
  }
  if (MPAP_DEBUG_CHECKS) {
    unsigned long long fails = 0;
    CKS(cudaMemcpyFromSymbol(&fails, g_dcheck_fail, sizeof(fails)));
    if (fails) return set_error(MPAP_ERR_CUDA, "MPAP_DEBUG_CHECKS: out-of-range store index in the search kernels");
  }
  return status;
}

}  // namespace mpap
