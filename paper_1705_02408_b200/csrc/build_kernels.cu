// paper_1705_02408_b200/csrc/build_kernels.cu -- roadmap build on sm_100a.
//
// Alg. 2 BuildGraph and Alg. 1 line 2, the perception
// heuristic precompute (heuristic §4.1, learned
// heuristic §5.2), as three kernels per batch of environments:
//
//   k_near   one warp per row u: Near(V \ {u}, u, r_n) = {v : Cost(u,v) < r}
//            (A2.3 P:213).  Kinematic cost is evaluated by every lane;
//            double-integrator pairs pass a conservative prefilter first and
//            the survivors are compacted into a per-warp shared-memory queue so
//            the root-isolation cascade (reading R7) always runs 32-wide.
//            Entries come out in ascending v (ballot-ordered appends).
//   k_scan   exclusive scan of the row counts -> CSR row_ptr (int64).
//   k_edges  one warp per row, one edge at a time: Collision(u,v) (P:190,
//            A2.5 P:215; reading R8) with lanes over polyline segments, then
//            the heuristic summary (R9, R10, R12) with lanes over timesteps;
//            per 32-step chunk the warp culls features/boxes against the
//            chunk's bounding box (exact: a culled item provably fails its
//            test), and folds the per-step increments in time
//            order with shuffles.  Writes the 16-byte EdgeRec.
//
// The position dimension D (2 or 3) and the dynamics are template parameters
// so every per-axis array lives in registers.  Every floating-point
// expression follows DESIGN.md §3 ("Numeric contract") operation by operation
// and is compiled with --fmad=false (no contraction), so results are
// bit-identical to the CPU oracle without sharing its code.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "mpap_internal.cuh"
#include "traj.cuh"

namespace mpap {

#define FULL 0xffffffffu
#ifndef MPAP_BBOX_WARP
#define MPAP_BBOX_WARP 1
#endif
#ifndef MPAP_STAT_WARP
#define MPAP_STAT_WARP 1
#endif
#ifndef MPAP_NEAR_F32
#define MPAP_NEAR_F32 1      // k_near's level-2 interval filter in single precision with certified margins
#endif
#ifndef MPAP_FOLD_SMEM_TRAJ
#define MPAP_FOLD_SMEM_TRAJ 1
#endif
#ifndef MPAP_FOLD_MIN_BLOCKS
#define MPAP_FOLD_MIN_BLOCKS 3
#endif
#ifndef MPAP_EDGES_MIN_BLOCKS
#define MPAP_EDGES_MIN_BLOCKS 4
#endif
#ifndef MPAP_KWARPS
#define MPAP_KWARPS 4
#endif
constexpr int kWarps = MPAP_KWARPS;       // warps per block of the edge kernels
constexpr int kNearWarps = 8;             // warps per block of k_near
constexpr double kCullMargin = 1e-6;      // absolute; >> rounding of O(100) coordinates

// min / max of finite doubles for the conservative culls (fmin / fmax carry
// NaN handling: ~10 instructions each on sm_100a; these are 3)
__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// Approximate single-precision sqrt / division (MUFU, ~1e-7 relative error)
// for the conservative culls and heading arcs only: their margins (1e-4 m,
// 2e-3 rad, 2e-4 in a cosine) exceed the error by three orders of magnitude.
// (The build compiles with -prec-sqrt/-prec-div: sqrtf and / are the
// correctly rounded multi-instruction sequences.)
__device__ __forceinline__ float sqrt_cull(float x) { return x > 0.0f ? x * rsqrtf(x) : 0.0f; }
__device__ __forceinline__ float div_cull(float a, float b) { return __fdividef(a, b); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// geometry (DESIGN.md §3 "slab")
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ bool seg_box(const double* A, const double* B, const double* box) {
  double t0 = 0.0, t1 = 1.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double lo = box[k], hi = box[D + k];
    const double dk = B[k] - A[k];
    if (dk == 0.0) {
      if (A[k] < lo || A[k] > hi) return false;
    } else {
      const double inv = __drcp_rn(dk);   // == 1.0 / dk (both correctly rounded)
      double ta = (lo - A[k]) * inv;
      double tb = (hi - A[k]) * inv;
      if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return false;
    }
  }
  return true;
}

template <int D>
__device__ __forceinline__ bool outside_ws(const double* p, const DevParams& P) {
  bool out = false;
#pragma unroll
  for (int k = 0; k < D; ++k)
    if (p[k] < P.ws_lo[k] || p[k] > P.ws_hi[k]) out = true;
  return out;
}

// ---------------------------------------------------------------------------
// double-integrator steering (reading R7)
// ---------------------------------------------------------------------------
struct DiCoef { double vv, av, aa, B, C, D, ru; };

template <int D>
__device__ __forceinline__ void di_coefs(const double* su, const double* sv, double ru, DiCoef& k) {
  double vv = 0.0, av = 0.0, aa = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double p0 = su[j], v0 = su[D + j], p1 = sv[j], v1 = sv[D + j];
    const double a = p1 - p0;
    vv = vv + ((v0 * v0 + v0 * v1) + v1 * v1);
    av = av + a * (v0 + v1);
    aa = aa + a * a;
  }
  k.vv = vv; k.av = av; k.aa = aa; k.ru = ru;
  k.B = (4.0 * ru) * vv;
  k.C = (24.0 * ru) * av;
  k.D = (36.0 * ru) * aa;
}

__device__ __forceinline__ double di_q(const DiCoef& k, double t) { return ((t * t - k.B) * t + k.C) * t - k.D; }
__device__ __forceinline__ double di_qp(const DiCoef& k, double t) {
  return ((4.0 * (t * t)) - (2.0 * k.B)) * t + k.C;
}
__device__ __forceinline__ double di_c(const DiCoef& k, double t) {
  const double t2 = t * t;
  const double t3 = t2 * t;
  return t + k.ru * ((((4.0 * k.vv) / t) - ((12.0 * k.av) / t2)) + ((12.0 * k.aa) / t3));
}

template <int WHICH>
__device__ __forceinline__ double di_f(const DiCoef& k, double t) { return WHICH == 0 ? di_q(k, t) : di_qp(k, t); }

template <int WHICH>
__device__ double di_bisect(const DiCoef& k, double lo, double hi, unsigned& iters) {
  const bool hi_pos = di_f<WHICH>(k, hi) > 0.0;
  for (int it = 0; it < 100; ++it) {
    const double mid = lo + 0.5 * (hi - lo);
    if (!(mid > lo && mid < hi)) break;
    ++iters;
    if ((di_f<WHICH>(k, mid) > 0.0) == hi_pos) hi = mid; else lo = mid;
  }
  return hi;
}

// Returns true and (c*, tau*) when c has a local minimiser on (0, r].
template <int D>
__device__ bool cost_di(const double* su, const double* sv, double ru, double r, double& c_out, double& tau_out,
                        unsigned& iters) {
  DiCoef k;
  di_coefs<D>(su, sv, ru, k);
  if (k.D == 0.0) return false;
  double bp[4];
  int nb = 0;
  bp[nb++] = 0.0;
  const double tc = (k.B > 0.0) ? sqrt(k.B / 6.0) : 0.0;
  double pieces[3];
  int np = 0;
  pieces[np++] = 0.0;
  if (tc > 0.0 && tc < r) pieces[np++] = tc;
  pieces[np++] = r;
  for (int s = 0; s + 1 < np; ++s) {
    const double a = pieces[s], b = pieces[s + 1];
    const double fa = di_qp(k, a), fb = di_qp(k, b);
    if ((fa > 0.0 && fb < 0.0) || (fa < 0.0 && fb > 0.0)) bp[nb++] = di_bisect<1>(k, a, b, iters);
  }
  bp[nb++] = r;
  for (int i = 1; i < nb; ++i) {  // ascending already; kept for the contract
    const double x = bp[i];
    int j = i - 1;
    while (j >= 0 && bp[j] > x) { bp[j + 1] = bp[j]; --j; }
    bp[j + 1] = x;
  }
  bool found = false;
  double best_c = 0.0, best_t = 0.0;
  for (int s = 0; s + 1 < nb; ++s) {
    const double a = bp[s], b = bp[s + 1];
    if (!(b > a)) continue;
    if (di_q(k, a) <= 0.0 && di_q(k, b) > 0.0) {
      const double t = di_bisect<0>(k, a, b, iters);
      const double c = di_c(k, t);
      if (!found || c < best_c || (c == best_c && t < best_t)) { found = true; best_c = c; best_t = t; }
    }
  }
  if (!found) return false;
  c_out = best_c;
  tau_out = best_t;
  return true;
}

// Work counters (always on; one atomicAdd per row per counter).
enum {
  W_PAIRS = 0, W_PREFILTER_PASS, W_BISECT_ITERS, W_EDGES, W_COLL_SEGS, W_COLL_BOX_TESTS, W_STEPS, W_RANGE_TESTS,
  W_FOV_TESTS, W_OCCL_SEGS, W_OCCL_BOX_TESTS, W_MLP, W_FREE_EDGES, W_CULL_TESTS, W_NUM
};

// ---------------------------------------------------------------------------
// k_near
// ---------------------------------------------------------------------------
template <int D, int DYN>
__global__ void __launch_bounds__(kNearWarps * 32) k_near(const double* __restrict__ samples,
                                                      const int64_t* __restrict__ node_base,
                                                      const int32_t* __restrict__ n_env, DevParams P, int cap,
                                                      int32_t* __restrict__ cnt, NearRec* __restrict__ scratch,
                                                      int* __restrict__ overflow,
                                                      unsigned long long* __restrict__ work) {
  constexpr int NS = DYN ? 2 * D : D;   // state doubles used by the cost
  __shared__ int queue[kNearWarps][64];
  // interval tables of the level-2 filter: [level][interval] = {ta, tb, 1/tb, 1/tb^3}
  // for the whole range (level 0), quarters (1) and sixteenths (2) of (0, r]
  __shared__ double s_near[3][16][4];
#if MPAP_NEAR_F32
  __shared__ float4 s_nearf[3][16];   // the same table in single precision (the FP32 filter)
#endif
  if (DYN == 1 && threadIdx.x < 21) {
    const int t = threadIdx.x;
    const int lvl = (t == 0) ? 0 : (t < 5) ? 1 : 2;
    const int jj = (t == 0) ? 0 : (t < 5) ? t - 1 : t - 5;
    const int nseg = (lvl == 0) ? 1 : (lvl == 1) ? 4 : 16;
    const double ta = P.r * (double)jj / (double)nseg;
    const double tb = P.r * (double)(jj + 1) / (double)nseg;
    s_near[lvl][jj][0] = ta;
    s_near[lvl][jj][1] = tb;
    s_near[lvl][jj][2] = 1.0 / tb;
    s_near[lvl][jj][3] = 1.0 / (tb * tb * tb);
#if MPAP_NEAR_F32
    s_nearf[lvl][jj] = make_float4((float)ta, (float)tb, (float)(1.0 / tb), (float)(1.0 / (tb * tb * tb)));
#endif
  }
  __syncthreads();
  const int b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = n_env[b];
  const int u = blockIdx.x * kNearWarps + warp;
  if (u >= nb) return;  // warp-uniform
  const int64_t row = node_base[b] + u;
  if (row < P.row_lo || row >= P.row_hi) {   // row-sharded build: another rank owns this row
    if (lane == 0) cnt[row] = 0;
    return;
  }
  const int stride = P.stride;
  const double* envs = samples + node_base[b] * stride;
  double su[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) su[j] = envs[(int64_t)u * stride + j];
  NearRec* out = scratch + row * (int64_t)cap;
  const double r = P.r;
  const unsigned lt = lanemask_lt();
  int count = 0;
  unsigned n_pass = 0, n_iter = 0;
  if (DYN == 0) {
    for (int v0 = 0; v0 < nb; v0 += 32) {
      const int v = v0 + lane;
      bool keep = false;
      double c = 0.0;
      if (v < nb && v != u) {
        const double* sv = envs + (int64_t)v * stride;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const double dk = sv[k] - su[k];
          acc = acc + dk * dk;
        }
        c = sqrt(acc);
        keep = c < r;
      }
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) {
        const int pos = count + __popc(m & lt);
        if (pos < cap) out[pos] = NearRec{v, (float)c, c / P.nominal_speed};
      }
      count += __popc(m);
    }
  } else {
    const double ru = P.control_weight;
    double v02 = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) v02 += su[D + j] * su[D + j];
    // level 1 (necessary conditions of c* < r): min energy to
    // move by Dp with free end velocity is 3|Dp|^2/tau^3, and by AM-GM
    // tau + r_u |dv|^2 / tau >= 2 sqrt(r_u) |dv|; 1e-9 relative slack
    const double bp = (sqrt(v02) * r + r * r / sqrt(3.0 * ru)) * (1.0 + 1e-9);
    const double bv = (r / (2.0 * sqrt(ru))) * (1.0 + 1e-9);
    const double bp2 = bp * bp, bv2 = bv * bv;
#if MPAP_NEAR_F32
    const float ruf = (float)ru, rf = __double2float_ru(r);
#endif
    int qn = 0;
    auto process = [&](int k) {
      bool ok = false;
      double c = 0.0, tau = 0.0;
      int v = -1;
      if (lane < k) {
        v = queue[warp][lane];
        double sv[NS];
        const double* svp = envs + (int64_t)v * stride;
#pragma unroll
        for (int j = 0; j < NS; ++j) sv[j] = svp[j];
        ++n_pass;
        ok = cost_di<D>(su, sv, ru, r, c, tau, n_iter) && (c < r);
      }
      const unsigned m = __ballot_sync(FULL, ok);
      if (ok) {
        const int pos = count + __popc(m & lt);
        if (pos < cap) out[pos] = NearRec{v, (float)c, tau};
      }
      count += __popc(m);
    };
    for (int v0 = 0; v0 < nb; v0 += 32) {
      const int v = v0 + lane;
      bool pf = false;
      if (v < nb && v != u) {
        const double* sv = envs + (int64_t)v * stride;
        double dp2 = 0.0, dv2 = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double a = sv[j] - su[j], e = sv[D + j] - su[D + j];
          dp2 += a * a;
          dv2 += e * e;
        }
        pf = !(dp2 > bp2 || dv2 > bv2);
        if (pf) {
          // level 2: c(tau) = tau + r_u (12 |a - s tau/2|^2 / tau^3 + |dv|^2 / tau)
          // (a = p1 - p0, s = v0 + v1).  On [ta, tb]: tau >= ta, |dv|^2/tau >=
          // |dv|^2/tb, and |a - s tau/2|^2 = aa - tau a.s + tau^2 ss/4 is a
          // convex quadratic whose minimum over [ta, tb] is taken at the
          // clamped vertex.  A pair whose bound reaches r on every interval
          // has no edge.
          double ss = 0.0, as = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const double e = sv[D + j] + su[D + j];
            const double a = sv[j] - su[j];
            ss += e * e;
            as += a * e;
          }
          // Lower bound of c on [ta, tb] (reciprocals of tb from the block's
          // table): tested on [0, r], then on its 4 quarters, then on the 4
          // sixteenths of each quarter that is still possible.
#if MPAP_NEAR_F32
          // The same bound in single precision, made conservative (DESIGN.md
          // §7): g2 is lowered by 1e-6 of the magnitude of its terms (> 16
          // float roundings of the conversions and the 5 operations), L by a
          // further 1e-6 relative (the table's and r_u's roundings), and r is
          // rounded up.  The float clamped vertex moves g by O(ss eps^2 r^2),
          // far inside the margin.  A pair with a tiny ss (float underflow)
          // is kept.
          const float dp2f = (float)dp2, asf = (float)as, ssf = (float)ss, dv2f = (float)dv2;
          const bool ss_ok = ssf > 1e-30f || ss == 0.0;
          const float tvf = (ssf > 1e-30f) ? 2.0f * asf / ssf : 0.0f;
          auto possible_on = [&](int lvl, int jj) -> bool {
            const float4 tt = s_nearf[lvl][jj];   // ta, tb, 1/tb, 1/tb^3
            const float tq = fminf(fmaxf(tvf, tt.x), tt.y);
            const float t1 = tq * asf, t2 = tq * tq * ssf * 0.25f;
            const float g2 = dp2f - t1 + t2;
            const float g2lo = fmaxf(g2 - 1e-6f * (dp2f + fabsf(t1) + t2), 0.0f);
            const float L = tt.x + ruf * (12.0f * g2lo * tt.w + dv2f * tt.z);
            return !ss_ok || L * (1.0f - 1e-6f) < rf;
          };
#else
          const double tv = (ss > 0.0) ? 2.0 * as / ss : 0.0;   // vertex of the quadratic
          auto possible_on = [&](int lvl, int jj) -> bool {
            const double ta = s_near[lvl][jj][0], tb = s_near[lvl][jj][1];
            const double tq = dmin(dmax(tv, ta), tb);   // finite operands: no NaN handling needed
            const double g2 = dmax(dp2 - tq * as + tq * tq * ss * 0.25, 0.0);
            const double L = ta + ru * (12.0 * g2 * s_near[lvl][jj][3] + dv2 * s_near[lvl][jj][2]);
            return L * (1.0 - 1e-9) < r;
          };
#endif
          bool possible = false;
          if (possible_on(0, 0)) {
            for (int q = 0; q < 4 && !possible; ++q) {
              if (!possible_on(1, q)) continue;
              for (int jj = 4 * q; jj < 4 * q + 4 && !possible; ++jj) possible = possible_on(2, jj);
            }
          }
          pf = possible;
        }
      }
      const unsigned m = __ballot_sync(FULL, pf);
      if (pf) queue[warp][qn + __popc(m & lt)] = v;
      qn += __popc(m);
      __syncwarp();
      if (qn >= 32) {
        process(32);
        const int rest = qn - 32;
        int tmp = 0;
        if (lane < rest) tmp = queue[warp][32 + lane];
        __syncwarp();
        if (lane < rest) queue[warp][lane] = tmp;
        __syncwarp();
        qn = rest;
      }
    }
    if (qn > 0) process(qn);
  }
  if (lane == 0) {
    cnt[row] = count;
    if (count > cap) atomicMax(overflow, count);
  }
  for (int o = 16; o > 0; o >>= 1) {
    n_pass += __shfl_xor_sync(FULL, n_pass, o);
    n_iter += __shfl_xor_sync(FULL, n_iter, o);
  }
  if (lane == 0) {
    atomicAdd(&work[W_PAIRS], (unsigned long long)(nb - 1));
    if (n_pass) atomicAdd(&work[W_PREFILTER_PASS], (unsigned long long)n_pass);
    if (n_iter) atomicAdd(&work[W_BISECT_ITERS], (unsigned long long)n_iter);
  }
}

// ---------------------------------------------------------------------------
// k_scan: single-block exclusive scan (int32 counts -> int64 offsets)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_scan(const int32_t* __restrict__ cnt, int64_t N,
                                               int64_t* __restrict__ row_ptr) {
  __shared__ int64_t wsum[32];
  const int t = threadIdx.x;
  const int64_t chunk = (N + 1023) / 1024;
  const int64_t lo = t * chunk, hi = min(N, lo + chunk);
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += cnt[i];
  const int lane = t & 31, w = t >> 5;
  int64_t x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t y = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t z = __shfl_up_sync(FULL, y, o);
      if (lane >= o) y += z;
    }
    wsum[lane] = y;
  }
  __syncthreads();
  int64_t excl = x - s + (w > 0 ? wsum[w - 1] : 0);
  for (int64_t i = lo; i < hi; ++i) {
    row_ptr[i] = excl;
    excl += cnt[i];
  }
  if (t == 1023) row_ptr[N] = wsum[31];
}

// ---------------------------------------------------------------------------
// k_edges: collision + heuristic summary per edge
// ---------------------------------------------------------------------------
// Per-warp shared scratch: culled feature coordinates (SoA) and culled boxes.
template <int D>
struct WarpLists {
  double* f[D];                 // [F_max] each; f[0], f[1] interleaved as (x, y) pairs (fxy), f[D-1] = z
  double2* fxy;                 // [F_max] (x, y) of the kept features: one LDS.128 per feature in the step loop
  double* box;                  // [O_max][2D]
  unsigned long long* fmask;    // [F_max] per-feature box masks
  float4* fenv;                 // [F_max] the current environment's features (float x, y, z), staged per env
  float* boxf;                  // [O_max][2D] the chunk's culled boxes (float), for the occluder masks
  int* fidx;                    // [F_max] the chunk's kept features' indices into fenv (MPAP_FMASK_F32), or
                                //         the edge's range candidates (MPAP_CULL_EDGE)
  const float* arc;             // [2] cos, sin of the bearing cull's half angle (block-shared)
};
#ifndef MPAP_CULL_FENV
#define MPAP_CULL_FENV 1     // feature cull from per-environment float copies staged in shared memory
#endif
#ifndef MPAP_FMASK_PAIRS
#define MPAP_FMASK_PAIRS 1   // occluder masks of <= 16 kept features: lanes over (feature, box) pairs
#endif
#ifndef MPAP_CULL_TWOSTAGE
#define MPAP_CULL_TWOSTAGE 1   // feature cull: range over all features, bearing over the compacted survivors
#endif
#ifndef MPAP_CULL_BRANCHFREE
#define MPAP_CULL_BRANCHFREE 1   // bearing cull evaluated by every lane (no divergent branches)
#endif
#ifndef MPAP_CULL_EDGE
#define MPAP_CULL_EDGE 1     // feature range cull per edge first, each chunk's range cull over the edge's list
#endif
#ifndef MPAP_FMASK_F32
#define MPAP_FMASK_F32 0     // occluder masks in single precision, lanes over boxes (measured slower: 177.4 -> 196.3 ms)
#endif
// Per-warp shared scratch layout (in doubles; counts fs, os rounded up to a
// multiple of 4 so every array stays 16-byte aligned):
//   f[D][fs], box[os][2D], fmask[fs], fenv[fs] float4 (MPAP_CULL_FENV),
//   boxf[os][2D] float (MPAP_FMASK_F32), fidx[fs] int (both).
__host__ __device__ constexpr size_t warp_scratch_doubles(int D, size_t fs, size_t os) {
  return fs * (D + 1) + os * 2 * D + (MPAP_CULL_FENV ? fs * 2 : 0) + (MPAP_FMASK_F32 ? os * D : 0) +
         ((MPAP_CULL_FENV && (MPAP_FMASK_F32 || MPAP_CULL_EDGE)) ? fs / 2 : 0);
}
__host__ __device__ constexpr size_t round4(int x) { return (size_t)((x + 3) & ~3); }

// Work counters: warp-uniform counts go to the warp's shared-memory slots
// (written by lane 0 only); per-lane counts live in four registers and are
// folded into the slots once per edge.
// kept feature i, axis q: x and y interleaved in fxy, z in its own array
#define FREF(L, q, i) ((q) < 2 ? (L).f[q][2 * (i)] : (L).f[q][i])

// One staged box (lo[D], hi[D] contiguous, 16-byte aligned) with 16-byte
// shared loads.
template <int D>
__device__ __forceinline__ void load_box(const double* bx, double* b) {
  const double2* p = reinterpret_cast<const double2*>(bx);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double2 v = p[k];
    b[2 * k] = v.x;
    b[2 * k + 1] = v.y;
  }
}

struct Work {
  unsigned* sm;   // [W_NUM] per warp
  unsigned occl_segs, occl_tests, coll_segs, coll_tests;
  __device__ __forceinline__ void add(int lane, int i, unsigned x) {
    if (lane == 0) sm[i] += x;
  }
  __device__ __forceinline__ void flush(int lane) {
    const unsigned a = __reduce_add_sync(FULL, occl_segs), b = __reduce_add_sync(FULL, occl_tests);
    const unsigned c = __reduce_add_sync(FULL, coll_segs), e = __reduce_add_sync(FULL, coll_tests);
    if (lane == 0) {
      sm[W_OCCL_SEGS] += a;
      sm[W_OCCL_BOX_TESTS] += b;
      sm[W_COLL_SEGS] += c;
      sm[W_COLL_BOX_TESTS] += e;
    }
    occl_segs = occl_tests = coll_segs = coll_tests = 0;
  }
};

__device__ __forceinline__ double warp_min(double x) {
  for (int o = 16; o > 0; o >>= 1) x = dmin(x, __shfl_xor_sync(FULL, x, o));
  return x;
}
__device__ __forceinline__ double warp_max(double x) {
  for (int o = 16; o > 0; o >>= 1) x = dmax(x, __shfl_xor_sync(FULL, x, o));
  return x;
}

// Boxes overlapping [lo - m, hi + m] -> coordinates in the warp's list.  A box
// outside that region cannot be hit by any segment inside [lo, hi] (its slab
// interval is empty by a margin far above rounding).
template <int D>
__device__ int cull_boxes(const double* __restrict__ box, int O, const double* lo, const double* hi, double m,
                          double* out, int lane, float* outf = nullptr) {
  int nc = 0;
  const unsigned lt = lanemask_lt();
  __syncwarp();
  for (int o0 = 0; o0 < O; o0 += 32) {
    const int o = o0 + lane;
    bool keep = false;
    double bl[2 * D];
    if (o < O) {
      keep = true;
      const double2* src = reinterpret_cast<const double2*>(box + (size_t)o * 2 * D);   // 16-byte aligned records
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double2 v = __ldg(src + k);
        bl[2 * k] = v.x;
        bl[2 * k + 1] = v.y;
      }
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (bl[k] > hi[k] + m || bl[D + k] < lo[k] - m) keep = false;
    }
    const unsigned msk = __ballot_sync(FULL, keep);
    if (keep) {
      const int pos = nc + __popc(msk & lt);
      double2* dst = reinterpret_cast<double2*>(out + (size_t)pos * 2 * D);
#pragma unroll
      for (int k = 0; k < D; ++k) dst[k] = make_double2(bl[2 * k], bl[2 * k + 1]);
      if (outf) {
#pragma unroll
        for (int k = 0; k < 2 * D; ++k) outf[(size_t)pos * 2 * D + k] = (float)bl[k];
      }
    }
    nc += __popc(msk);
  }
  __syncwarp();
  return nc;
}

// Does the closed segment [A, B] (Dv = B - A) hit one of the listed boxes?
// The slab test of DESIGN.md §3 with the per-axis reciprocal 1/Dv_k computed
// once per segment (the value the per-box formula computes); a box separated
// from the segment's bounding box by more than kCullMargin is skipped (its
// slab test is provably false).  With USE_MASK only the boxes whose bit is
// set in `mask` are visited (a superset of the boxes that can be hit).
// Returns hit | (slab tests executed << 1).
template <int D, bool USE_MASK>
__device__ __forceinline__ unsigned seg_hits_boxes(const double* A, const double* B, const double* Dv,
                                                   const double* bl, int nl, unsigned long long mask) {
  double inv[D], slo[D], shi[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    inv[k] = (Dv[k] != 0.0) ? __drcp_rn(Dv[k]) : 0.0;   // == 1.0 / Dv[k]
    slo[k] = dmin(A[k], B[k]) - kCullMargin;
    shi[k] = dmax(A[k], B[k]) + kCullMargin;
  }
  unsigned tests = 0;
  int i = -1;
  for (;;) {
    if (USE_MASK) {
      if (!mask) break;
      i = __ffsll((long long)mask) - 1;
      mask &= mask - 1;
    } else {
      if (++i >= nl) break;
    }
    double bx[2 * D];
    load_box<D>(bl + (size_t)i * 2 * D, bx);
    bool sep = false;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (bx[k] > shi[k] || bx[D + k] < slo[k]) sep = true;
    }
    if (sep) continue;
    ++tests;
    double t0 = 0.0, t1 = 1.0;
    bool hit = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double lo = bx[k], hi = bx[D + k];
      if (Dv[k] == 0.0) {
        if (A[k] < lo || A[k] > hi) hit = false;
      } else {
        double ta = (lo - A[k]) * inv[k];
        double tb = (hi - A[k]) * inv[k];
        if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t0 > t1) hit = false;
      }
    }
    if (hit) return 1u | (tests << 1);
  }
  return tests << 1;
}

// di_traj (traj.cuh) for a whole warp: lane j < D forms c2[j], lane D + j
// forms c3[j] -- the same expressions, one division per lane instead of 2 D
// in sequence -- and every lane receives all of them.
template <int D>
__device__ __forceinline__ void di_traj_warp(const double* su, const double* sv, double tau, int lane, double* c2,
                                             double* c3) {
  const int j = (lane < D) ? lane : (lane < 2 * D) ? lane - D : 0;
  const double tau2 = tau * tau;
  const double tau3 = tau2 * tau;
  const double dp = (sv[j] - su[j]) - su[D + j] * tau;
  const double dl = sv[D + j] - su[D + j];
  const double num = (lane < D) ? (3.0 * dp - dl * tau) : (dl * tau - 2.0 * dp);
  const double q = num / ((lane < D) ? tau2 : tau3);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    c2[i] = __shfl_sync(FULL, q, i);
    c3[i] = __shfl_sync(FULL, q, D + i);
  }
}

// Collision(u,v) of reading R8, warp-cooperative; every lane returns the result.
template <int D, int DYN>
__device__ __forceinline__ bool edge_collision(const DevParams& P, const double* su, const double* sv, double tau,
                               const double* __restrict__ box, int O, WarpLists<D>& L, int lane, Work& W) {
  if (DYN == 0) {
    bool hit = false;
    for (int o0 = 0; o0 < O; o0 += 32) {
      const int o = o0 + lane;
      if (o < O) {
        ++W.coll_tests;
        double bl[2 * D];
#pragma unroll
        for (int k = 0; k < 2 * D; ++k) bl[k] = __ldg(box + (size_t)o * 2 * D + k);
        if (seg_box<D>(su, sv, bl)) hit = true;
      }
      if (__any_sync(FULL, hit)) return true;
    }
    W.add(lane, W_COLL_SEGS, 1);
    return false;
  }
  double c2[D], c3[D];
  di_traj_warp<D>(su, sv, tau, lane, c2, c3);
  const double kc = ceil(tau / P.collision_dt);
  const int Kc = (kc < 1.0) ? 1 : (int)kc;
  // bounding box of the polyline vertices P_0..P_Kc
  double lo[D], hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) { lo[j] = 1e300; hi[j] = -1e300; }
  bool out = false;
  for (int k = lane; k <= Kc; k += 32) {
    const double t = (k == 0) ? 0.0 : ((double)k * tau) / (double)Kc;
    double x[D];
    di_pos<D>(su, c2, c3, t, x);
    if (outside_ws<D>(x, P)) out = true;
#pragma unroll
    for (int j = 0; j < D; ++j) { lo[j] = dmin(lo[j], x[j]); hi[j] = dmax(hi[j], x[j]); }
  }
  if (__any_sync(FULL, out)) return true;
#pragma unroll
  for (int j = 0; j < D; ++j) { lo[j] = warp_min(lo[j]); hi[j] = warp_max(hi[j]); }
  const int nl = cull_boxes<D>(box, O, lo, hi, kCullMargin, L.box, lane);
  W.add(lane, W_CULL_TESTS, O);
  if (nl == 0) return false;
  // segment k = [P_{k-1}, P_k]: each lane forms its end vertex P_k, the
  // start vertex is the previous lane's (the previous chunk's last for lane
  // 0, P_0 = p(0) first) -- the same values as forming both per lane
  for (int k0 = 1; k0 <= Kc; k0 += 32) {
    const int k = k0 + lane;
    bool hit = false;
    if (k <= Kc) {
      const double ta = (k - 1 == 0) ? 0.0 : ((double)(k - 1) * tau) / (double)Kc;
      const double tb = ((double)k * tau) / (double)Kc;
      double A[D], B[D], Dv[D];
      di_pos<D>(su, c2, c3, ta, A);
      di_pos<D>(su, c2, c3, tb, B);
#pragma unroll
      for (int j = 0; j < D; ++j) Dv[j] = B[j] - A[j];
      ++W.coll_segs;
      const unsigned rr = seg_hits_boxes<D, false>(A, B, Dv, L.box, nl, 0ull);
      hit = rr & 1u;
      W.coll_tests += rr >> 1;
    }
    if (__any_sync(FULL, hit)) return true;
  }
  return false;
}

// Output 0 of the 3-8-8-1 MLP (reading R12) for two inputs that share z1
// (two steps of one edge), each in the contract's operation order: hidden-1
// units b1 + W1 z by fma in input order, ReLU; o = b3 then, as each hidden-2
// unit (b2 + W2 h1 in index order, ReLU) is produced, o = fma(W3_i, h2_i, o).
// The weights are read straight from the kernel's parameter bank (a
// __grid_constant__ DevParams) at compile-time indices, so they reach the
// DFMAs through uniform registers -- no shared-memory load per weight (that
// load issue rate had capped k_fold's FP64 pipe at ~45 %).
__device__ __forceinline__ double2 mlp_out0_x2(const double (&w)[kMlpSize], double z0a, double z0b, double z1,
                                                 double z2a, double z2b) {
  double ha[8], hb[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double a = fma(w[i * 3 + 0], z0a, w[24 + i]), b = fma(w[i * 3 + 0], z0b, w[24 + i]);
    a = fma(w[i * 3 + 1], z1, a);
    b = fma(w[i * 3 + 1], z1, b);
    a = fma(w[i * 3 + 2], z2a, a);
    b = fma(w[i * 3 + 2], z2b, b);
    ha[i] = (a > 0.0) ? a : 0.0;
    hb[i] = (b > 0.0) ? b : 0.0;
  }
  double oa = w[120], ob = w[120];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double a = w[96 + i], b = w[96 + i];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a = fma(w[32 + i * 8 + j], ha[j], a);
      b = fma(w[32 + i * 8 + j], hb[j], b);
    }
    oa = fma(w[104 + i], (a > 0.0) ? a : 0.0, oa);
    ob = fma(w[104 + i], (b > 0.0) ? b : 0.0, ob);
  }
  return make_double2(oa, ob);
}

// Stationary points of the cubic position p_j(t) per axis (roots of
// p'(t) = v0 + 2 c2 t + 3 c3 t^2), computed once per edge; -1 = none.
template <int D>
__device__ __forceinline__ void cubic_stationary(const double* su, const double* c2, const double* c3, double* r0,
                                                 double* r1) {
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double A = 3.0 * c3[j], Bq = 2.0 * c2[j], Cq = su[D + j];
    r0[j] = -1.0;
    r1[j] = -1.0;
    if (A != 0.0) {
      const double disc = Bq * Bq - 4.0 * A * Cq;
      if (disc >= 0.0) {
        const double sq = sqrt(disc);
        r0[j] = (-Bq - sq) / (2.0 * A);
        r1[j] = (-Bq + sq) / (2.0 * A);
      }
    } else if (Bq != 0.0) {
      r0[j] = -Cq / Bq;
    }
  }
}

// Bounding box of the positions of steps t in [ta, tb] along the edge: the
// endpoints plus the interior stationary points of the cubic.  It contains
// the contract's step positions up to rounding (~1e-15 relative), far inside
// the culling margins.  Warp-uniform (every lane computes the same box).
template <int D, int DYN>
__device__ __forceinline__ void chunk_bbox(const double* su, const double* sv, const double* c2, const double* c3,
                                           const double* r0, const double* r1, double T, double ta, double tb,
                                           double* lo, double* hi) {
  double xa[D], xb[D];
  if (DYN == 0) {
    const double sa = ta / T, sb = tb / T;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      xa[j] = fma(sa, sv[j] - su[j], su[j]);
      xb[j] = fma(sb, sv[j] - su[j], su[j]);
    }
  } else {
    di_pos<D>(su, c2, c3, ta, xa);
    di_pos<D>(su, c2, c3, tb, xb);
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    lo[j] = dmin(xa[j], xb[j]);
    hi[j] = dmax(xa[j], xb[j]);
    if (DYN == 1) {
      if (r0[j] > ta && r0[j] < tb) {
        const double x = fma(r0[j], fma(r0[j], fma(r0[j], c3[j], c2[j]), su[D + j]), su[j]);
        lo[j] = dmin(lo[j], x);
        hi[j] = dmax(hi[j], x);
      }
      if (r1[j] > ta && r1[j] < tb) {
        const double x = fma(r1[j], fma(r1[j], fma(r1[j], c3[j], c2[j]), su[D + j]), su[j]);
        lo[j] = dmin(lo[j], x);
        hi[j] = dmax(hi[j], x);
      }
    }
  }
}

// chunk_bbox with lane j < D forming axis j (the same expressions: di_pos's
// component j, the stationary points' values), then shuffles.
template <int D, int DYN>
__device__ __forceinline__ void chunk_bbox_warp(const double* su, const double* sv, const double* c2,
                                                const double* c3, const double* r0, const double* r1, double T,
                                                double ta, double tb, int lane, double* lo, double* hi) {
  const int j = (lane < D) ? lane : 0;
  double xa, xb;
  if (DYN == 0) {
    const double sa = ta / T, sb = tb / T;
    xa = fma(sa, sv[j] - su[j], su[j]);
    xb = fma(sb, sv[j] - su[j], su[j]);
  } else {
    xa = fma(ta, fma(ta, fma(ta, c3[j], c2[j]), su[D + j]), su[j]);
    xb = fma(tb, fma(tb, fma(tb, c3[j], c2[j]), su[D + j]), su[j]);
  }
  double l = dmin(xa, xb), h = dmax(xa, xb);
  if (DYN == 1) {
    const double a0 = r0[j], a1 = r1[j];
    if (a0 > ta && a0 < tb) {
      const double x = fma(a0, fma(a0, fma(a0, c3[j], c2[j]), su[D + j]), su[j]);
      l = dmin(l, x);
      h = dmax(h, x);
    }
    if (a1 > ta && a1 < tb) {
      const double x = fma(a1, fma(a1, fma(a1, c3[j], c2[j]), su[D + j]), su[j]);
      l = dmin(l, x);
      h = dmax(h, x);
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    lo[i] = __shfl_sync(FULL, l, i);
    hi[i] = __shfl_sync(FULL, h, i);
  }
}

// Visible-feature counts of a collision-free edge (the k_v of P:324-328, per
// step of reading R9).  Steps are processed 32 at a time (one per lane).  Per
// chunk every lane computes the chunk's bounding box and heading arc
// analytically; the warp culls the features that can be visible from the
// chunk and the boxes that can occlude a sight line into shared memory
// (ballot compaction); each lane then counts the visible features of its
// step and stores the count in `kv_out[k]`.  The increments, the learned
// heuristic and the ordered fold run in k_fold (one thread per edge).
template <int D, int DYN, int HEUR>
__device__ void edge_visible(const DevParams& P, const double* su, const double* sv, double T,
                             const double* __restrict__ feat, int F, const double* __restrict__ box, int O,
                             WarpLists<D>& L, double* ec, int lane, uint16_t* __restrict__ kv_out, Work& W) {
  const double kk = ceil(T / P.dt);
  const int K = (kk < 1.0) ? 1 : (int)kk;
  const double Dl = T / (double)K;
  // per-edge trajectory constants live in the warp's shared scratch `ec`
  // (read per chunk / per step) instead of 4*D registers
  {
    double t2[D], t3[D], q0[D], q1[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { t2[j] = 0.0; t3[j] = 0.0; q0[j] = -1.0; q1[j] = -1.0; }
    if (DYN == 1) {
      di_traj_warp<D>(su, sv, T, lane, t2, t3);
#if MPAP_STAT_WARP
      {   // stationary points: lane j < D solves axis j (cubic_stationary's expressions), then shuffles
        double a2 = t2[0], a3 = t3[0];
#pragma unroll
        for (int i = 1; i < D; ++i)
          if (lane == i) { a2 = t2[i]; a3 = t3[i]; }
        const double A = 3.0 * a3, Bq = 2.0 * a2, Cq = su[D + ((lane < D) ? lane : 0)];
        double x0 = -1.0, x1 = -1.0;
        if (A != 0.0) {
          const double disc = Bq * Bq - 4.0 * A * Cq;
          if (disc >= 0.0) {
            const double sq = sqrt(disc);
            x0 = (-Bq - sq) / (2.0 * A);
            x1 = (-Bq + sq) / (2.0 * A);
          }
        } else if (Bq != 0.0) {
          x0 = -Cq / Bq;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
          q0[i] = __shfl_sync(FULL, x0, i);
          q1[i] = __shfl_sync(FULL, x1, i);
        }
      }
#else
      cubic_stationary<D>(su, t2, t3, q0, q1);
#endif
    }
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < D; ++j) { ec[j] = t2[j]; ec[D + j] = t3[j]; ec[2 * D + j] = q0[j]; ec[3 * D + j] = q1[j]; }
    }
    __syncwarp();
  }
  const double* c2 = ec;
  const double* c3 = ec + D;
  const double* r0 = ec + 2 * D;
  const double* r1 = ec + 3 * D;
  const int hoff = P.hoff;
#define hu0 su[hoff]
#define hu1 su[hoff + 1]
#define hv0 sv[hoff]
#define hv1 sv[hoff + 1]
  const double R = P.max_range;
  const double m = R + kCullMargin;
  const double R2 = R * R;
  const double cos2 = P.fov_cos_half * P.fov_cos_half;
  constexpr int heur = HEUR;
  const unsigned lt = lanemask_lt();
  // bearing cull half angle: FOV half angle + 2e-3 rad margin (cos, sin),
  // computed once per block (k_edges)
  const float chf = (heur >= 2) ? L.arc[0] : 0.0f, shf = (heur >= 2) ? L.arc[1] : 0.0f;
  const float invT = 1.0f / (float)T;   // heading-arc parameters only (culling)
#if MPAP_CULL_EDGE && MPAP_CULL_TWOSTAGE && MPAP_CULL_FENV && !MPAP_FMASK_F32
  // Edge-level range candidates: features within R + 2e-3 of the bounding
  // box of all the edge's steps (float test).  Every chunk box lies inside
  // it up to rounding (~1e-14 m, and one float ulp ~2e-6 m after conversion),
  // so a feature passing a chunk's range test (margin R + 1e-3) is on this
  // list: the chunks' kept sets, in index order, are unchanged.
  int* elist = L.fidx;
  int ne = 0;
  {
    double elo[D], ehi[D];
    chunk_bbox_warp<D, DYN>(su, sv, c2, c3, r0, r1, T, 0.0, (double)(K - 1) * Dl, lane, elo, ehi);
    const float ax = (float)elo[0], bx = (float)ehi[0], ay = (float)elo[1], by = (float)ehi[1];
    const float az = (D == 3) ? (float)elo[D - 1] : 0.0f, bz = (D == 3) ? (float)ehi[D - 1] : 0.0f;
    const float me = (float)R + 2e-3f, me2 = me * me;
    __syncwarp();
    for (int f0 = 0; f0 < F; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      if (f < F) {
        const float4 fv = L.fenv[f];
        const float ex = fmaxf(fmaxf(ax - fv.x, fv.x - bx), 0.0f);
        const float ey = fmaxf(fmaxf(ay - fv.y, fv.y - by), 0.0f);
        const float ez = (D == 3) ? fmaxf(fmaxf(az - fv.z, fv.z - bz), 0.0f) : 0.0f;
        keep = ex * ex + ey * ey + ez * ez <= me2;
      }
      const unsigned msk = __ballot_sync(FULL, keep);
      if (keep) elist[ne + __popc(msk & lt)] = f;
      ne += __popc(msk);
    }
    __syncwarp();
  }
#endif
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int nk = min(32, K - k0);
    const double ta = (double)k0 * Dl, tb = (double)(k0 + nk - 1) * Dl;
    double lo[D], hi[D];
#if MPAP_BBOX_WARP
    chunk_bbox_warp<D, DYN>(su, sv, c2, c3, r0, r1, T, ta, tb, lane, lo, hi);
#else
    chunk_bbox<D, DYN>(su, sv, c2, c3, r0, r1, T, ta, tb, lo, hi);
#endif
    // Heading arc of the chunk (heading heuristics): the step headings lie on
    // the chord between the interpolated headings at the chunk's first and
    // last step, so their directions are within dev of the chord's mid
    // direction (ux, uy).  beta0 = half FOV + margin + dev; a feature whose
    // bearing from the chunk is beyond beta0 (+ the chunk's angular radius)
    // fails every step's FOV test.
    bool ang = false;
    float ux = 0.0f, uy = 0.0f, c1 = 0.0f, s1 = 0.0f, smax = -1.0f;
    if (heur >= 2) {
      const float sa = (float)ta * invT, sb = (float)tb * invT;
      const float hx0 = (float)hu0, hy0 = (float)hu1, gx = (float)hv0 - hx0, gy = (float)hv1 - hy0;
      const float ax = fmaf(sa, gx, hx0), ay = fmaf(sa, gy, hy0);
      const float bx = fmaf(sb, gx, hx0), by = fmaf(sb, gy, hy0);
      const float ex = bx - ax, ey = by - ay;
      const float ee = ex * ex + ey * ey;
      float tq = (ee > 0.0f) ? -div_cull(ax * ex + ay * ey, ee) : 0.0f;
      tq = fminf(fmaxf(tq, 0.0f), 1.0f);
      const float qx = ax + tq * ex, qy = ay + tq * ey;
      if (qx * qx + qy * qy > 1e-4f) {
        const float na = rsqrtf(ax * ax + ay * ay), nb2 = rsqrtf(bx * bx + by * by);
        const float dax = ax * na, day = ay * na, dbx = bx * nb2, dby = by * nb2;
        const float mx = dax + dbx, my = day + dby;
        const float mn = sqrt_cull(mx * mx + my * my);
        if (mn > 1e-2f) {
          ux = div_cull(mx, mn);
          uy = div_cull(my, mn);
          // |da + db| = 2 cos(dev), |da - db| = 2 sin(dev)
          const float cd = 0.5f * mn;
          const float sd = 0.5f * sqrt_cull((dax - dbx) * (dax - dbx) + (day - dby) * (day - dby));
          c1 = chf * cd - shf * sd;   // cos(beta0)
          s1 = shf * cd + chf * sd;   // sin(beta0)
          if (c1 > -0.99995f) {       // beta0 < pi - 0.01
            ang = true;
            // omega may reach pi - 0.01 - beta0: unbounded if that is >= pi / 2,
            // else sin(pi - 0.01 - beta0) = sin(beta0 + 0.01)
            smax = (c1 >= 0.0099998f) ? 2.0f : s1 * 0.99995f + c1 * 0.0099998f;
          }
        }
      }
    }
    // Conservative single-precision culls (only discard features whose exact
    // test provably fails; margins >> float rounding):
    //  * range: distance(feature, chunk box) > R + 1e-3;
    //  * bearing (heading heuristics): see the per-edge heading arc above.
    const float flx = (float)lo[0], fhx = (float)hi[0], fly = (float)lo[1], fhy = (float)hi[1];
    const float flz = (D == 3) ? (float)lo[D - 1] : 0.0f, fhz = (D == 3) ? (float)hi[D - 1] : 0.0f;
    const float ccx = 0.5f * (flx + fhx), ccy = 0.5f * (fly + fhy);
    const float rho = 0.5f * sqrt_cull((fhx - flx) * (fhx - flx) + (fhy - fly) * (fhy - fly)) + 1e-4f;
    const float rho2 = rho * rho;
    const float mf = (float)R + 1e-3f;
    const float mf2 = mf * mf;
    int nf = 0;
    __syncwarp();
#if MPAP_CULL_TWOSTAGE && MPAP_CULL_FENV
    {
      // stage 1: range only, survivors' indices compacted into the (not yet
      // used) occluder-mask array; stage 2: bearing over the survivors only,
      // every lane busy
      int* rsel = reinterpret_cast<int*>(L.fmask);
      int nr = 0;
#if MPAP_CULL_EDGE && !MPAP_FMASK_F32
      for (int i0 = 0; i0 < ne; i0 += 32) {
        const int f = (i0 + lane < ne) ? elist[i0 + lane] : 0;
        bool keep = false;
        if (i0 + lane < ne) {
#else
      for (int f0 = 0; f0 < F; f0 += 32) {
        const int f = f0 + lane;
        bool keep = false;
        if (f < F) {
#endif
          const float4 fv = L.fenv[f];
          const float ex = fmaxf(fmaxf(flx - fv.x, fv.x - fhx), 0.0f);
          const float ey = fmaxf(fmaxf(fly - fv.y, fv.y - fhy), 0.0f);
          const float ez = (D == 3) ? fmaxf(fmaxf(flz - fv.z, fv.z - fhz), 0.0f) : 0.0f;
          keep = ex * ex + ey * ey + ez * ez <= mf2;
        }
        const unsigned msk = __ballot_sync(FULL, keep);
        if (keep) rsel[nr + __popc(msk & lt)] = f;
        nr += __popc(msk);
      }
      __syncwarp();
      for (int i0 = 0; i0 < nr; i0 += 32) {
        const int i = i0 + lane;
        bool keep = false;
        int f = 0;
        if (i < nr) {
          f = rsel[i];
          keep = true;
          if (ang) {
            const float4 fv = L.fenv[f];
            const float dx = fv.x - ccx, dy = fv.y - ccy;
            const float dc2 = dx * dx + dy * dy;
            const float inv = rsqrtf(fmaxf(dc2, 1e-30f));
            const float sw = rho * inv;
            const float cw = sqrt_cull(1.0f - sw * sw);
            const float cosb = c1 * cw - s1 * sw;            // cos(beta0 + omega)
            const float dotv = (ux * dx + uy * dy) * inv;      // cos(angle to the centre direction)
            keep = !(dc2 > rho2 && sw < smax && dotv < cosb - 2e-4f);
          }
        }
        const unsigned msk = __ballot_sync(FULL, keep);
        if (keep) {
          const int pos = nf + __popc(msk & lt);
          {   // exact coordinates: (x, y) with one 16-byte store, z
            const double* fp = feat + (size_t)f * D;
            L.fxy[pos] = make_double2(__ldg(fp), __ldg(fp + 1));
            if (D == 3) L.f[D - 1][pos] = __ldg(fp + D - 1);
          }
        }
        nf += __popc(msk);
      }
      __syncwarp();
    }
#else
    for (int f0 = 0; f0 < F; f0 += 32) {
      const int f = f0 + lane;
      bool keep = false;
      if (f < F) {
#if MPAP_CULL_FENV
        const float4 fv = L.fenv[f];   // the environment's features, staged as float once per environment
        const float fx = fv.x, fy = fv.y, fz = fv.z;
#else
        const double* fp = feat + (size_t)f * D;
        const float fx = (float)__ldg(fp), fy = (float)__ldg(fp + 1), fz = (D == 3) ? (float)__ldg(fp + D - 1) : 0.0f;
#endif
        const float ex = fmaxf(fmaxf(flx - fx, fx - fhx), 0.0f);
        const float ey = fmaxf(fmaxf(fly - fy, fy - fhy), 0.0f);
        const float ez = (D == 3) ? fmaxf(fmaxf(flz - fz, fz - fhz), 0.0f) : 0.0f;
        keep = ex * ex + ey * ey + ez * ez <= mf2;
#if MPAP_CULL_BRANCHFREE
        {   // the same decision as the nested form below, without divergent branches
          const float dx = fx - ccx, dy = fy - ccy;
          const float dc2 = dx * dx + dy * dy;
          const float inv = rsqrtf(fmaxf(dc2, 1e-30f));
          const float sw = rho * inv;
          const float cw = sqrt_cull(1.0f - sw * sw);
          const float cosb = c1 * cw - s1 * sw;            // cos(beta0 + omega)
          const float dotv = (ux * dx + uy * dy) * inv;      // cos(angle to the centre direction)
          const bool out = ang && dc2 > rho2 && sw < smax && dotv < cosb - 2e-4f;
          keep = keep && !out;
        }
#else
        if (keep && ang) {
          const float dx = fx - ccx, dy = fy - ccy;
          const float dc2 = dx * dx + dy * dy;
          if (dc2 > rho2) {
            const float inv = rsqrtf(dc2);
            const float sw = rho * inv;
            if (sw < smax) {
              const float cw = sqrtf(fmaxf(1.0f - sw * sw, 0.0f));
              const float cosb = c1 * cw - s1 * sw;            // cos(beta0 + omega)
              const float dotv = (ux * dx + uy * dy) * inv;      // cos(angle to the centre direction)
              if (dotv < cosb - 2e-4f) keep = false;
            }
          }
        }
#endif
      }
      const unsigned msk = __ballot_sync(FULL, keep);
      if (keep) {
        const int pos = nf + __popc(msk & lt);
#pragma unroll
        for (int q = 0; q < D; ++q) FREF(L, q, pos) = __ldg(feat + (size_t)f * D + q);   // exact coordinates
        if (MPAP_CULL_FENV && MPAP_FMASK_F32) L.fidx[pos] = f;
      }
      nf += __popc(msk);
    }
#endif
    const int nb = (nf > 0) ? cull_boxes<D>(box, O, lo, hi, m, L.box, lane, MPAP_FMASK_F32 ? L.boxf : nullptr) : 0;
    W.add(lane, W_CULL_TESTS, F + (nf > 0 ? O : 0));
    // per kept feature: which of the chunk's boxes meet the box spanned by the
    // chunk and the feature (every sight line to it lies inside that box).
    // Lanes over boxes (lane j: boxes j and j + 32), one ballot per feature;
    // single precision with a 1e-4 m margin (>> the float rounding of
    // coordinates below 1e3 m): a superset of the exact overlaps.
    const bool use_mask = nb > 0 && nb <= 64;
#if MPAP_FMASK_F32 == 2
    if (use_mask) {   // one kept feature per lane, boxes in single precision (1e-4 m margin)
      constexpr float mg = 1e-4f;
      const float clo[3] = {flx, fly, flz}, chi[3] = {fhx, fhy, fhz};
      for (int i = lane; i < nf; i += 32) {
        float fl[D], fh[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const float fq = (float)FREF(L, q, i);
          fl[q] = fminf(clo[q], fq) - mg;
          fh[q] = fmaxf(chi[q], fq) + mg;
        }
        unsigned long long msk = 0ull;
        for (int bb = 0; bb < nb; ++bb) {
          const float* bx = L.boxf + (size_t)bb * 2 * D;
          bool sep = false;
#pragma unroll
          for (int q = 0; q < D; ++q) sep |= bx[q] > fh[q] || bx[D + q] < fl[q];
          if (!sep) msk |= 1ull << bb;
        }
        L.fmask[i] = msk;
      }
      W.add(lane, W_CULL_TESTS, nf * nb);
      __syncwarp();
    }
#elif !MPAP_FMASK_F32
    if (use_mask && MPAP_FMASK_PAIRS && nf <= 16) {
      // few kept features: lanes over (feature, box) pairs -- feature i =
      // lane mod nfp, boxes sub, sub + g, ... (g = 32 / nfp lane groups); the
      // groups' partial masks are OR-ed with shuffles
      int nfp = 1;
      while (nfp < nf) nfp <<= 1;
      const int lg = __ffs(nfp) - 1;   // nfp is a power of two
      const int g = 32 >> lg, i = lane & (nfp - 1), sub = lane >> lg;
      unsigned long long msk = 0ull;
      if (i < nf) {
        double fl[D], fh[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const double fq = FREF(L, q, i);
          fl[q] = dmin(lo[q], fq) - kCullMargin;
          fh[q] = dmax(hi[q], fq) + kCullMargin;
        }
        for (int bb = sub; bb < nb; bb += g) {
          double bx[2 * D];
          load_box<D>(L.box + (size_t)bb * 2 * D, bx);
          bool sep = false;
#pragma unroll
          for (int q = 0; q < D; ++q)
            if (bx[q] > fh[q] || bx[D + q] < fl[q]) sep = true;
          if (!sep) msk |= 1ull << bb;
        }
      }
      for (int o = nfp; o < 32; o <<= 1) msk |= __shfl_xor_sync(FULL, msk, o);
      if (sub == 0 && i < nf) L.fmask[i] = msk;
      W.add(lane, W_CULL_TESTS, nf * nb);
      __syncwarp();
    } else if (use_mask) {
      for (int i = lane; i < nf; i += 32) {
        double fl[D], fh[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const double fq = FREF(L, q, i);
          fl[q] = dmin(lo[q], fq) - kCullMargin;
          fh[q] = dmax(hi[q], fq) + kCullMargin;
        }
        unsigned long long msk = 0ull;
        for (int bb = 0; bb < nb; ++bb) {
          double bx[2 * D];
          load_box<D>(L.box + (size_t)bb * 2 * D, bx);
          bool sep = false;
#pragma unroll
          for (int q = 0; q < D; ++q)
            if (bx[q] > fh[q] || bx[D + q] < fl[q]) sep = true;
          if (!sep) msk |= 1ull << bb;
        }
        L.fmask[i] = msk;
      }
      W.add(lane, W_CULL_TESTS, nf * nb);
      __syncwarp();
    }
#else
    if (use_mask) {
      constexpr float mg = 1e-4f;
      const bool h0 = lane < nb, h1 = lane + 32 < nb;
      float b0[2 * D], b1[2 * D];
#pragma unroll
      for (int k = 0; k < 2 * D; ++k) {
        b0[k] = h0 ? L.boxf[(size_t)lane * 2 * D + k] : 0.0f;
        b1[k] = h1 ? L.boxf[(size_t)(lane + 32) * 2 * D + k] : 0.0f;
      }
      const float clo[3] = {flx, fly, flz}, chi[3] = {fhx, fhy, fhz};
      for (int i = 0; i < nf; ++i) {
#if MPAP_CULL_FENV
        const float4 fk = L.fenv[L.fidx[i]];
#else
        const float4 fk = make_float4((float)FREF(L, 0, i), (float)FREF(L, 1, i), (D == 3) ? (float)FREF(L, D - 1, i) : 0.0f, 0.0f);
#endif
        const float fq[3] = {fk.x, fk.y, fk.z};
        bool s0 = !h0, s1 = !h1;
#pragma unroll
        for (int q = 0; q < D; ++q) {
          const float fl = fminf(clo[q], fq[q]) - mg;
          const float fh = fmaxf(chi[q], fq[q]) + mg;
          s0 |= b0[q] > fh || b0[D + q] < fl;
          s1 |= b1[q] > fh || b1[D + q] < fl;
        }
        const unsigned m0 = __ballot_sync(FULL, !s0), m1 = __ballot_sync(FULL, !s1);
        if (lane == 0) L.fmask[i] = (unsigned long long)m0 | ((unsigned long long)m1 << 32);
      }
      W.add(lane, W_CULL_TESTS, nf * nb);
      __syncwarp();
    }
#endif
    W.add(lane, W_STEPS, nk);
    W.add(lane, W_RANGE_TESTS, nk * nf);
    if (heur != 0) W.add(lane, W_FOV_TESTS, nk * nf);
    if (heur == 3) W.add(lane, W_MLP, nk);
    const int k = k0 + lane;
    if (k < K) {
      const double t = (double)k * Dl;
      double x[D], hv[D];
#pragma unroll
      for (int j = 0; j < D; ++j) hv[j] = 0.0;
      if (DYN == 0) {
        const double sp = t / T;
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = fma(sp, sv[j] - su[j], su[j]);
        if (heur == 1) {
#pragma unroll
          for (int j = 0; j < D; ++j) hv[j] = sv[j] - su[j];
        }
      } else {
        di_pos<D>(su, c2, c3, t, x);
        if (heur == 1) di_vel<D>(su, c2, c3, t, hv);
      }
      if (heur >= 2) {
        const double sp = t / T;
        hv[0] = fma(sp, hv0, (1.0 - sp) * hu0);
        hv[1] = fma(sp, hv1, (1.0 - sp) * hu1);
      }
      // heading heuristics: hv is horizontal (hv_z = 0), so the z terms of hh
      // and of the FOV dot product add exact zeros -- skipped (a zero's sign
      // can differ, which no comparison below sees)
      constexpr int DH = (HEUR >= 2) ? 2 : D;
      double hh = 0.0;
#pragma unroll
      for (int j = 0; j < DH; ++j) hh = fma(hv[j], hv[j], hh);
      int kv = 0;
      for (int i = 0; i < nf; ++i) {
        double dl[D];
        double dd = 0.0;
        double fc[D];
        {
          const double2 xy = L.fxy[i];   // one 16-byte load for (x, y)
          fc[0] = xy.x;
          fc[1] = xy.y;
          if (D == 3) fc[D - 1] = L.f[D - 1][i];
        }
#pragma unroll
        for (int j = 0; j < D; ++j) { dl[j] = fc[j] - x[j]; dd = fma(dl[j], dl[j], dd); }
        if (dd > R2) continue;
        if (heur != 0) {
          double dot = 0.0;
#pragma unroll
          for (int j = 0; j < DH; ++j) dot = fma(hv[j], dl[j], dot);
          if (!(hh > 0.0)) continue;
          if (dot < 0.0) continue;
          if (dot * dot < cos2 * (hh * dd)) continue;
        }
        ++W.occl_segs;
        const unsigned long long fm = use_mask ? L.fmask[i] : ~0ull;
        if (fm == 0ull) {   // no box meets the chunk-feature box: unobstructed (warp-uniform)
          ++kv;
          continue;
        }
        double fp[D];
#pragma unroll
        for (int j = 0; j < D; ++j) fp[j] = fc[j];
        const unsigned rr = use_mask ? seg_hits_boxes<D, true>(x, fp, dl, L.box, nb, fm)
                                     : seg_hits_boxes<D, false>(x, fp, dl, L.box, nb, 0ull);
        W.occl_tests += rr >> 1;
        if (!(rr & 1u)) ++kv;
      }
      kv_out[k] = (uint16_t)kv;
    }
    __syncwarp();
  }
#undef hu0
#undef hu1
#undef hv0
#undef hv1
}

// Persistent: each warp pulls work items from an atomic counter, so no block
// waits on its slowest item.  Build mode (items == nullptr): item = one row
// (over all environments of the batch), its r-disc entries from the
// neighbour scratch.  Update mode (NEXT-1, mpap_roadmap_update): item = one
// edge {row, global edge index} of the affected list; its dst, w and tau come
// from the roadmap itself.  PHASE 0 computes the collision bit and writes the
// edge record; PHASE 1 fills the heuristic summary (s, c) (and peaks) of the
// collision-free ones.  Two kernels keep each one's code and register
// footprint small.
template <int PHASE>
struct EdgeBounds { static constexpr int kMin = (PHASE == 0) ? 2 : MPAP_EDGES_MIN_BLOCKS; };

template <int D, int DYN, int PHASE, int HEUR>
__global__ void __launch_bounds__(kWarps * 32, EdgeBounds<PHASE>::kMin) k_edges(const double* __restrict__ samples,
                                                          const int64_t* __restrict__ node_base, int B,
                                                          const double* __restrict__ obst,
                                                          const int32_t* __restrict__ obst_base,
                                                          const double* __restrict__ feat,
                                                          const int32_t* __restrict__ feat_base, DevParams P,
                                                          int cap, int o_max, int f_max,
                                                          const NearRec* __restrict__ scratch,
                                                          const int64_t* __restrict__ row_ptr,
                                                          EdgeRec* __restrict__ edges,
                                                          double* __restrict__ tau_arr,
                                                          int32_t* __restrict__ esrc,
                                                          long long* __restrict__ koff,
                                                          uint16_t* __restrict__ kvbuf,
                                                          unsigned long long* __restrict__ kv_total,
                                                          longlong2* __restrict__ flist,
                                                          unsigned long long* __restrict__ fcount,
                                                          float2* __restrict__ peak,
                                                          const longlong2* __restrict__ items, int64_t n_items,
                                                          unsigned long long* __restrict__ nnz_free,
                                                          unsigned long long* __restrict__ work,
                                                          unsigned long long* __restrict__ next_item) {
  constexpr int NS = 2 * D + 2;   // p, v (double integrator), heading
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_state[kWarps][2][NS];
  __shared__ unsigned s_work[kWarps][W_NUM];
  __shared__ double s_ec[kWarps][12];
  __shared__ float s_arc[2];
  if (threadIdx.x == 0) {
    const float hf = acosf((float)P.fov_cos_half) + 2e-3f;
    s_arc[0] = cosf(hf);
    s_arc[1] = sinf(hf);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpLists<D> L;
  {
    const size_t fs = round4(f_max), os = round4(o_max);
    // PHASE 0 (collision) stages only the culled boxes: its own, smaller
    // per-warp slice (more of the SM's L1 stays cache)
    double* base = smem + (size_t)warp * (PHASE == 0 ? os * 2 * D : warp_scratch_doubles(D, fs, os));
    L.fxy = reinterpret_cast<double2*>(base);   // (x, y) pairs
    L.f[0] = base;                               // (x, y) strided: accessed through FREF
    L.f[1] = base + 1;
    if (D == 3) L.f[D - 1] = base + 2 * fs;      // z
    L.box = (PHASE == 0) ? base : base + (size_t)D * fs;
    L.fmask = reinterpret_cast<unsigned long long*>(L.box + os * 2 * D);
    double* nxt = reinterpret_cast<double*>(L.fmask + fs);
    L.fenv = reinterpret_cast<float4*>(nxt);
    if (MPAP_CULL_FENV) nxt += fs * 2;
    L.boxf = reinterpret_cast<float*>(nxt);
    if (MPAP_FMASK_F32) nxt += os * D;
    L.fidx = reinterpret_cast<int*>(nxt);
    L.arc = s_arc;
  }
  int staged_env = -1;   // environment whose features L.fenv holds (PHASE 1)
  const int64_t NI = items ? n_items : node_base[B];
  const int stride = P.stride;
  Work W;
  W.sm = s_work[warp];
  W.occl_segs = W.occl_tests = W.coll_segs = W.coll_tests = 0;
  if (lane < W_NUM) W.sm[lane] = 0;
  double* su = s_state[warp][0];
  double* sv = s_state[warp][1];
  __syncwarp();
  for (;;) {
    unsigned long long rr = 0;
    if (lane == 0) rr = atomicAdd(next_item, 1ull);
    const int64_t idx = (int64_t)__shfl_sync(FULL, rr, 0);
    if (idx >= NI) break;
    int64_t row, e_begin, e_end;
    if (items) {
      const longlong2 it = items[idx];
      row = it.x;
      e_begin = it.y;
      e_end = it.y + 1;
    } else {
      row = idx;
      e_begin = row_ptr[row];
      e_end = row_ptr[row + 1];
    }
    int lo_b = 0, hi_b = B;   // env = last b with node_base[b] <= row
    while (hi_b - lo_b > 1) {
      const int mid = (lo_b + hi_b) >> 1;
      if (node_base[mid] <= row) lo_b = mid; else hi_b = mid;
    }
    const int b = lo_b;
    const int64_t u = row - node_base[b];
    const int O = obst_base[b + 1] - obst_base[b];
    const int F = feat_base[b + 1] - feat_base[b];
    const double* ebox = obst + (size_t)obst_base[b] * 2 * D;
    const double* efeat = feat + (size_t)feat_base[b] * D;
    const double* envs = samples + node_base[b] * stride;
    if (MPAP_CULL_FENV && PHASE == 1 && b != staged_env) {   // stage the environment's features as float
      __syncwarp();
      for (int i = lane; i < F; i += 32) {
        const double* fp = efeat + (size_t)i * D;
        L.fenv[i] = make_float4((float)__ldg(fp), (float)__ldg(fp + 1), (D == 3) ? (float)__ldg(fp + D - 1) : 0.0f,
                                0.0f);
      }
      staged_env = b;
    }
    __syncwarp();
    if (lane < NS) su[lane] = (lane < stride) ? envs[u * stride + lane] : 0.0;
    int nfree = 0;
    long long kv_local = 0;   // PHASE 0: kv slots of the row's free edges (multiples of 8)
    for (int64_t e = e_begin; e < e_end; ++e) {
      if constexpr (PHASE == 0) {
        int v;
        float w;
        double tau;
        int old_coll = 0;
        if (items) {
          const EdgeRec old = edges[e];
          v = (int)(old.dst_coll & 0x7fffffffu);
          old_coll = (int)(old.dst_coll >> 31);
          w = old.w;
          tau = tau_arr[e];
        } else {
          const NearRec rec = scratch[row * (int64_t)cap + (e - e_begin)];
          v = rec.v;
          w = rec.w;
          tau = rec.tau;
        }
        __syncwarp();
        if (lane < NS) sv[lane] = (lane < stride) ? envs[(int64_t)v * stride + lane] : 0.0;
        __syncwarp();
        const bool coll = edge_collision<D, DYN>(P, su, sv, tau, ebox, O, L, lane, W);
        nfree += items ? (old_coll - (coll ? 1 : 0)) : (coll ? 0 : 1);
        W.flush(lane);
        if (lane == 0) {
          EdgeRec er;
          er.dst_coll = (uint32_t)v | (coll ? 0x80000000u : 0u);
          er.w = w;
          er.s = 0.0f;
          er.c = 0.0f;
          edges[e] = er;
          if (!items) {
            tau_arr[e] = tau;
            esrc[e] = (int32_t)row;
          }
          if (peak) peak[e] = make_float2(0.0f, 0.0f);
          if (!coll) {   // kv slots for k_heuristic / k_fold: K steps rounded up to 8
            const double kk = ceil(tau / P.dt);
            const long long K8 = (((kk < 1.0) ? 1 : (long long)kk) + 7) & ~7ll;
            if (items) {
              koff[e] = (long long)atomicAdd(kv_total, (unsigned long long)K8);
            } else {
              koff[e] = kv_local;
              kv_local += K8;
            }
          }
        }
      } else {
        const uint32_t dc = edges[e].dst_coll;
        if (dc >> 31) continue;   // colliding edges keep s = c = 0 (never relaxed)
        const double tau = tau_arr[e];
        __syncwarp();
        if (lane < NS) sv[lane] = (lane < stride) ? envs[(int64_t)(dc & 0x7fffffffu) * stride + lane] : 0.0;
        __syncwarp();
        edge_visible<D, DYN, HEUR>(P, su, sv, tau, efeat, F, ebox, O, L, s_ec[warp], lane, kvbuf + koff[e], W);
        W.flush(lane);
      }
    }
    if (PHASE == 0) {
      if (!items) {   // one atomic per row, then rebase the row's offsets
        long long base = 0;
        if (lane == 0 && kv_local) base = (long long)atomicAdd(kv_total, (unsigned long long)kv_local);
        base = __shfl_sync(FULL, base, 0);
        kv_local = __shfl_sync(FULL, kv_local, 0);
        __syncwarp();   // lane 0's koff / edge stores are visible to the warp
        // the row's free edges, in order, into the free list (k_fold's work)
        unsigned long long fbase = 0;
        if (lane == 0 && nfree) fbase = atomicAdd(fcount, (unsigned long long)nfree);
        fbase = __shfl_sync(FULL, fbase, 0);
        int fr = 0;
        for (int64_t e0 = e_begin; e0 < e_end; e0 += 32) {
          const int64_t e = e0 + lane;
          const bool fe = (e < e_end) && !(edges[e].dst_coll >> 31);
          if (fe) koff[e] += base;
          const unsigned fm = __ballot_sync(FULL, fe);
          if (fe) flist[fbase + fr + __popc(fm & lanemask_lt())] = make_longlong2(row, e);
          fr += __popc(fm);
        }
      }
      W.add(lane, W_EDGES, (unsigned)(e_end - e_begin));
      if (!items) W.add(lane, W_FREE_EDGES, nfree);
      if (lane == 0 && nfree) atomicAdd(&nnz_free[b], (unsigned long long)(long long)nfree);
    }
  }
  __syncwarp();
  if (lane >= W_EDGES && lane < W_NUM && W.sm[lane]) atomicAdd(&work[lane], (unsigned long long)W.sm[lane]);
}


// Increments and ordered fold (reading R10) of every collision-free edge, one
// thread per edge, from the per-step visible counts k_v written by
// k_heuristic: inc_k = Dl - k_v (Dl / n_f), plus Dl * gamma * o_k
// for the learned heuristic (o_k = MLP(|v(t_k)| / v_ref, omega / w_ref,
// k_v / n_f), reading R12); then c <- max(0, c + inc_k), s <- s + inc_k in
// step order (and the running maxima S, C of NEXT-3).  The same operations in
// the same order as the per-step definition.
constexpr int kFoldThreads = 256;

template <int D, int DYN, int HEUR>
__global__ void __launch_bounds__(kFoldThreads, MPAP_FOLD_MIN_BLOCKS) k_fold(const double* __restrict__ samples,
                                                      const int64_t* __restrict__ node_base, int B,
                                                      const __grid_constant__ DevParams P,
                                                      const int32_t* __restrict__ esrc,
                                                      const double* __restrict__ tau_arr,
                                                      const long long* __restrict__ koff,
                                                      const uint16_t* __restrict__ kvbuf,
                                                      EdgeRec* __restrict__ edges, float2* __restrict__ peak,
                                                      const longlong2* __restrict__ items, int64_t n) {
  // MLP input k_v / n_f for the small counts, each entry the same correctly
  // rounded division the step would do (a lookup instead of a DDIV per step)
  constexpr int kZ2 = 256;
  __shared__ double s_z2[kZ2];
#if MPAP_FOLD_SMEM_TRAJ
  // the thread's velocity polynomial v(t) = v0 + t (2 c2 + t 3 c3) per axis,
  // kept in shared memory (its registers go to the two MLP evaluations)
  __shared__ double s_tr[(HEUR == 3 && DYN == 1) ? 3 * D : 1][kFoldThreads];
#endif
  if (HEUR == 3) {
    for (int i = threadIdx.x; i < kZ2; i += blockDim.x) s_z2[i] = (double)i / P.n_f;
  }
  __syncthreads();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int64_t e = items ? items[idx].y : idx;
  const uint32_t dc = edges[e].dst_coll;
  if (dc >> 31) return;   // colliding: s = c = 0
  const int64_t row = esrc[e];
  int lo_b = 0, hi_b = B;   // env = last b with node_base[b] <= row
  while (hi_b - lo_b > 1) {
    const int mid = (lo_b + hi_b) >> 1;
    if (node_base[mid] <= row) lo_b = mid; else hi_b = mid;
  }
  const int stride = P.stride;
  const double* envs = samples + node_base[lo_b] * stride;
  const double* su = envs + (row - node_base[lo_b]) * stride;
  const double* sv = envs + (int64_t)(dc & 0x7fffffffu) * stride;
  const double T = tau_arr[e];
  const double kk = ceil(T / P.dt);
  const int K = (kk < 1.0) ? 1 : (int)kk;
  const double Dl = T / (double)K;
  double omega = 0.0;
  double su_l[2 * D], sv_l[2 * D];
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) {
    su_l[j] = (DYN == 1 || j < D) ? su[j] : 0.0;
    sv_l[j] = (DYN == 1 || j < D) ? sv[j] : 0.0;
  }
  if (HEUR == 3 && P.has_heading) {
    const double ex = sv[P.hoff] - su[P.hoff], ey = sv[P.hoff + 1] - su[P.hoff + 1];
    omega = sqrt(ex * ex + ey * ey) / T;
  }
  double c2[D], c3[D];
#pragma unroll
  for (int j = 0; j < D; ++j) { c2[j] = 0.0; c3[j] = 0.0; }
  if (HEUR == 3 && DYN == 1) di_traj<D>(su_l, sv_l, T, c2, c3);
#if MPAP_FOLD_SMEM_TRAJ
  if (HEUR == 3 && DYN == 1) {
#pragma unroll
    for (int j = 0; j < D; ++j) {   // the factors di_vel forms per call (the same products)
      s_tr[j][threadIdx.x] = 3.0 * c3[j];
      s_tr[D + j][threadIdx.x] = 2.0 * c2[j];
      s_tr[2 * D + j][threadIdx.x] = su_l[D + j];
    }
  }
#endif
  const bool unit_vref = P.v_ref == 1.0;
  const double z1 = omega / P.w_ref;   // per-edge MLP input (one division per edge)
  const uint16_t* kvp = kvbuf + koff[e];
  const double q = Dl / P.n_f;
  double s = 0.0, c = 0.0, Sp = 0.0, Cp = 0.0;
  // the edge's counts are 8-aligned: one 16-byte load per 8 steps; the MLP
  // runs two steps per call (mlp_out0_x2), the fold stays in step order
  for (int k0 = 0; k0 < K; k0 += 8) {
    const uint4 q8 = __ldg(reinterpret_cast<const uint4*>(kvp + k0));
#pragma unroll 1
    for (int jp = 0; jp < 8; jp += 2) {   // not unrolled: one inlined copy of the MLP
      const unsigned wvp = (jp < 4) ? ((jp < 2) ? q8.x : q8.y) : ((jp < 6) ? q8.z : q8.w);   // steps jp, jp + 1
      if (k0 + jp >= K) break;
      double inc2[2];
      int kv2[2];
      double z0[2] = {0.0, 0.0};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + jp + u;
        kv2[u] = (int)((wvp >> (16 * u)) & 0xffffu);
        inc2[u] = Dl - (double)kv2[u] * q;
        if (HEUR == 3) {
          double speed = P.nominal_speed;   // |v(t)| for the MLP (kinematic: nominal)
          if (DYN == 1) {
            const double t = (double)k * Dl;
            double vel[D];
#if MPAP_FOLD_SMEM_TRAJ
#pragma unroll
            for (int j = 0; j < D; ++j)   // = di_vel: fma(t, fma(t, 3 c3, 2 c2), v0)
              vel[j] = fma(t, fma(t, s_tr[j][threadIdx.x], s_tr[D + j][threadIdx.x]), s_tr[2 * D + j][threadIdx.x]);
#else
            di_vel<D>(su_l, c2, c3, t, vel);
#endif
            double ss = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) ss = fma(vel[j], vel[j], ss);
            speed = sqrt(ss);
          }
          z0[u] = unit_vref ? speed : speed / P.v_ref;   // x / 1.0 == x exactly (IEEE)
        }
      }
      if (HEUR == 3) {
        const double za = kv2[0] < kZ2 ? s_z2[kv2[0]] : (double)kv2[0] / P.n_f;
        const double zb = kv2[1] < kZ2 ? s_z2[kv2[1]] : (double)kv2[1] / P.n_f;
        const double2 o = mlp_out0_x2(P.mlp, z0[0], z0[1], z1, za, zb);
        inc2[0] = inc2[0] + Dl * (P.mlp_gain * o.x);
        inc2[1] = inc2[1] + Dl * (P.mlp_gain * o.y);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (k0 + jp + u >= K) break;
        const double inc = inc2[u];
        const double tt = c + inc;
        c = (tt > 0.0) ? tt : 0.0;
        s = s + inc;
        Sp = (s > Sp) ? s : Sp;   // running maxima of the prefix values (NEXT-3)
        Cp = (c > Cp) ? c : Cp;
      }
    }
  }
  *reinterpret_cast<float2*>(&edges[e].s) = make_float2((float)s, (float)c);
  if (peak) peak[e] = make_float2((float)Sp, (float)Cp);
}

// NEXT-1: edges of one environment whose collision bit or
// heuristic summary can change when the boxes `cbox` [nb][2D] and features
// `cfeat` [nf][D] (the symmetric differences of the old and new sets) change.
// Warp per row, lane per edge.  With E = the edge trajectory's bounding box
// over [0, tau] (every step point and collision-polyline vertex lies in it,
// up to rounding far below the margins):
//  * a changed feature matters only if it is within R + 1e-3 of E per axis
//    (else it is out of range of every step point);
//  * a changed box matters only if it overlaps, grown by 1e-3, the bounding
//    box V of E and of every feature (current or changed) within R + 1e-3 of
//    E: every polyline segment lies in E and every sight line from a step
//    point to an in-range feature lies in V.
// So an unlisted edge's collision bit and heuristic summary are provably
// unchanged.
template <int D, int DYN>
__global__ void __launch_bounds__(kWarps * 32) k_affected(const double* __restrict__ env_samples, int stride,
                                                            int64_t row0, int64_t n_rows,
                                                            const int64_t* __restrict__ row_ptr,
                                                            const EdgeRec* __restrict__ edges,
                                                            const double* __restrict__ tau_arr, double R,
                                                            const double* __restrict__ efeat, int F,
                                                            const double* __restrict__ cbox, int nb,
                                                            const double* __restrict__ cfeat, int nf,
                                                            longlong2* __restrict__ items,
                                                            unsigned long long* __restrict__ n_items) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (r >= n_rows) return;
  const int64_t row = row0 + r;   // global row (row_ptr); r and dst are env-local node ids
  const unsigned lt = lanemask_lt();
  const double m = R + 1e-3;
  double su[2 * D];
#pragma unroll
  for (int j = 0; j < 2 * D; ++j) su[j] = (DYN == 1 || j < D) ? env_samples[r * stride + j] : 0.0;
  const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
  for (int64_t eb = e0; eb < e1; eb += 32) {
    const int64_t e = eb + lane;
    bool hit = false;
    if (e < e1) {
      const int v = (int)(edges[e].dst_coll & 0x7fffffffu);
      const double tau = tau_arr[e];
      double sv[2 * D];
      const double* vrow = env_samples + (int64_t)v * stride;
#pragma unroll
      for (int j = 0; j < 2 * D; ++j) sv[j] = (DYN == 1 || j < D) ? vrow[j] : 0.0;
      double c2[D], c3[D], r0[D], r1[D], lo[D], hi[D];
#pragma unroll
      for (int j = 0; j < D; ++j) { c2[j] = 0.0; c3[j] = 0.0; r0[j] = -1.0; r1[j] = -1.0; }
      if (DYN == 1) {
        di_traj<D>(su, sv, tau, c2, c3);
        cubic_stationary<D>(su, c2, c3, r0, r1);
      }
      chunk_bbox<D, DYN>(su, sv, c2, c3, r0, r1, tau, 0.0, tau, lo, hi);
      for (int i = 0; i < nf && !hit; ++i) {
        bool sep = false;
#pragma unroll
        for (int k = 0; k < D; ++k)
          if (cfeat[i * D + k] > hi[k] + m || cfeat[i * D + k] < lo[k] - m) sep = true;
        hit = !sep;
      }
      if (!hit && nb > 0) {
        double vlo[D], vhi[D];
#pragma unroll
        for (int k = 0; k < D; ++k) { vlo[k] = lo[k]; vhi[k] = hi[k]; }
        for (int pass = 0; pass < 2; ++pass) {
          const double* fl = pass ? cfeat : efeat;
          const int nfl = pass ? nf : F;
          for (int i = 0; i < nfl; ++i) {
            double fc[D];
            bool near = true;
#pragma unroll
            for (int k = 0; k < D; ++k) {
              fc[k] = fl[(size_t)i * D + k];
              if (fc[k] > hi[k] + m || fc[k] < lo[k] - m) near = false;
            }
            if (near) {
#pragma unroll
              for (int k = 0; k < D; ++k) { vlo[k] = dmin(vlo[k], fc[k]); vhi[k] = dmax(vhi[k], fc[k]); }
            }
          }
        }
        for (int i = 0; i < nb && !hit; ++i) {
          bool sep = false;
#pragma unroll
          for (int k = 0; k < D; ++k)
            if (cbox[i * 2 * D + k] > vhi[k] + 1e-3 || cbox[i * 2 * D + D + k] < vlo[k] - 1e-3) sep = true;
          hit = !sep;
        }
      }
    }
    const unsigned msk = __ballot_sync(FULL, hit);
    if (msk) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(n_items, (unsigned long long)__popc(msk));
      base = __shfl_sync(FULL, base, 0);
      if (hit) items[base + __popc(msk & lt)] = make_longlong2(row, e);
    }
  }
}

// ---------------------------------------------------------------------------
// host driver
// ---------------------------------------------------------------------------
#define CK(x)                                          \
  do {                                                 \
    cudaError_t _e = (x);                              \
    if (_e != cudaSuccess) return cuda_error(_e, #x);  \
  } while (0)

// SM count of the current device (grid sizes: multiples of it)
int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 1;
}

// exclusive scan of int32 row counts -> int64 row offsets (k_scan), for the
// other translation units (device-side row-block assembly)
cudaError_t scan_row_counts(const int32_t* cnt, int64_t n, int64_t* row_ptr, cudaStream_t st) {
  k_scan<<<1, 1024, 0, st>>>(cnt, n, row_ptr);
  note_launch();
  return cudaGetLastError();
}

namespace {
template <int D, int DYN>
cudaError_t launch_near(dim3 grid, cudaStream_t st, const mpap_roadmap* rm, const int32_t* d_n, int cap,
                        int32_t* d_cnt, NearRec* d_scr, int* d_over, unsigned long long* d_work) {
  k_near<D, DYN><<<grid, kNearWarps * 32, 0, st>>>(rm->d_samples, rm->d_node_base, d_n, rm->prm, cap, d_cnt, d_scr,
                                               d_over, d_work);
  return cudaGetLastError();
}

// NEXT-1 part i (lazy roadmap): the edge records of every row from the
// neighbour scratch -- dst and w (coll = 0, s = c = 0 until the row is
// evaluated), tau and the source row -- warp per row.
__global__ void k_lazy_init(const NearRec* __restrict__ scratch, int cap, const int64_t* __restrict__ row_ptr,
                            int64_t N, EdgeRec* __restrict__ edges, double* __restrict__ tau_arr,
                            int32_t* __restrict__ esrc, float2* __restrict__ peak) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < N;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const NearRec rec = scratch[row * (int64_t)cap + (e - e0)];
      EdgeRec er;
      er.dst_coll = (uint32_t)rec.v;
      er.w = rec.w;
      er.s = 0.0f;
      er.c = 0.0f;
      edges[e] = er;
      tau_arr[e] = rec.tau;
      esrc[e] = (int32_t)row;
      if (peak) peak[e] = make_float2(0.0f, 0.0f);
    }
  }
}

// Items {row, edge} of the requested rows (or of every row not yet ready),
// warp per row; marks the rows ready (the evaluation that follows is stream-
// ordered before any later search).
__global__ void k_row_items(const int32_t* __restrict__ rows, int64_t n_req, int64_t N,
                            const int64_t* __restrict__ row_ptr, int32_t* __restrict__ ready,
                            longlong2* __restrict__ items, unsigned long long* __restrict__ n_items) {
  const int lane = threadIdx.x & 31;
  const int64_t n = rows ? n_req : N;
  for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < n;
       k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = rows ? rows[k] : k;
    if (ready[row] == 1) continue;
    const int64_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
    unsigned long long base = 0;
    if (lane == 0 && e1 > e0) base = atomicAdd(n_items, (unsigned long long)(e1 - e0));
    base = __shfl_sync(FULL, base, 0);
    for (int64_t e = e0 + lane; e < e1; e += 32) items[base + (e - e0)] = make_longlong2(row, e);
    __syncwarp();
    if (lane == 0) ready[row] = 1;
  }
}

struct EdgeWork {            // what one k_edges launch processes
  const NearRec* scratch;    // build mode: neighbour scratch (cap entries per row)
  int cap;
  const longlong2* items;    // update mode: affected edges (else nullptr)
  int64_t n_items;
  unsigned long long* nnz_free;
  unsigned long long* work;
  unsigned long long* next;  // item counters (zeroed), one per phase
  long long* koff;           // per-edge offsets into kvbuf
  uint16_t* kvbuf;           // per-step visible counts (phase 1 output)
  unsigned long long* kv_total;
  longlong2* flist;          // build mode: free edges {row, edge} (k_fold's items)
  unsigned long long* fcount;
};

template <int D, int DYN, int PHASE, int HEUR>
cudaError_t launch_edges_phase(size_t smem, cudaStream_t st, const mpap_roadmap* rm, const EdgeWork& ew) {
  auto kern = k_edges<D, DYN, PHASE, HEUR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 1));
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarps * 32, smem);
  if (e != cudaSuccess) return e;
  const int64_t NI = ew.items ? ew.n_items : rm->node_base[rm->B];
  const int64_t need = (NI + kWarps - 1) / kWarps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(per_sm, 1), need));
  kern<<<grid, kWarps * 32, smem, st>>>(rm->d_samples, rm->d_node_base, rm->B, rm->d_obst, rm->d_obst_base,
                                        rm->d_feat, rm->d_feat_base, rm->prm, ew.cap, rm->o_max, rm->f_max,
                                        ew.scratch, rm->d_row_ptr, rm->d_edges, rm->d_tau, rm->d_esrc, ew.koff,
                                        ew.kvbuf, ew.kv_total, ew.flist, ew.fcount, rm->d_peak, ew.items,
                                        ew.n_items, ew.nnz_free, ew.work, ew.next);
  return cudaGetLastError();
}

template <int D, int DYN>
cudaError_t launch_edges(int phase, size_t smem, cudaStream_t st, const mpap_roadmap* rm, EdgeWork ew) {
  if (phase == 0) return launch_edges_phase<D, DYN, 0, 0>(smem, st, rm, ew);
  ew.next += 1;
  switch (rm->prm.heuristic) {
    case 0: return launch_edges_phase<D, DYN, 1, 0>(smem, st, rm, ew);
    case 1: return launch_edges_phase<D, DYN, 1, 1>(smem, st, rm, ew);
    case 2: return launch_edges_phase<D, DYN, 1, 2>(smem, st, rm, ew);
    default: return launch_edges_phase<D, DYN, 1, 3>(smem, st, rm, ew);
  }
}

cudaError_t launch_edges_any(int phase, size_t smem, cudaStream_t st, const mpap_roadmap* rm, const EdgeWork& ew) {
  const int d = rm->prm.pos_dim, dyn = rm->prm.dynamics;
  if (d == 2) return dyn ? launch_edges<2, 1>(phase, smem, st, rm, ew) : launch_edges<2, 0>(phase, smem, st, rm, ew);
  return dyn ? launch_edges<3, 1>(phase, smem, st, rm, ew) : launch_edges<3, 0>(phase, smem, st, rm, ew);
}

template <int D, int DYN>
cudaError_t launch_fold_dd(cudaStream_t st, const mpap_roadmap* rm, const EdgeWork& ew) {
  const int64_t n = ew.items ? ew.n_items : rm->nnz_total;
  if (n == 0) return cudaSuccess;
  const dim3 grid((unsigned)((n + kFoldThreads - 1) / kFoldThreads));
#define MPAP_FOLD_ARGS rm->d_samples, rm->d_node_base, rm->B, rm->prm, rm->d_esrc, rm->d_tau, ew.koff, ew.kvbuf, \
    rm->d_edges, rm->d_peak, ew.items, n
  switch (rm->prm.heuristic) {
    case 3: k_fold<D, DYN, 3><<<grid, kFoldThreads, 0, st>>>(MPAP_FOLD_ARGS); break;
    default: k_fold<D, DYN, 0><<<grid, kFoldThreads, 0, st>>>(MPAP_FOLD_ARGS); break;
  }
#undef MPAP_FOLD_ARGS
  return cudaGetLastError();
}

cudaError_t launch_fold(cudaStream_t st, const mpap_roadmap* rm, const EdgeWork& ew) {
  const int d = rm->prm.pos_dim, dyn = rm->prm.dynamics;
  if (d == 2) return dyn ? launch_fold_dd<2, 1>(st, rm, ew) : launch_fold_dd<2, 0>(st, rm, ew);
  return dyn ? launch_fold_dd<3, 1>(st, rm, ew) : launch_fold_dd<3, 0>(st, rm, ew);
}

size_t edges_smem(const mpap_roadmap* rm);

// collide (+ kv slot offsets) -> size the kv buffer -> visible counts -> fold
cudaError_t edge_phases(size_t smem, cudaStream_t st, const mpap_roadmap* rm, EdgeWork ew) {
  {
    ProfScope ps("k_collide", st);
    const size_t smem0 = sizeof(double) * (size_t)kWarps * round4(rm->o_max) * 2 * rm->prm.pos_dim;
    cudaError_t e = launch_edges_any(0, smem0, st, rm, ew);
    if (e != cudaSuccess) return e;
  }
  note_launch();
  unsigned long long total = 0, nfree = 0;
  cudaError_t e = cudaMemcpyAsync(&total, ew.kv_total, sizeof(total), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && !ew.items) e = cudaMemcpyAsync(&nfree, ew.fcount, sizeof(nfree), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  ew.kvbuf = static_cast<uint16_t*>(workspace(st, WS_KV, sizeof(uint16_t) * std::max<unsigned long long>(total, 8)));
  if (!ew.kvbuf) return cudaErrorMemoryAllocation;
  {
    ProfScope ps("k_heuristic", st);
    e = launch_edges_any(1, smem, st, rm, ew);
    if (e != cudaSuccess) return e;
  }
  note_launch();
  {
    ProfScope ps("k_fold", st);
    EdgeWork fw = ew;
    if (!ew.items) {   // build: the free-edge list written by k_collide
      fw.items = ew.flist;
      fw.n_items = (int64_t)nfree;
    }
    e = launch_fold(st, rm, fw);
    if (e != cudaSuccess) return e;
  }
  note_launch();
  return cudaSuccess;
}

size_t edges_smem(const mpap_roadmap* rm) {
  return sizeof(double) * (size_t)kWarps * warp_scratch_doubles(rm->prm.pos_dim, round4(rm->f_max), round4(rm->o_max));
}
}  // namespace

mpap_status build_roadmap_device(mpap_roadmap* rm, cudaStream_t st) {
  HostTimer total("build_roadmap_device total");
  const int B = rm->B;
  const int64_t N = rm->node_base[B];
  const int d = rm->prm.pos_dim;
  const int dyn = rm->prm.dynamics;
  int32_t* d_n = nullptr;
  int32_t* d_cnt = nullptr;
  int* d_over = nullptr;
  NearRec* d_scr = nullptr;
  unsigned long long* d_free = nullptr;
  unsigned long long* d_work = nullptr;
  static_assert(W_NUM <= kWorkCounters, "work counter array too small");
  int cap = 128;
  CK(cudaMallocAsync(&d_n, sizeof(int32_t) * B, st));
  CK(cudaMemcpyAsync(d_n, rm->n.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
  CK(cudaMallocAsync(&d_cnt, sizeof(int32_t) * N, st));
  CK(cudaMallocAsync(&d_over, sizeof(int), st));
  CK(cudaMallocAsync(&d_free, sizeof(unsigned long long) * B, st));
  CK(cudaMemsetAsync(d_free, 0, sizeof(unsigned long long) * B, st));
  CK(cudaMallocAsync(&d_work, sizeof(unsigned long long) * W_NUM, st));
  CK(cudaMemsetAsync(d_work, 0, sizeof(unsigned long long) * W_NUM, st));
  rm->d_row_ptr = static_cast<int64_t*>(rm_alloc(sizeof(int64_t) * (N + 1), st));
  if (!rm->d_row_ptr) return MPAP_ERR_OUT_OF_MEMORY;
  const dim3 grid((rm->n_max + kNearWarps - 1) / kNearWarps, B);
  for (int attempt = 0; attempt < 8; ++attempt) {
    const size_t bytes = sizeof(NearRec) * (size_t)N * (size_t)cap;
    d_scr = static_cast<NearRec*>(workspace(st, WS_NEAR, bytes));
    if (!d_scr) return set_error(MPAP_ERR_OUT_OF_MEMORY, "neighbour scratch allocation failed");
    CK(cudaMemsetAsync(d_over, 0, sizeof(int), st));
    CK(cudaMemsetAsync(d_work, 0, sizeof(unsigned long long) * 3, st));
    {
      ProfScope ps("k_near", st);
      cudaError_t e;
      if (d == 2) e = dyn ? launch_near<2, 1>(grid, st, rm, d_n, cap, d_cnt, d_scr, d_over, d_work)
                          : launch_near<2, 0>(grid, st, rm, d_n, cap, d_cnt, d_scr, d_over, d_work);
      else e = dyn ? launch_near<3, 1>(grid, st, rm, d_n, cap, d_cnt, d_scr, d_over, d_work)
                   : launch_near<3, 0>(grid, st, rm, d_n, cap, d_cnt, d_scr, d_over, d_work);
      CK(e);
    }
    note_launch();
    int over = 0;
    CK(cudaMemcpyAsync(&over, d_over, sizeof(int), cudaMemcpyDeviceToHost, st));
    {
      HostTimer tn("near sync");
      CK(cudaStreamSynchronize(st));
    }
    if (over == 0) break;
    cap = ((over + 31) / 32) * 32;   // exact regrow: re-run with room for the widest row
  }
  HostTimer tnear_done("after near loop -> end");
  {
    ProfScope ps("k_scan", st);
    k_scan<<<1, 1024, 0, st>>>(d_cnt, N, rm->d_row_ptr);
  }
  note_launch();
  CK(cudaGetLastError());
  std::vector<int64_t> bounds(B + 1);
  for (int b = 0; b <= B; ++b) {
    CK(cudaMemcpyAsync(&bounds[b], rm->d_row_ptr + rm->node_base[b], sizeof(int64_t), cudaMemcpyDeviceToHost,
                       st));
  }
  {
    HostTimer tb("bounds sync");
    CK(cudaStreamSynchronize(st));
  }
  rm->edge_base = bounds;
  rm->nnz_total = bounds[B];
  HostTimer te("edges alloc");
  rm->d_edges = static_cast<EdgeRec*>(rm_alloc(sizeof(EdgeRec) * std::max<int64_t>(rm->nnz_total, 1), st));
  if (!rm->d_edges) return set_error(MPAP_ERR_OUT_OF_MEMORY, "edge array allocation failed");
  if (rm->prm.edge_peaks) {
    rm->d_peak = static_cast<float2*>(rm_alloc(sizeof(float2) * std::max<int64_t>(rm->nnz_total, 1), st));
    if (!rm->d_peak) return set_error(MPAP_ERR_OUT_OF_MEMORY, "peak array allocation failed");
  }
  rm->d_tau = static_cast<double*>(rm_alloc(sizeof(double) * std::max<int64_t>(rm->nnz_total, 1), st));
  if (!rm->d_tau) return set_error(MPAP_ERR_OUT_OF_MEMORY, "tau array allocation failed");
  rm->d_esrc = static_cast<int32_t*>(rm_alloc(sizeof(int32_t) * std::max<int64_t>(rm->nnz_total, 1), st));
  if (!rm->d_esrc) return set_error(MPAP_ERR_OUT_OF_MEMORY, "edge source array allocation failed");
  const size_t smem = edges_smem(rm);
  unsigned long long* d_next = nullptr;   // [0..1] item counters of the two edge phases, [2] kv slots, [3] free edges
  CK(cudaMallocAsync(&d_next, 4 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(d_next, 0, 4 * sizeof(unsigned long long), st));
  if (rm->lazy) {   // NEXT-1 part i: Near + Cost only; rows are evaluated on demand
    rm->d_ready = static_cast<int32_t*>(rm_alloc(sizeof(int32_t) * std::max<int64_t>(N, 1), st));
    if (!rm->d_ready) return set_error(MPAP_ERR_OUT_OF_MEMORY, "ready flags allocation failed");
    CK(cudaMemsetAsync(rm->d_ready, 0, sizeof(int32_t) * N, st));
    if (rm->nnz_total > 0) {
      ProfScope ps("k_lazy_init", st);
      k_lazy_init<<<(unsigned)std::min<int64_t>((N + 7) / 8, (int64_t)device_sms() * 16), 256, 0, st>>>(
          d_scr, cap, rm->d_row_ptr, N, rm->d_edges, rm->d_tau, rm->d_esrc, rm->d_peak);
      CK(cudaGetLastError());
      note_launch();
    }
    std::vector<unsigned long long> fr(B);
    for (int b = 0; b < B; ++b) fr[b] = (unsigned long long)(bounds[b + 1] - bounds[b]);   // coll = 0 until evaluated
    CK(cudaMemcpyAsync(d_free, fr.data(), sizeof(unsigned long long) * B, cudaMemcpyHostToDevice, st));
  } else if (rm->nnz_total > 0) {
    EdgeWork ew{d_scr, cap, nullptr, 0, d_free, d_work, d_next, nullptr, nullptr, d_next + 2, nullptr, d_next + 3};
    ew.flist = static_cast<longlong2*>(workspace(st, WS_FLIST, sizeof(longlong2) * rm->nnz_total));
    if (!ew.flist) return set_error(MPAP_ERR_OUT_OF_MEMORY, "free-edge list workspace allocation failed");
    ew.koff = static_cast<long long*>(workspace(st, WS_KOFF, sizeof(long long) * rm->nnz_total));
    if (!ew.koff) return set_error(MPAP_ERR_OUT_OF_MEMORY, "kv offset workspace allocation failed");
    CK(edge_phases(smem, st, rm, ew));
  }
  std::vector<unsigned long long> fr(B);
  CK(cudaMemcpyAsync(fr.data(), d_free, sizeof(unsigned long long) * B, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(rm->work, d_work, sizeof(unsigned long long) * W_NUM, cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d_cnt, st));
  CK(cudaFreeAsync(d_over, st));
  CK(cudaFreeAsync(d_free, st));
  CK(cudaFreeAsync(d_work, st));
  CK(cudaFreeAsync(d_next, st));
  CK(cudaFreeAsync(d_n, st));
  {
    HostTimer tf("final sync");
    CK(cudaStreamSynchronize(st));
  }
  rm->nnz_free.assign(fr.begin(), fr.end());
  return MPAP_OK;
}

// NEXT-1: online update of one environment.  The obstacle and
// feature arrays of rm already hold the new sets; cbox / cfeat are the
// changed boxes and features (symmetric differences, host).  Lists the
// affected edges (k_affected) and re-runs collision and heuristic on exactly
// those (k_edges in item mode), so the roadmap equals a full build of the new
// environment bit for bit.
mpap_status update_roadmap_device(mpap_roadmap* rm, int env, const std::vector<double>& cbox,
                                  const std::vector<double>& cfeat, int64_t* n_reeval, cudaStream_t st) {
  const int d = rm->prm.pos_dim, dyn = rm->prm.dynamics;
  const int nb = (int)(cbox.size() / (2 * d)), nf = (int)(cfeat.size() / d);
  const int64_t row0 = rm->node_base[env], n_rows = rm->n[env];
  const int64_t nnz_env = rm->edge_base[env + 1] - rm->edge_base[env];
  if (n_reeval) *n_reeval = 0;
  if ((nb == 0 && nf == 0) || nnz_env == 0) return MPAP_OK;
  double* d_cb = nullptr;
  double* d_cf = nullptr;
  longlong2* d_items = nullptr;
  unsigned long long* d_ctr = nullptr;   // [0] n_items, [1..2] item counters, [3] kv slots, [4..] work
  CK(cudaMallocAsync(&d_cb, sizeof(double) * std::max<size_t>(cbox.size(), 1), st));
  CK(cudaMallocAsync(&d_cf, sizeof(double) * std::max<size_t>(cfeat.size(), 1), st));
  if (nb) CK(cudaMemcpyAsync(d_cb, cbox.data(), sizeof(double) * cbox.size(), cudaMemcpyHostToDevice, st));
  if (nf) CK(cudaMemcpyAsync(d_cf, cfeat.data(), sizeof(double) * cfeat.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMallocAsync(&d_items, sizeof(longlong2) * nnz_env, st));
  CK(cudaMallocAsync(&d_ctr, sizeof(unsigned long long) * (4 + W_NUM), st));
  CK(cudaMemsetAsync(d_ctr, 0, sizeof(unsigned long long) * (4 + W_NUM), st));
  {
    ProfScope ps("k_affected", st);
    const dim3 grid((unsigned)((n_rows + kWarps - 1) / kWarps));
    const double* es = rm->d_samples + row0 * rm->prm.stride;
    const double R = rm->prm.max_range;
    int64_t fb = 0;
    for (int b = 0; b < env; ++b) fb += rm->n_feat[b];
    const double* ef = rm->d_feat + fb * d;
    const int F = rm->n_feat[env];
    if (d == 2) {
      if (dyn) k_affected<2, 1><<<grid, kWarps * 32, 0, st>>>(es, rm->prm.stride, row0, n_rows, rm->d_row_ptr,
                                                              rm->d_edges, rm->d_tau, R, ef, F, d_cb, nb, d_cf, nf,
                                                              d_items, d_ctr);
      else k_affected<2, 0><<<grid, kWarps * 32, 0, st>>>(es, rm->prm.stride, row0, n_rows, rm->d_row_ptr,
                                                          rm->d_edges, rm->d_tau, R, ef, F, d_cb, nb, d_cf, nf, d_items,
                                                          d_ctr);
    } else {
      if (dyn) k_affected<3, 1><<<grid, kWarps * 32, 0, st>>>(es, rm->prm.stride, row0, n_rows, rm->d_row_ptr,
                                                              rm->d_edges, rm->d_tau, R, ef, F, d_cb, nb, d_cf, nf,
                                                              d_items, d_ctr);
      else k_affected<3, 0><<<grid, kWarps * 32, 0, st>>>(es, rm->prm.stride, row0, n_rows, rm->d_row_ptr,
                                                          rm->d_edges, rm->d_tau, R, ef, F, d_cb, nb, d_cf, nf, d_items,
                                                          d_ctr);
    }
    CK(cudaGetLastError());
  }
  note_launch();
  unsigned long long n_items = 0;
  CK(cudaMemcpyAsync(&n_items, d_ctr, sizeof(n_items), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (n_items > 0) {
    // the free-edge delta is accumulated in a per-env array indexed by env
    unsigned long long* d_free = nullptr;
    CK(cudaMallocAsync(&d_free, sizeof(unsigned long long) * rm->B, st));
    CK(cudaMemsetAsync(d_free, 0, sizeof(unsigned long long) * rm->B, st));
    const size_t smem = edges_smem(rm);
    EdgeWork ew{nullptr, 0, d_items, (int64_t)n_items, d_free, d_ctr + 4 - W_EDGES, d_ctr + 1, nullptr, nullptr,
                d_ctr + 3, nullptr, nullptr};
    ew.koff = static_cast<long long*>(workspace(st, WS_KOFF, sizeof(long long) * rm->nnz_total));
    if (!ew.koff) return set_error(MPAP_ERR_OUT_OF_MEMORY, "kv offset workspace allocation failed");
    CK(edge_phases(smem, st, rm, ew));
    unsigned long long delta = 0;
    CK(cudaMemcpyAsync(&delta, d_free + env, sizeof(delta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaFreeAsync(d_free, st));
    rm->nnz_free[env] += (int64_t)(long long)delta;
  }
  CK(cudaFreeAsync(d_cb, st));
  CK(cudaFreeAsync(d_cf, st));
  CK(cudaFreeAsync(d_items, st));
  CK(cudaFreeAsync(d_ctr, st));
  CK(cudaStreamSynchronize(st));
  if (n_reeval) *n_reeval = (int64_t)n_items;
  return MPAP_OK;
}

mpap_status evaluate_rows_device(mpap_roadmap* rm, const int32_t* d_rows, int64_t n_req, cudaStream_t st) {
  if (!rm->lazy || rm->nnz_total == 0) return MPAP_OK;
  const int64_t N = rm->node_base[rm->B];
  if (d_rows && n_req <= 0) return MPAP_OK;
  longlong2* d_items = nullptr;
  unsigned long long* d_ctr = nullptr;   // [0] n_items, [1..2] item counters, [3] kv slots, [4..] work
  CK(cudaMallocAsync(&d_items, sizeof(longlong2) * rm->nnz_total, st));
  CK(cudaMallocAsync(&d_ctr, sizeof(unsigned long long) * (4 + W_NUM), st));
  CK(cudaMemsetAsync(d_ctr, 0, sizeof(unsigned long long) * (4 + W_NUM), st));
  {
    ProfScope ps("k_row_items", st);
    const int64_t n = d_rows ? n_req : N;
    k_row_items<<<(unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)device_sms() * 16), 256, 0, st>>>(d_rows, n_req, N, rm->d_row_ptr,
                                                                                    rm->d_ready, d_items, d_ctr);
    CK(cudaGetLastError());
  }
  note_launch();
  unsigned long long n_items = 0;
  CK(cudaMemcpyAsync(&n_items, d_ctr, sizeof(n_items), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (n_items > 0) {
    unsigned long long* d_free = nullptr;
    CK(cudaMallocAsync(&d_free, sizeof(unsigned long long) * rm->B, st));
    CK(cudaMemsetAsync(d_free, 0, sizeof(unsigned long long) * rm->B, st));
    EdgeWork ew{nullptr, 0, d_items, (int64_t)n_items, d_free, d_ctr + 4 - W_EDGES, d_ctr + 1, nullptr, nullptr,
                d_ctr + 3, nullptr, nullptr};
    ew.koff = static_cast<long long*>(workspace(st, WS_KOFF, sizeof(long long) * rm->nnz_total));
    if (!ew.koff) return set_error(MPAP_ERR_OUT_OF_MEMORY, "kv offset workspace allocation failed");
    CK(edge_phases(edges_smem(rm), st, rm, ew));
    std::vector<unsigned long long> delta(rm->B), work(W_NUM - W_EDGES);
    CK(cudaMemcpyAsync(delta.data(), d_free, sizeof(unsigned long long) * rm->B, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(work.data(), d_ctr + 4, sizeof(unsigned long long) * (W_NUM - W_EDGES), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    CK(cudaFreeAsync(d_free, st));
    for (int b = 0; b < rm->B; ++b) rm->nnz_free[b] += (int64_t)(long long)delta[b];
    for (int i = W_EDGES; i < W_NUM; ++i) rm->work[i] += work[i - W_EDGES];
  }
  CK(cudaFreeAsync(d_items, st));
  CK(cudaFreeAsync(d_ctr, st));
  CK(cudaStreamSynchronize(st));
  return MPAP_OK;
}

}  // namespace mpap
