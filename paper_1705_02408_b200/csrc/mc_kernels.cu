// paper_1705_02408_b200/csrc/mc_kernels.cu -- Monte Carlo verification on sm_100a.
//
// Alg. 1 step 4: "an asymptotically exact probability of
// motion plan p satisfying a localization error bound through MC sampling"
// (§3), with the simulation model of §4.1: the 6D
// double integrator tracks the plan's nominal trajectory with a
// feedback law on its ESTIMATED state, an inertial estimate from a
// noisy accelerometer, a translation-only 3D-to-3D position fix from
// the features in view from the TRUE state and a Kalman filter
// (P:320).  Readings R31-R36 fix the model, the operation
// order and the counter-based noise generator; the CPU oracle implements the
// same contract independently, so per-trial results are bit-identical.
//
//   k_mc_plan  thread per plan edge: finds the edge in the roadmap CSR (it
//              must be collision-free), reads its duration tau (built by
//              k_near) and writes the trajectory segment (cubic coefficients,
//              K = ceil(tau/dt) steps of Dl = tau/K).
//   k_mc       warp per (plan, trial), persistent over a grid of 148 x
//              resident blocks.  The vehicle/filter state is warp-uniform
//              (every lane computes it, so no broadcasts); the per-step
//              visibility test runs lane-per-feature against the env's
//              features and boxes staged in the warp's shared memory; the
//              noise of each visible feature is drawn by its lane at counter
//              index base + rank * d + axis (rank = ballot prefix), and the
//              fix is summed in feature-index order from shared memory.
//
// Trials are independent (one counter-based stream each), so the batch
// shards across GPUs like the searches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "mpap_internal.cuh"
#include "traj.cuh"

namespace mpap {

#define FULLW 0xffffffffu
constexpr int kMcWarps = 4;                 // warps per k_mc block
#ifndef MPAP_MC_MIN_BLOCKS
#define MPAP_MC_MIN_BLOCKS 4                // 4 x 4 warps per SM: at most 128 registers
#endif

constexpr float kMcCullMarginF = 1e-4f;     // box vs sight-line bounding-box gap (f32) that provably misses:
                                            // rounding of O(100) m coordinates is < 1e-5

// per-warp shared memory: features [F][D], boxes [O][2D] (doubles); the
// candidate sight-line boxes [F][2D] (floats, phases a-b of a step) share
// their space with the fix contributions [F][D] (doubles, phases d-e);
// candidate list and occluded flags [F] each, near-box list [O] (ints);
// boxes [O][2D] (floats, for the exact culls)
__host__ __device__ constexpr size_t mc_warp_doubles(int d, int f_max, int o_max) {
  return (size_t)f_max * d * 2 + (size_t)o_max * 2 * d + (size_t)f_max + ((size_t)o_max + 1) / 2 +
         (size_t)o_max * d;
}

struct McSeg {
  double su[6];      // source node p0[D], v0[D]
  double hu[2], hv[2];  // source / destination heading (cos yaw, sin yaw)
  double c2[3], c3[3];
  double T, Dl;
  int K, pad;
};

struct McParamsDev {
  uint64_t seed, trial0;
  double sigma_imu, sigma_vis, u_max, k_p, k_d, p0_pos, p0_vel, delta;
  int trials;
};

// SplitMix64 finaliser over a Weyl sequence (reading R33).
__device__ __forceinline__ uint64_t mc_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// normal number idx of the stream with key mc_mix(seed + G (trial + 1)):
// Irwin-Hall sum of the 12 32-bit halves of 6 draws, minus 6 (exact in f64).
__device__ __forceinline__ double mc_normal(uint64_t key, uint64_t idx) {
  const uint64_t G = 0x9E3779B97F4A7C15ULL;
  uint64_t S = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint64_t w = mc_mix(key + G * (idx * 6ULL + (uint64_t)i + 1ULL));
    S += (w & 0xffffffffULL) + (w >> 32);
  }
  return __ull2double_rn(S) * (1.0 / 4294967296.0) - 6.0;
}

template <int D>
__global__ void k_mc_plan(const double* __restrict__ samples, int stride, int hoff,
                          const int64_t* __restrict__ node_base, const int64_t* __restrict__ row_ptr,
                          const EdgeRec* __restrict__ edges, const double* __restrict__ tau,
                          const int32_t* __restrict__ envs, const int32_t* __restrict__ paths, int path_stride,
                          const int32_t* __restrict__ path_lens, const int64_t* __restrict__ seg_off, int n_plans,
                          double dt, McSeg* __restrict__ segs, int* __restrict__ bad,
                          unsigned long long* __restrict__ steps) {
  const int64_t total = seg_off[n_plans];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_plans - 1;   // plan of segment g: last p with seg_off[p] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg_off[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const int p = lo;
    const int j = (int)(g - seg_off[p]);
    const int32_t* path = paths + (size_t)p * path_stride;
    const int u = path[j], v = path[j + 1];
    const int64_t nb = node_base[envs[p]];
    const int64_t e0 = row_ptr[nb + u], e1 = row_ptr[nb + u + 1];
    int64_t e = -1;
    for (int64_t k = e0; k < e1; ++k)
      if ((int)(edges[k].dst_coll & 0x7fffffffu) == v) { e = k; break; }
    McSeg S;
    memset(&S, 0, sizeof(S));
    if (e < 0 || (edges[e].dst_coll >> 31)) {
      bad[p] = 1;
      segs[g] = S;
      continue;
    }
    const double* su = samples + (size_t)(nb + u) * stride;
    const double* sv = samples + (size_t)(nb + v) * stride;
    const double T = tau[e];
    for (int q = 0; q < 2 * D; ++q) S.su[q] = su[q];
    if (hoff >= 0) {
      S.hu[0] = su[hoff]; S.hu[1] = su[hoff + 1];
      S.hv[0] = sv[hoff]; S.hv[1] = sv[hoff + 1];
    }
    di_traj<D>(su, sv, T, S.c2, S.c3);
    const double kk = ceil(T / dt);
    S.K = (kk < 1.0) ? 1 : (int)kk;
    S.T = T;
    S.Dl = T / (double)S.K;
    segs[g] = S;
    atomicAdd(&steps[p], (unsigned long long)S.K);
  }
}

// Closed segment [A, B] (Dv = B - A) vs closed box: the slab test of the
// contract (R8), 1/Dv_k correctly rounded.
template <int D>
__device__ __forceinline__ bool mc_seg_box(const double* A, const double* Dv, const double* inv, const double* bx) {
  double t0 = 0.0, t1 = 1.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double lo = bx[k], hi = bx[D + k];
    if (Dv[k] == 0.0) {
      if (A[k] < lo || A[k] > hi) return false;
    } else {
      double ta = (lo - A[k]) * inv[k];
      double tb = (hi - A[k]) * inv[k];
      if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
      if (t0 > t1) return false;
    }
  }
  return true;
}

template <int D, int HEUR>
__global__ void __launch_bounds__(kMcWarps * 32, MPAP_MC_MIN_BLOCKS) k_mc(const double* __restrict__ feat_all,
                                                       const int32_t* __restrict__ feat_base,
                                                       const double* __restrict__ box_all,
                                                       const int32_t* __restrict__ obst_base,
                                                       const int32_t* __restrict__ envs,
                                                       const int64_t* __restrict__ seg_off,
                                                       const McSeg* __restrict__ segs, const int* __restrict__ bad,
                                                       int n_plans, McParamsDev M, double max_range,
                                                       double fov_cos_half, int f_max, int o_max,
                                                       double* __restrict__ max_err, double* __restrict__ max_dev,
                                                       unsigned long long* __restrict__ exceed,
                                                       unsigned long long* __restrict__ fixes) {
  extern __shared__ double mc_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wf = mc_smem + (size_t)warp * mc_warp_doubles(D, f_max, o_max);
  double* wb = wf + (size_t)f_max * D;       // boxes [O][2D]
  double* wc = wb + (size_t)o_max * 2 * D;   // fix contributions [F][D] in rank order
  float* wsb = reinterpret_cast<float*>(wc);  // candidate sight-line boxes, f32 [F][2D] (aliases wc)
  int* wl = reinterpret_cast<int*>(wc + (size_t)f_max * D);   // candidate / visible feature list [F]
  int* wo = wl + f_max;                                        // candidate occluded flags [F]
  int* wn = wo + f_max;                                        // boxes near x this step [O]
  float* wbf = reinterpret_cast<float*>(wn + ((o_max + 1) & ~1));   // boxes, f32 [O][2D]
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  const double R2 = max_range * max_range;
  const float rnear = (float)max_range + 1e-3f;
  const float rnear2 = rnear * rnear;
  const double cos2 = fov_cos_half * fov_cos_half;
  const double q = M.sigma_imu * M.sigma_imu;
  const double rv = M.sigma_vis * M.sigma_vis;
  const int64_t items = (int64_t)n_plans * M.trials;
  const int64_t nwarps = (int64_t)gridDim.x * kMcWarps;
  int cur_env = -1, F = 0, O = 0;
  for (int64_t it = (int64_t)blockIdx.x * kMcWarps + warp; it < items; it += nwarps) {
    const int p = (int)(it / M.trials);
    const int64_t tr = (int64_t)M.trial0 + it % M.trials;
    if (bad[p]) continue;
    const int env = envs[p];
    if (env != cur_env) {   // stage the environment's features and boxes
      __syncwarp();
      const int fb = feat_base[env], ob = obst_base[env];
      F = feat_base[env + 1] - fb;
      O = obst_base[env + 1] - ob;
      for (int i = lane; i < F * D; i += 32) wf[i] = feat_all[(size_t)fb * D + i];
      for (int i = lane; i < O * 2 * D; i += 32) {
        const double b = box_all[(size_t)ob * 2 * D + i];
        wb[i] = b;
        wbf[i] = (float)b;
      }
      cur_env = env;
      __syncwarp();
    }
    const uint64_t key = mc_mix(M.seed + 0x9E3779B97F4A7C15ULL * ((uint64_t)tr + 1ULL));
    const int64_t s0 = seg_off[p], s1 = seg_off[p + 1];
    double x[D], v[D], xh[D], vh[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { x[j] = 0.0; v[j] = 0.0; }
    if (s0 < s1) {   // a zero-edge plan (start in goal) has no steps and zero errors
      const McSeg& S = segs[s0];
#pragma unroll
      for (int j = 0; j < D; ++j) { x[j] = S.su[j]; v[j] = S.su[D + j]; }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) { xh[j] = x[j]; vh[j] = v[j]; }
    double p11 = M.p0_pos, p12 = 0.0, p22 = M.p0_vel;
    double me = 0.0, md = 0.0;
    uint64_t ctr = 0;
    unsigned long long nfix = 0;
    for (int64_t sg = s0; sg < s1; ++sg) {
      const McSeg& S = segs[sg];
      const double T = S.T, Dl = S.Dl, D2 = Dl * Dl;
      double c2[D], c3[D], su[2 * D];
#pragma unroll
      for (int j = 0; j < D; ++j) { c2[j] = S.c2[j]; c3[j] = S.c3[j]; su[j] = S.su[j]; su[D + j] = S.su[D + j]; }
      const double hu0 = S.hu[0], hu1 = S.hu[1], hv0 = S.hv[0], hv1 = S.hv[1];
      for (int k = 0; k < S.K; ++k) {
        const double t = (double)k * Dl;
        double xn[D], vn[D];
        di_pos<D>(su, c2, c3, t, xn);
        di_vel<D>(su, c2, c3, t, vn);
        // (1) control on the estimate, saturated; (2) true dynamics
        double u[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double an = fma(t, 6.0 * c3[j], 2.0 * c2[j]);
          double uj = (an + M.k_p * (xn[j] - xh[j])) + M.k_d * (vn[j] - vh[j]);
          if (uj > M.u_max) uj = M.u_max;
          if (uj < -M.u_max) uj = -M.u_max;
          u[j] = uj;
          v[j] = v[j] + uj * Dl;
          x[j] = x[j] + v[j] * Dl;
        }
        // (3) accelerometer + filter prediction: lane j draws axis j's noise
        double nz = 0.0;
        if (lane < D) nz = mc_normal(key, ctr + (uint64_t)lane);
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double am = u[j] + M.sigma_imu * __shfl_sync(FULLW, nz, j);
          vh[j] = vh[j] + am * Dl;
          xh[j] = xh[j] + vh[j] * Dl;
        }
        ctr += D;
        {
          const double a = Dl * p12;
          const double n11 = (((p11 + a) + a) + D2 * p22) + q * (D2 * D2);
          const double n12 = (p12 + Dl * p22) + q * (D2 * Dl);
          const double n22 = p22 + q * D2;
          p11 = n11; p12 = n12; p22 = n22;
        }
        // (4) features in view from the true state at t + Dl
        const double t1 = (double)(k + 1) * Dl;
        double hvec[D];
#pragma unroll
        for (int j = 0; j < D; ++j) hvec[j] = 0.0;
        if (HEUR == 1) {
#pragma unroll
          for (int j = 0; j < D; ++j) hvec[j] = v[j];
        } else if (HEUR >= 2) {
          const double s = t1 / T;
          hvec[0] = fma(s, hv0, (1.0 - s) * hu0);
          hvec[1] = fma(s, hv1, (1.0 - s) * hu1);
        }
        double hh = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) hh = fma(hvec[j], hvec[j], hh);
        // (a) range and FOV, lane per feature -> candidate list (index order)
        int nc = 0;
        for (int f0 = 0; f0 < F; f0 += 32) {
          const int f = f0 + lane;
          bool cand = false;
          if (f < F) {
            double dl[D];
            double dd = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) { dl[j] = wf[f * D + j] - x[j]; dd = fma(dl[j], dl[j], dd); }
            cand = !(dd > R2);
            if (cand && HEUR != 0) {
              double dot = 0.0;
#pragma unroll
              for (int j = 0; j < D; ++j) dot = fma(hvec[j], dl[j], dot);
              if (!(hh > 0.0) || dot < 0.0 || dot * dot < cos2 * (hh * dd)) cand = false;
            }
          }
          const unsigned cm = __ballot_sync(FULLW, cand);
          if (cand) {
            const int pos = nc + __popc(cm & lt);
            wl[pos] = f;
            wo[pos] = 0;
#pragma unroll
            for (int j = 0; j < D; ++j) {   // bounding box of the sight line [x, f], grown
              const double fj = wf[f * D + j];
              wsb[pos * 2 * D + j] = (float)fmin(x[j], fj) - kMcCullMarginF;
              wsb[pos * 2 * D + D + j] = (float)fmax(x[j], fj) + kMcCullMarginF;
            }
          }
          nc += __popc(cm);
        }
        // boxes that can meet a sight line: within max_range + 1e-3 of x (every
        // candidate is within max_range, so its sight line is in that ball)
        int nn = 0;
        if (nc > 0) {
          float xf[D];
#pragma unroll
          for (int j = 0; j < D; ++j) xf[j] = (float)x[j];
          for (int o0 = 0; o0 < O; o0 += 32) {
            const int o = o0 + lane;
            bool near = false;
            if (o < O) {
              float g2 = 0.0f;
#pragma unroll
              for (int j = 0; j < D; ++j) {
                const float e = fmaxf(fmaxf(wbf[o * 2 * D + j] - xf[j], xf[j] - wbf[o * 2 * D + D + j]), 0.0f);
                g2 += e * e;
              }
              near = g2 <= rnear2;
            }
            const unsigned nm = __ballot_sync(FULLW, near);
            if (near) wn[nn + __popc(nm & lt)] = o;
            nn += __popc(nm);
          }
        }
        __syncwarp();
        // (b) occlusion, lane per (candidate, box) pair: a candidate is in
        // view iff no box meets its sight line [x, f] (order-free OR)
        if (nn > 0 && nc > 0) {
          const int npair = nc * nn;
          int c = lane / nn, o = lane - c * nn;
          for (int p0 = 0; p0 < npair; p0 += 32) {
            if (p0 + lane < npair && !wo[c]) {
              const int b = wn[o];
              const float* bf = wbf + b * 2 * D;
              const float* sb = wsb + c * 2 * D;
              bool sep = false;
#pragma unroll
              for (int j = 0; j < D; ++j)
                if (bf[j] > sb[D + j] || bf[D + j] < sb[j]) sep = true;
              if (!sep) {
                double dl[D], inv[D];
#pragma unroll
                for (int j = 0; j < D; ++j) {
                  dl[j] = wf[wl[c] * D + j] - x[j];
                  inv[j] = (dl[j] != 0.0) ? 1.0 / dl[j] : 0.0;
                }
                if (mc_seg_box<D>(x, dl, inv, wb + b * 2 * D)) wo[c] = 1;
              }
            }
            o += 32;
            while (o >= nn) { o -= nn; ++c; }
          }
          __syncwarp();
        }
        // (c) visible list in index order (in-place compaction, pos <= i)
        int kv = 0;
        for (int i0 = 0; i0 < nc; i0 += 32) {
          const int i = i0 + lane;
          const bool vis = (i < nc) && !wo[i];
          const int f = vis ? wl[i] : 0;
          const unsigned vm = __ballot_sync(FULLW, vis);
          __syncwarp();
          if (vis) wl[kv + __popc(vm & lt)] = f;
          kv += __popc(vm);
        }
        __syncwarp();
        // (d) z_f = (f - x) + noise, normal index base + rank * d + axis,
        // lane per (rank, axis); contribution f - z_f
        for (int n0 = 0; n0 < kv * D; n0 += 32) {
          const int n = n0 + lane;
          if (n < kv * D) {
            const int i = n / D, j = n - (n / D) * D;
            double xj = x[0];
#pragma unroll
            for (int jj = 1; jj < D; ++jj)
              if (j == jj) xj = x[jj];
            const double fc = wf[wl[i] * D + j];
            const double z = (fc - xj) + M.sigma_vis * mc_normal(key, ctr + (uint64_t)n);
            wc[n] = fc - z;
          }
        }
        __syncwarp();
        if (kv > 0) {
          double sum[D];
#pragma unroll
          for (int j = 0; j < D; ++j) sum[j] = 0.0;
          for (int i = 0; i < kv; ++i) {
#pragma unroll
            for (int j = 0; j < D; ++j) sum[j] = sum[j] + wc[i * D + j];
          }
          ctr += (uint64_t)kv * D;
          const double Rm = rv / (double)kv;
          const double Sv = p11 + Rm;
          double K1 = 0.0, K2 = 0.0;
          if (Sv > 0.0) { K1 = p11 / Sv; K2 = p12 / Sv; }
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const double fix = sum[j] / (double)kv;
            const double y = fix - xh[j];
            xh[j] = xh[j] + K1 * y;
            vh[j] = vh[j] + K2 * y;
          }
          const double n11 = p11 - K1 * p11;
          const double n12 = p12 - K1 * p12;
          const double n22 = p22 - K2 * p12;
          p11 = n11; p12 = n12; p22 = n22;
          ++nfix;
        }
        __syncwarp();   // wc is rewritten next step
        // (6) localisation error and deviation at t + Dl
        double xn1[D];
        di_pos<D>(su, c2, c3, t1, xn1);
        double ee = 0.0, dv = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double a = xh[j] - x[j];
          const double b = xn1[j] - x[j];
          ee = ee + a * a;
          dv = dv + b * b;
        }
        const double err = sqrt(ee), dev = sqrt(dv);
        if (err > me) me = err;
        if (dev > md) md = dev;
      }
    }
    if (lane == 0) {
      max_err[it] = me;
      max_dev[it] = md;
      if (me >= M.delta) atomicAdd(&exceed[p], 1ull);
      if (nfix) atomicAdd(&fixes[p], nfix);
    }
  }
}

#define CKM(x)                                         \
  do {                                                 \
    cudaError_t _e = (x);                              \
    if (_e != cudaSuccess) return cuda_error(_e, #x);  \
  } while (0)

template <int D, int HEUR>
static cudaError_t launch_mc(int nsm, size_t smem, cudaStream_t st, const mpap_roadmap* rm, const int32_t* d_envs,
                             const int64_t* d_off, const McSeg* d_segs, const int* d_bad, int n_plans,
                             const McParamsDev& M, double* d_err, double* d_dev, unsigned long long* d_ctr) {
  auto kern = k_mc<D, HEUR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMcWarps * 32, smem);
  if (e != cudaSuccess) return e;
  const int64_t items = (int64_t)n_plans * M.trials;
  const int64_t want = (items + kMcWarps - 1) / kMcWarps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(occ, 1), want));
  ProfScope ps("k_mc", st);
  kern<<<grid, kMcWarps * 32, smem, st>>>(rm->d_feat, rm->d_feat_base, rm->d_obst, rm->d_obst_base, d_envs, d_off,
                                          d_segs, d_bad, n_plans, M, rm->prm.max_range, rm->prm.fov_cos_half,
                                          std::max(rm->f_max, 1), std::max(rm->o_max, 1), d_err, d_dev, d_ctr,
                                          d_ctr + n_plans);
  note_launch();
  return cudaGetLastError();
}

mpap_status mc_verify_device(const mpap_roadmap* rm, int32_t n_plans, const int32_t* envs, const int32_t* paths,
                             int32_t path_stride, const int32_t* path_lens, const mpap_mc_params* mc,
                             uint64_t trial0, double* max_err, double* max_dev, mpap_mc_result* results,
                             cudaStream_t st) {
  if (n_plans <= 0) return MPAP_OK;
  const int d = rm->prm.pos_dim;
  int dev = 0, nsm = 0;
  CKM(cudaGetDevice(&dev));
  CKM(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  std::vector<int64_t> off(n_plans + 1, 0);
  for (int p = 0; p < n_plans; ++p) off[p + 1] = off[p] + (path_lens[p] - 1);
  const int64_t nseg = off[n_plans];
  const int64_t items = (int64_t)n_plans * mc->trials;
  // one stream-ordered arena for the launch
  size_t o_envs = 0, o_paths = 256 * ((sizeof(int32_t) * n_plans + 255) / 256);
  size_t o_lens = o_paths + 256 * ((sizeof(int32_t) * (size_t)n_plans * path_stride + 255) / 256);
  size_t o_off = o_lens + 256 * ((sizeof(int32_t) * n_plans + 255) / 256);
  size_t o_segs = o_off + 256 * ((sizeof(int64_t) * (n_plans + 1) + 255) / 256);
  size_t o_bad = o_segs + 256 * ((sizeof(McSeg) * std::max<int64_t>(nseg, 1) + 255) / 256);
  size_t o_ctr = o_bad + 256 * ((sizeof(int) * n_plans + 255) / 256);
  size_t o_err = o_ctr + 256 * ((sizeof(unsigned long long) * 3 * n_plans + 255) / 256);
  size_t o_dev = o_err + 256 * ((sizeof(double) * items + 255) / 256);
  size_t bytes = o_dev + 256 * ((sizeof(double) * items + 255) / 256);
  char* base = nullptr;
  CKM(cudaMallocAsync(&base, bytes, st));
  int32_t* d_envs = reinterpret_cast<int32_t*>(base + o_envs);
  int32_t* d_paths = reinterpret_cast<int32_t*>(base + o_paths);
  int32_t* d_lens = reinterpret_cast<int32_t*>(base + o_lens);
  int64_t* d_off = reinterpret_cast<int64_t*>(base + o_off);
  McSeg* d_segs = reinterpret_cast<McSeg*>(base + o_segs);
  int* d_bad = reinterpret_cast<int*>(base + o_bad);
  unsigned long long* d_ctr = reinterpret_cast<unsigned long long*>(base + o_ctr);   // exceed, fixes, steps
  double* d_err = reinterpret_cast<double*>(base + o_err);
  double* d_dev = reinterpret_cast<double*>(base + o_dev);
  mpap_status status = MPAP_OK;
  do {
    cudaError_t e;
#define CKB(x)                                     \
  if ((e = (x)) != cudaSuccess) {                  \
    status = cuda_error(e, #x);                    \
    break;                                         \
  }
    CKB(cudaMemcpyAsync(d_envs, envs, sizeof(int32_t) * n_plans, cudaMemcpyHostToDevice, st));
    CKB(cudaMemcpyAsync(d_paths, paths, sizeof(int32_t) * (size_t)n_plans * path_stride, cudaMemcpyHostToDevice, st));
    CKB(cudaMemcpyAsync(d_lens, path_lens, sizeof(int32_t) * n_plans, cudaMemcpyHostToDevice, st));
    CKB(cudaMemcpyAsync(d_off, off.data(), sizeof(int64_t) * (n_plans + 1), cudaMemcpyHostToDevice, st));
    CKB(cudaMemsetAsync(d_bad, 0, sizeof(int) * n_plans, st));
    CKB(cudaMemsetAsync(d_ctr, 0, sizeof(unsigned long long) * 3 * n_plans, st));
    const int hoff = rm->prm.has_heading ? 2 * d : -1;
    if (nseg > 0) {
      const int thr = 128;
      const int grid = (int)std::min<int64_t>((nseg + thr - 1) / thr, (int64_t)nsm * 8);
      ProfScope ps("k_mc_plan", st);
      if (d == 3)
        k_mc_plan<3><<<grid, thr, 0, st>>>(rm->d_samples, rm->prm.stride, hoff, rm->d_node_base, rm->d_row_ptr,
                                           rm->d_edges, rm->d_tau, d_envs, d_paths, path_stride, d_lens, d_off,
                                           n_plans, rm->prm.dt, d_segs, d_bad, d_ctr + 2 * n_plans);
      else
        k_mc_plan<2><<<grid, thr, 0, st>>>(rm->d_samples, rm->prm.stride, hoff, rm->d_node_base, rm->d_row_ptr,
                                           rm->d_edges, rm->d_tau, d_envs, d_paths, path_stride, d_lens, d_off,
                                           n_plans, rm->prm.dt, d_segs, d_bad, d_ctr + 2 * n_plans);
      note_launch();
      CKB(cudaGetLastError());
    }
    McParamsDev M;
    M.seed = mc->seed;
    M.trial0 = trial0;
    M.sigma_imu = mc->sigma_imu;
    M.sigma_vis = mc->sigma_vis;
    M.u_max = mc->u_max;
    M.k_p = mc->k_p;
    M.k_d = mc->k_d;
    M.p0_pos = mc->p0_pos;
    M.p0_vel = mc->p0_vel;
    M.delta = mc->delta;
    M.trials = mc->trials;
    const size_t smem = sizeof(double) * kMcWarps * mc_warp_doubles(d, std::max(rm->f_max, 1), std::max(rm->o_max, 1));
    const int heur = rm->prm.heuristic;
    cudaError_t le;
    if (d == 3) {
      if (heur == 0) le = launch_mc<3, 0>(nsm, smem, st, rm, d_envs, d_off, d_segs, d_bad, n_plans, M, d_err, d_dev, d_ctr);
      else if (heur == 1) le = launch_mc<3, 1>(nsm, smem, st, rm, d_envs, d_off, d_segs, d_bad, n_plans, M, d_err, d_dev, d_ctr);
      else le = launch_mc<3, 2>(nsm, smem, st, rm, d_envs, d_off, d_segs, d_bad, n_plans, M, d_err, d_dev, d_ctr);
    } else {
      if (heur == 0) le = launch_mc<2, 0>(nsm, smem, st, rm, d_envs, d_off, d_segs, d_bad, n_plans, M, d_err, d_dev, d_ctr);
      else if (heur == 1) le = launch_mc<2, 1>(nsm, smem, st, rm, d_envs, d_off, d_segs, d_bad, n_plans, M, d_err, d_dev, d_ctr);
      else le = launch_mc<2, 2>(nsm, smem, st, rm, d_envs, d_off, d_segs, d_bad, n_plans, M, d_err, d_dev, d_ctr);
    }
    CKB(le);
    std::vector<unsigned long long> ctr(3 * (size_t)n_plans);
    std::vector<int> hbad(n_plans);
    CKB(cudaMemcpyAsync(ctr.data(), d_ctr, sizeof(unsigned long long) * 3 * n_plans, cudaMemcpyDeviceToHost, st));
    CKB(cudaMemcpyAsync(hbad.data(), d_bad, sizeof(int) * n_plans, cudaMemcpyDeviceToHost, st));
    if (max_err) CKB(cudaMemcpyAsync(max_err, d_err, sizeof(double) * items, cudaMemcpyDeviceToHost, st));
    if (max_dev) CKB(cudaMemcpyAsync(max_dev, d_dev, sizeof(double) * items, cudaMemcpyDeviceToHost, st));
    CKB(cudaStreamSynchronize(st));
    for (int p = 0; p < n_plans; ++p) {
      mpap_mc_result r;
      memset(&r, 0, sizeof(r));
      r.status = hbad[p] ? MPAP_ERR_INVALID_ARGUMENT : MPAP_OK;
      r.trials = mc->trials;
      r.exceed = (int64_t)ctr[p];
      r.fixes = (int64_t)ctr[n_plans + p];
      r.steps = (int64_t)ctr[2 * n_plans + p];
      r.p_hat = hbad[p] ? 0.0 : (double)r.exceed / (double)mc->trials;
      results[p] = r;
    }
#undef CKB
  } while (0);
  cudaFreeAsync(base, st);
  return status;
}

}  // namespace mpap
