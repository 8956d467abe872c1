// paper_1705_02408_b200/csrc/traj.cuh -- double-integrator edge trajectory
// (reading R7 step 6): p(t) = p0 + v0 t + c2 t^2 + c3 t^3 on
// [0, tau], shared by the build kernels (collision polyline, heuristic steps)
// and the Monte Carlo kernel (nominal trajectory).  Operation order is the
// numeric contract's; compiled with --fmad=false.
#pragma once

namespace mpap {

template <int D>
__device__ __forceinline__ void di_traj(const double* su, const double* sv, double tau, double* c2, double* c3) {
  const double tau2 = tau * tau;
  const double tau3 = tau2 * tau;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double dp = (sv[j] - su[j]) - su[D + j] * tau;
    const double dl = sv[D + j] - su[D + j];
    c2[j] = (3.0 * dp - dl * tau) / tau2;
    c3[j] = (dl * tau - 2.0 * dp) / tau3;
  }
}

template <int D>
__device__ __forceinline__ void di_pos(const double* su, const double* c2, const double* c3, double t, double* x) {
#pragma unroll
  for (int j = 0; j < D; ++j) x[j] = fma(t, fma(t, fma(t, c3[j], c2[j]), su[D + j]), su[j]);
}

template <int D>
__device__ __forceinline__ void di_vel(const double* su, const double* c2, const double* c3, double t, double* v) {
#pragma unroll
  for (int j = 0; j < D; ++j) v[j] = fma(t, fma(t, 3.0 * c3[j], 2.0 * c2[j]), su[D + j]);
}

}  // namespace mpap
