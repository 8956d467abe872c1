// paper_1705_02408_b200/csrc/peak_kernels.cu -- FP64 issue-rate microbenchmark.
//
// The build kernels are bound by the FP64 pipe, whose peak is
// not in MEASURED_PEAKS.json (that file holds HBM copy and bf16 GEMM only).
// bench.py measures it live with this kernel on the same GPU and clocks as
// the step it reports: one persistent block per resident slot, every thread
// runs kChains independent dependency chains of the timed instruction (DFMA,
// DADD or DMUL; one instruction = one counted op, the convention of the
// build's work counters), enough chains x warps to cover the pipe latency.
#include <cuda_runtime.h>

#include "mpap_internal.cuh"

namespace mpap {

constexpr int kPeakThreads = 256;
constexpr int kChains = 8;

template <int KIND>
__global__ void __launch_bounds__(kPeakThreads) k_fp64_peak(double seed, int iters, double* __restrict__ sink) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed + (double)(threadIdx.x * kChains + c) * 1e-9;
  const double m = 0.999999999, b = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if (KIND == 0) a[c] = fma(a[c], m, b);
        else if (KIND == 1) a[c] = a[c] + b;
        else a[c] = a[c] * m;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c];
  if (s == 12345.678) sink[blockIdx.x] = s;   // never true; keeps the chains live
}

}  // namespace mpap

using namespace mpap;

extern "C" mpap_status mpap_prof_fp64_peak(int32_t kind, double* ops_per_s, double* ms) {
  if (!ops_per_s || kind < 0 || kind > 2) return set_error(MPAP_ERR_INVALID_ARGUMENT, "fp64_peak: bad argument");
  int dev = 0, sms = 0, per_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_error(e, "cudaGetDevice");
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void (*fn)(double, int, double*) = kind == 0 ? k_fp64_peak<0> : (kind == 1 ? k_fp64_peak<1> : k_fp64_peak<2>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPeakThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const int blocks = sms * per_sm;
  double* sink = nullptr;
  e = cudaMalloc(&sink, sizeof(double) * (size_t)blocks);
  if (e != cudaSuccess) return cuda_error(e, "cudaMalloc");
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  fn<<<blocks, kPeakThreads>>>(1.0, 64, sink);   // warm-up (clocks ramp)
  note_launch();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    fn<<<blocks, kPeakThreads>>>(1.0, iters, sink);
    note_launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t = 0.0f;
    cudaEventElapsedTime(&t, a, b);
    if (t < best) best = t;
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (e != cudaSuccess) return cuda_error(e, "k_fp64_peak");
  const double ops = (double)blocks * kPeakThreads * (double)iters * 16.0 * kChains;
  *ops_per_s = ops / (best * 1e-3);
  if (ms) *ms = best;
  return MPAP_OK;
}
