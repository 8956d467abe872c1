// paper_1705_02408_b200/csrc/rowshard.cu -- device-resident row blocks of a
// row-sharded roadmap build ("rank g builds rows [g n/G,
// (g+1) n/G) ... one all-gather of the CSR blocks"; "embarrassingly
// parallel").
//
//   mpap_roadmap_block_device   a rank's block as device arrays (row counts +
//                               16-byte edge records), ready for one NCCL
//                               all-gather without a host round trip;
//   mpap_roadmap_assemble_device  the gathered blocks -> a search roadmap:
//                               one scan of the concatenated row counts and
//                               one copy kernel placing every block's records
//                               at its row offset (the device counterpart of
//                               mpap_roadmap_import).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "mpap_internal.cuh"

namespace mpap {
namespace {

__global__ void k_block_counts(const int64_t* __restrict__ row_ptr, int64_t row_lo, int64_t rows,
                               int32_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) counts[i] = (int32_t)(row_ptr[row_lo + i + 1] - row_ptr[row_lo + i]);
}

// concatenated row counts of the gathered blocks (block b's rows first in its slot)
__global__ void k_gather_counts(const int32_t* __restrict__ counts, int32_t stride,
                                const int32_t* __restrict__ row_begin, int32_t n_blocks, int32_t n,
                                int32_t* __restrict__ cnt) {
  const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  int lo = 0, hi = n_blocks;   // block b with row_begin[b] <= u < row_begin[b + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (row_begin[mid] <= u) lo = mid; else hi = mid;
  }
  cnt[u] = counts[(size_t)lo * stride + (u - row_begin[lo])];
}

// every output edge e: its block (by the row offsets at the block starts),
// the record at the same position within that block's slot; dst range check
// and collision-free count on the way
__global__ void k_assemble_edges(const EdgeRec* __restrict__ edges, int64_t stride,
                                 const int32_t* __restrict__ row_begin, int32_t n_blocks, int32_t n,
                                 const int64_t* __restrict__ row_ptr, int64_t nnz, EdgeRec* __restrict__ out,
                                 unsigned long long* __restrict__ nfree, int* __restrict__ bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned fr = 0;
  if (e < nnz) {
    int lo = 0, hi = n_blocks;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (row_ptr[row_begin[mid]] <= e) lo = mid; else hi = mid;
    }
    const EdgeRec r = edges[(size_t)lo * stride + (e - row_ptr[row_begin[lo]])];
    if ((int64_t)(r.dst_coll & 0x7fffffffu) >= n) atomicOr(bad, 1);
    out[e] = r;
    fr = (r.dst_coll >> 31) == 0u ? 1u : 0u;
  }
  fr = __reduce_add_sync(0xffffffffu, fr);
  if ((threadIdx.x & 31) == 0 && fr) atomicAdd(nfree, (unsigned long long)fr);
}

}  // namespace
}  // namespace mpap

using namespace mpap;

#define CKR(x)                                          \
  do {                                                  \
    cudaError_t _e = (x);                               \
    if (_e != cudaSuccess) return cuda_error(_e, #x);   \
  } while (0)

extern "C" {

mpap_status mpap_roadmap_block_device(const mpap_roadmap* rm, int32_t* counts, void* edges, int64_t capacity,
                                      int64_t* nnz, void* cuda_stream) {
  if (!rm || !counts || !nnz || capacity < 0 || (capacity > 0 && !edges))
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL argument or capacity < 0");
  if (rm->B != 1 || !rm->d_row_ptr) return set_error(MPAP_ERR_INVALID_ARGUMENT, "needs a one-environment build");
  if (rm->lazy) return set_error(MPAP_ERR_INVALID_ARGUMENT, "lazy roadmaps have no block to export");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != rm->device) return set_error(MPAP_ERR_INVALID_ARGUMENT, "roadmap bound to another device");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int64_t lo = std::max<int64_t>(0, rm->prm.row_lo), hi = std::min<int64_t>(rm->n[0], rm->prm.row_hi);
  const int64_t rows = std::max<int64_t>(0, hi - lo);
  int64_t e0 = 0, e1 = 0;
  if (rows > 0) {
    CKR(cudaMemcpyAsync(&e0, rm->d_row_ptr + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CKR(cudaMemcpyAsync(&e1, rm->d_row_ptr + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CKR(cudaStreamSynchronize(st));
  }
  *nnz = e1 - e0;
  if (*nnz > capacity) return set_error(MPAP_ERR_BUFFER_TOO_SMALL, "edge capacity below the block's records");
  if (rows > 0) {
    k_block_counts<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(rm->d_row_ptr, lo, rows, counts);
    note_launch();
    CKR(cudaGetLastError());
    if (*nnz > 0)
      CKR(cudaMemcpyAsync(edges, rm->d_edges + e0, sizeof(EdgeRec) * (size_t)*nnz, cudaMemcpyDeviceToDevice, st));
  }
  CKR(cudaStreamSynchronize(st));
  return MPAP_OK;
}

mpap_status mpap_roadmap_assemble_device(int32_t n, int32_t pos_dim, const double* positions, int32_t n_blocks,
                                         const int32_t* row_begin, const int32_t* counts, int32_t counts_stride,
                                         const void* edges, int64_t edges_stride, double r, void* cuda_stream,
                                         mpap_roadmap** out) {
  if (!out) return set_error(MPAP_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n < 1 || (pos_dim != 2 && pos_dim != 3) || !positions || n_blocks < 1 || !row_begin || !counts ||
      counts_stride < 0 || edges_stride < 0)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "bad n/pos_dim/positions/blocks");
  if (!(r > 0.0) || !std::isfinite(r)) return set_error(MPAP_ERR_INVALID_ARGUMENT, "r must be finite and > 0");
  if (row_begin[0] != 0 || row_begin[n_blocks] != n)
    return set_error(MPAP_ERR_INVALID_ARGUMENT, "row blocks must tile [0, n)");
  for (int32_t b = 0; b < n_blocks; ++b)
    if (row_begin[b + 1] < row_begin[b] || row_begin[b + 1] - row_begin[b] > counts_stride)
      return set_error(MPAP_ERR_INVALID_ARGUMENT, "row blocks decreasing or wider than counts_stride");
  for (int64_t k = 0; k < (int64_t)n * pos_dim; ++k)
    if (!std::isfinite(positions[k])) return set_error(MPAP_ERR_INVALID_ARGUMENT, "non-finite position");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  mpap_roadmap* rm = new (std::nothrow) mpap_roadmap();
  if (!rm) return set_error(MPAP_ERR_OUT_OF_MEMORY, "host allocation failed");
  auto fail = [&](mpap_status s) {
    mpap_roadmap_free(rm);
    return s;
  };
  cudaError_t ce = cudaGetDevice(&rm->device);
  if (ce != cudaSuccess) return fail(cuda_error(ce, "cudaGetDevice"));
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
  rm->n_max = n;
  int32_t* d_rb = nullptr;
  int32_t* d_cnt = nullptr;
  unsigned long long* d_nfree = nullptr;
  int* d_bad = nullptr;
  rm->d_samples = static_cast<double*>(rm_alloc(sizeof(double) * (size_t)n * pos_dim, st));
  rm->d_node_base = static_cast<int64_t*>(rm_alloc(sizeof(int64_t) * 2, st));
  rm->d_row_ptr = static_cast<int64_t*>(rm_alloc(sizeof(int64_t) * ((size_t)n + 1), st));
  if (!rm->d_samples || !rm->d_node_base || !rm->d_row_ptr)
    return fail(set_error(MPAP_ERR_OUT_OF_MEMORY, "roadmap allocation failed"));
  ce = cudaMemcpyAsync(rm->d_samples, positions, sizeof(double) * (size_t)n * pos_dim, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(rm->d_node_base, rm->node_base.data(), sizeof(int64_t) * 2, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&d_rb, sizeof(int32_t) * (n_blocks + 1), st);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&d_cnt, sizeof(int32_t) * (size_t)n, st);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&d_nfree, sizeof(unsigned long long), st);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&d_bad, sizeof(int), st);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(d_rb, row_begin, sizeof(int32_t) * (n_blocks + 1), cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(d_nfree, 0, sizeof(unsigned long long), st);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(d_bad, 0, sizeof(int), st);
  if (ce != cudaSuccess) return fail(cuda_error(ce, "assemble setup"));
  k_gather_counts<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(counts, counts_stride, d_rb, n_blocks, n, d_cnt);
  note_launch();
  ce = scan_row_counts(d_cnt, n, rm->d_row_ptr, st);
  if (ce != cudaSuccess) return fail(cuda_error(ce, "row scan"));
  int64_t nnz = 0;
  ce = cudaMemcpyAsync(&nnz, rm->d_row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return fail(cuda_error(ce, "row scan"));
  // every block's records must fit its slot
  std::vector<int64_t> rp_b(n_blocks + 1);
  for (int32_t b = 0; b <= n_blocks; ++b) {
    ce = cudaMemcpyAsync(&rp_b[b], rm->d_row_ptr + row_begin[b], sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (ce != cudaSuccess) return fail(cuda_error(ce, "block offsets"));
  }
  ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return fail(cuda_error(ce, "block offsets"));
  for (int32_t b = 0; b < n_blocks; ++b)
    if (rp_b[b + 1] - rp_b[b] > edges_stride)
      return fail(set_error(MPAP_ERR_INVALID_ARGUMENT, "a block's edge count exceeds edges_stride"));
  if (nnz > 0 && !edges) return fail(set_error(MPAP_ERR_INVALID_ARGUMENT, "NULL edges"));
  rm->d_edges = static_cast<EdgeRec*>(rm_alloc(sizeof(EdgeRec) * (size_t)std::max<int64_t>(nnz, 1), st));
  if (!rm->d_edges) return fail(set_error(MPAP_ERR_OUT_OF_MEMORY, "edge allocation failed"));
  if (nnz > 0) {
    k_assemble_edges<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(static_cast<const EdgeRec*>(edges), edges_stride,
                                                                    d_rb, n_blocks, n, rm->d_row_ptr, nnz,
                                                                    rm->d_edges, d_nfree, d_bad);
    note_launch();
  }
  unsigned long long nfree = 0;
  int bad = 0;
  ce = cudaMemcpyAsync(&nfree, d_nfree, sizeof(nfree), cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaFreeAsync(d_rb, st);
  if (ce == cudaSuccess) ce = cudaFreeAsync(d_cnt, st);
  if (ce == cudaSuccess) ce = cudaFreeAsync(d_nfree, st);
  if (ce == cudaSuccess) ce = cudaFreeAsync(d_bad, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return fail(cuda_error(ce, "assemble"));
  if (bad) return fail(set_error(MPAP_ERR_INVALID_ARGUMENT, "dst out of range in a gathered block"));
  rm->edge_base = {0, nnz};
  rm->nnz_total = nnz;
  rm->nnz_free.assign(1, (int64_t)nfree);
  *out = rm;
  return MPAP_OK;
}

}  // extern "C"
