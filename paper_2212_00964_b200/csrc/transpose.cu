// Explicit transposes for the adjoint solve.
//
// Reference: CsrMatrix.transpose (sparse.py:53-62) sorts the entries stably by column,
// so row r of A^T lists the rows of A that hold column r, ascending, with the same values.
//
// * FEM workspaces: the pattern is structurally symmetric (node adjacency), so A^T has
//   exactly A's indptr/indices and only the values move: entry (3n+c, 3m+k) of A^T is
//   entry (3m+k, 3n+c) of A.  One warp per node, one lane per neighbour m; the lane finds
//   n in m's sorted neighbour list by binary search and copies the transposed 3x3 block.
//   A pure permutation, so the values are bit-identical to the reference's transpose.
// * Generic CSR (user-built CsrMatrix): column histogram -> scan -> indptr_t, then a stable
//   radix sort of the column keys carries the entry ids (cub, LSD radix: stable), and the
//   rows / values are gathered through the permutation.  Same result as the reference's
//   stable argsort.

#include <cub/cub.cuh>

#include "internal.cuh"

namespace b200 {

template <int VEC>
__global__ void k_transpose_fem(const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr,
                                const double *__restrict__ A, double *__restrict__ At, int64_t n_nodes) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = w0; n < n_nodes; n += nw) {
    const int p0 = __ldg(nbr_ptr + n), cn = __ldg(nbr_ptr + n + 1) - p0;
    for (int j = lane; j < cn; j += 32) {
      const int m = __ldg(nbr + p0 + j);
      const int q0 = __ldg(nbr_ptr + m), cm = __ldg(nbr_ptr + m + 1) - q0;
      int lo = 0, hi = cm - 1;  // n is in m's list (symmetric adjacency)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(nbr + q0 + mid) < n) lo = mid + 1;
        else hi = mid;
      }
      if (VEC == 1) {
        At[p0 + j] = A[q0 + lo];
      } else {
        const double *src = A + 9 * (int64_t)q0;
        double *dst = At + 9 * (int64_t)p0;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int k = 0; k < 3; ++k) dst[3 * c * cn + 3 * j + k] = src[3 * k * cm + 3 * lo + c];
      }
    }
  }
}

__global__ void k_col_count(const int32_t *__restrict__ indices, int64_t nnz, int32_t *__restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + indices[i], 1);
}

__global__ void k_rows_iota(const int32_t *__restrict__ indptr, int64_t n, int32_t *__restrict__ rows,
                            int32_t *__restrict__ ids) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    for (int k = indptr[r]; k < indptr[r + 1]; ++k) rows[k] = (int32_t)r, ids[k] = k;
}

__global__ void k_permute(const int32_t *__restrict__ order, const int32_t *__restrict__ rows,
                          const double *__restrict__ data, int64_t nnz, int32_t *__restrict__ indices_t,
                          double *__restrict__ data_t) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = order[i];
    indices_t[i] = rows[o];
    data_t[i] = data[o];
  }
}

static int grid_for(int64_t items) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (items + kThreads - 1) / kThreads));
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_transpose_fem(b200fem_ctx *ctx, const double *data, double *data_t) {
  Ctx *c = (Ctx *)ctx;
  if (!c || !data || !data_t || data == data_t) return B200FEM_E_INVALID;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (c->n_nodes + 7) / 8));
  if (c->vec == 3)
    k_transpose_fem<3><<<g, 256, 0, c->stream>>>(c->nbr_ptr, c->nbr, data, data_t, c->n_nodes);
  else
    k_transpose_fem<1><<<g, 256, 0, c->stream>>>(c->nbr_ptr, c->nbr, data, data_t, c->n_nodes);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int b200fem_csr_transpose(int64_t n, int64_t nnz, const int32_t *indptr, const int32_t *indices, const double *data,
                          int32_t *indptr_t, int32_t *indices_t, double *data_t, void *stream) {
  if (n < 0 || nnz < 0 || nnz >= (int64_t)INT32_MAX || n >= (int64_t)INT32_MAX) return B200FEM_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  B200_CUDA(cudaMemsetAsync(indptr_t, 0, (n + 1) * sizeof(int32_t), s));
  if (n == 0 || nnz == 0) return cudaStreamSynchronize(s) == cudaSuccess ? 0 : B200FEM_E_CUDA;
  int32_t *cnt = nullptr, *rows = nullptr, *ids = nullptr, *keys_out = nullptr, *order = nullptr;
  void *tmp = nullptr;
  int st = B200FEM_E_CUDA;
  int end_bit = 1;
  while (end_bit < 31 && (int64_t(1) << end_bit) < n) ++end_bit;
  size_t scan_bytes = 0, sort_bytes = 0;
  do {
    if (dalloc(&cnt, n + 1) || dalloc(&rows, nnz) || dalloc(&ids, nnz) || dalloc(&keys_out, nnz) ||
        dalloc(&order, nnz))
      break;
    if (cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int32_t), s)) break;
    k_col_count<<<grid_for(nnz), kThreads, 0, s>>>(indices, nnz, cnt);
    k_rows_iota<<<grid_for(n), kThreads, 0, s>>>(indptr, n, rows, ids);
    count_launch(2);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, indptr_t, (int)(n + 1), s);
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, indices, keys_out, ids, order, (int)nnz, 0, end_bit, s);
    if (cudaMalloc(&tmp, std::max(scan_bytes, sort_bytes))) break;
    if (cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, cnt, indptr_t, (int)(n + 1), s)) break;
    if (cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, indices, keys_out, ids, order, (int)nnz, 0, end_bit, s))
      break;
    k_permute<<<grid_for(nnz), kThreads, 0, s>>>(order, rows, data, nnz, indices_t, data_t);
    count_launch();
    if (cudaStreamSynchronize(s) != cudaSuccess) break;
    st = 0;
  } while (false);
  cudaFree(tmp);
  cudaFree(cnt);
  cudaFree(rows);
  cudaFree(ids);
  cudaFree(keys_out);
  cudaFree(order);
  return st;
}

}  // extern "C"
