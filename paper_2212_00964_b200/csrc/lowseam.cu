// The reference's low seam (SURVEY §8(b) seam 1): gradfem.kernels.csr_matvec and
// scatter_add (kernels.py:21-55), which the reference's assembly and Krylov code call and its
// tests monkeypatch.  Both keep the reference's accumulation order exactly:
//
// * csr_matvec: y_i = ((0 + d_k0 x_c0) + d_k1 x_c1) + ... in storage order, one rounded
//   multiply and one rounded add per term (numba does not contract to FMA), so y is
//   bit-identical to the numba kernel for any matrix.  A thread per row: this seam serves
//   user-built matrices; the Newton operators have their own layouts (spmv.cu).
// * scatter_add: values[dest[k]] += contribs[k] in ascending k.  Per destination that is a
//   fixed left-to-right sum starting from the old value, so a stable radix sort of (dest, k)
//   followed by one sequential sum per destination run reproduces the sequential loop bit
//   for bit, with all destinations in parallel.

#include <cub/cub.cuh>

#include "internal.cuh"

namespace b200 {

__global__ void k_csr_matvec_seq(int64_t n, const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                                 const double *__restrict__ data, const double *__restrict__ x,
                                 double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = __ldg(indptr + i), k1 = __ldg(indptr + i + 1); k < k1; ++k)
      acc = __dadd_rn(acc, __dmul_rn(__ldg(data + k), __ldg(x + __ldg(indices + k))));
    y[i] = acc;
  }
}

__global__ void k_iota(int64_t n, int64_t *__restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    ids[i] = i;
}

// one thread per run of equal destinations in the sorted order
__global__ void k_scatter_runs(int64_t n, const int64_t *__restrict__ sdest, const int64_t *__restrict__ sid,
                               const double *__restrict__ contribs, double *__restrict__ values) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = sdest[i];
    if (i > 0 && sdest[i - 1] == d) continue;
    double v = values[d];
    for (int64_t j = i; j < n && sdest[j] == d; ++j) v = __dadd_rn(v, __ldg(contribs + sid[j]));
    values[d] = v;
  }
}

__global__ void k_dest_range(int64_t n, const int64_t *__restrict__ dest, int64_t n_values, int *__restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (dest[i] < 0 || dest[i] >= n_values) atomicExch(bad, 1);
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (n + kThreads - 1) / kThreads)); }

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_csr_matvec_seq(int64_t n, const int32_t *indptr, const int32_t *indices, const double *data,
                           const double *x, double *y, void *stream) {
  if (n <= 0) return 0;
  k_csr_matvec_seq<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, indptr, indices, data, x, y);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int b200fem_scatter_add(double *values, int64_t n_values, const int64_t *dest, const double *contribs, int64_t n,
                        void *stream, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (n <= 0) return 0;
  if (n > INT32_MAX) {  // cub's item count
    set_err(err, B200FEM_E_INVALID, "scatter_add: more than 2^31-1 contributions per call");
    return B200FEM_E_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *ids = nullptr, *sdest = nullptr, *sid = nullptr;
  int *bad = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = B200FEM_E_CUDA;
  int end_bit = 1;
  while (end_bit < 63 && (int64_t(1) << end_bit) < n_values) ++end_bit;
  do {
    if (cudaMalloc((void **)&ids, n * sizeof(int64_t)) || cudaMalloc((void **)&sdest, n * sizeof(int64_t)) ||
        cudaMalloc((void **)&sid, n * sizeof(int64_t)) || cudaMalloc((void **)&bad, sizeof(int)))
      break;
    if (cudaMemsetAsync(bad, 0, sizeof(int), s)) break;
    k_dest_range<<<grid_for(n), kThreads, 0, s>>>(n, dest, n_values, bad);
    int hbad = 0;
    if (cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s)) break;
    if (hbad) {
      set_err(err, B200FEM_E_INVALID, "scatter_add: destination index out of range [0, %lld)", (long long)n_values);
      rc = B200FEM_E_INVALID;
      break;
    }
    k_iota<<<grid_for(n), kThreads, 0, s>>>(n, ids);
    // LSD radix sort: stable, so equal destinations keep ascending k
    if (cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dest, sdest, ids, sid, (int)n, 0, end_bit, s)) break;
    if (cudaMalloc(&tmp, tmp_bytes)) break;
    if (cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dest, sdest, ids, sid, (int)n, 0, end_bit, s)) break;
    k_scatter_runs<<<grid_for(n), kThreads, 0, s>>>(n, sdest, sid, contribs, values);
    count_launch(4);
    if (cudaStreamSynchronize(s) || cudaGetLastError()) break;
    rc = 0;
  } while (false);
  if (rc == B200FEM_E_CUDA) set_err(err, rc, "scatter_add: %s", cudaGetErrorString(cudaGetLastError()));
  cudaFree(tmp);
  cudaFree(ids);
  cudaFree(sdest);
  cudaFree(sid);
  cudaFree(bad);
  return rc;
}

}  // extern "C"
