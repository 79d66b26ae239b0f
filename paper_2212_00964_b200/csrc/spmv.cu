// FP64 sparse matrix-vector products with the Krylov epilogues fused in.
//
// Reference being replaced: kernels._csr_matvec_nb (kernels.py:21-28, numba prange over
// rows, sequential per-row accumulation) and CsrMatrix.matvec/diagonal (sparse.py:32-51).
//
// Two storage views of the SAME CSR values array (bit-identical to the reference's
// `data`):
//  * FEM3 (vec = 3 FEM patterns): the three rows of node n are contiguous in `data`
//    (rows 3n..3n+2, each 3*cnt(n) long) and share one column-node list nbr[n].  A warp
//    streams the node's 9*cnt contiguous values (coalesced) and rebuilds the column as
//    3*nbr[j]+k, so the 4-byte column index is read once per 9 values:
//    8 + 4/9 bytes per nonzero instead of 12.
//  * CSR (any square matrix): LANES lanes per row, vector-CSR.
// Epilogues (all optional, chosen at compile time): Jacobi scaling y = D^-1 A x, the
// dot products BiCGSTAB needs right after each matvec (r0.v; t.t and t.s), and the
// explicit residual r = D^-1 (b - A x) with ||D r||^2 and ||r||^2 (solvers.py:115-116).
// Reductions use a fixed grid and a last-block finish -> deterministic.

#include "internal.cuh"

namespace b200 {

// Post-process row i's dot-product value `acc` for the mode; accumulate reduction terms.
template <int MODE>
__device__ __forceinline__ void spmv_epilogue(int64_t i, double acc, const SpmvArgs &a, double &red0,
                                              double &red1) {
  if (MODE == SP_PLAIN) {
    a.y[i] = acc;
  } else if (MODE == SP_JACOBI_R0) {
    const double v = a.inv[i] * acc;
    a.y[i] = v;
    red0 = fma(a.aux[i], v, red0);
  } else if (MODE == SP_JACOBI_TT) {
    const double t = a.inv[i] * acc;
    a.y[i] = t;
    red0 = fma(t, t, red0);
    red1 = fma(t, a.x[i], red1);
  } else {  // SP_RESIDUAL
    const double r = a.inv[i] * (a.aux[i] - acc);
    a.y[i] = r;
    a.aux2[i] = r;
    const double dr = a.dg[i] * r;
    red0 = fma(dr, dr, red0);
    red1 = fma(r, r, red1);
  }
}

// Scalar updates performed by the last block of a reduction launch.
template <int MODE>
__device__ __forceinline__ void spmv_stage(KrylovScalars *S, const double (&tot)[2]) {
  if (!S) return;
  if (MODE == SP_JACOBI_R0) {
    S->mv += 1;
    S->r0v = tot[0];
    if (tot[0] == 0.0) S->status = KS_BREAKDOWN;
    else S->alpha = S->rho / tot[0];
  } else if (MODE == SP_JACOBI_TT) {
    S->mv += 1;
    S->tt = tot[0];
    S->ts = tot[1];
    S->omega = tot[0] > 0.0 ? tot[1] / tot[0] : 0.0;
  } else if (MODE == SP_RESIDUAL) {
    S->mv += 1;
    S->res = sqrt(tot[0]);
    S->r0r0 = S->r0r = S->rr = tot[1];
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) k_spmv_fem3(const int32_t *__restrict__ nbr_ptr,
                                                        const int32_t *__restrict__ nbr,
                                                        const double *__restrict__ data, int64_t n_nodes,
                                                        SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double *__restrict__ x = a.x;
  double red0 = 0.0, red1 = 0.0;
  for (int64_t n = warp0; n < n_nodes; n += nwarps) {
    const int p0 = nbr_ptr[n];
    const int cnt = nbr_ptr[n + 1] - p0;
    const int L = 3 * cnt;
    const double *__restrict__ blk = data + 9 * (int64_t)p0;
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    if (cnt <= 32) {
      const int mine = lane < cnt ? nbr[p0 + lane] : 0;
      for (int e0 = 0; e0 < 3 * L; e0 += 32) {  // warp-uniform trip count: shuffles see all lanes
        const int e = e0 + lane;
        const bool ok = e < 3 * L;
        const int c = (e >= L) + (e >= 2 * L);
        const int r = e - c * L;
        const int j = ok ? r / 3 : 0;
        const int k = r - 3 * j;
        const int m = __shfl_sync(0xffffffffu, mine, j);
        if (ok) {
          const double prod = __ldg(blk + e) * __ldg(x + 3 * (int64_t)m + k);
          if (c == 0) y0 += prod;
          else if (c == 1) y1 += prod;
          else y2 += prod;
        }
      }
    } else {
      for (int e = lane; e < 3 * L; e += 32) {
        const int c = (e >= L) + (e >= 2 * L);
        const int r = e - c * L;
        const int j = r / 3;
        const int k = r - 3 * j;
        const int m = nbr[p0 + j];
        const double prod = __ldg(blk + e) * __ldg(x + 3 * (int64_t)m + k);
        if (c == 0) y0 += prod;
        else if (c == 1) y1 += prod;
        else y2 += prod;
      }
    }
    y0 = warp_sum(y0);
    y1 = warp_sum(y1);
    y2 = warp_sum(y2);
    if (lane < 3) {
      const double acc = lane == 0 ? y0 : (lane == 1 ? y1 : y2);
      spmv_epilogue<MODE>(3 * n + lane, acc, a, red0, red1);
    }
  }
  if (MODE != SP_PLAIN) {
    double v[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2>(v, red, tot) && threadIdx.x == 0) spmv_stage<MODE>(a.sc, tot);
  }
}

template <int MODE, int LANES>
__global__ void __launch_bounds__(kThreads) k_spmv_csr(const int32_t *__restrict__ indptr,
                                                       const int32_t *__restrict__ indices,
                                                       const double *__restrict__ data, int64_t n, SpmvArgs a,
                                                       RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LANES, sl = lane % LANES;
  constexpr int kPerWarp = 32 / LANES;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double red0 = 0.0, red1 = 0.0;
  for (int64_t base = warp0 * kPerWarp; base < n; base += nwarps * kPerWarp) {
    const int64_t row = base + sub;
    double acc = 0.0;
    if (row < n) {
      const int k1 = indptr[row + 1];
      for (int k = indptr[row] + sl; k < k1; k += LANES) acc = fma(__ldg(data + k), __ldg(a.x + indices[k]), acc);
    }
#pragma unroll
    for (int o = LANES / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < n && sl == 0) spmv_epilogue<MODE>(row, acc, a, red0, red1);
  }
  if (MODE != SP_PLAIN) {
    double v[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2>(v, red, tot) && threadIdx.x == 0) spmv_stage<MODE>(a.sc, tot);
  }
}

template <int MODE>
static void spmv_dispatch(const Matrix *m, const SpmvArgs &a, RedScratch *red) {
  const int grid = MODE == SP_PLAIN ? (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (m->n + 63) / 64)) : kRedBlocks;
  RedScratch r = red ? *red : RedScratch{};
  if (m->kind == MK_FEM3) {
    k_spmv_fem3<MODE><<<grid, kThreads, 0, m->stream>>>(m->nbr_ptr, m->nbr, m->data, m->n / 3, a, r);
  } else {
    switch (m->lanes) {
      case 4: k_spmv_csr<MODE, 4><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, m->n, a, r); break;
      case 8: k_spmv_csr<MODE, 8><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, m->n, a, r); break;
      case 16: k_spmv_csr<MODE, 16><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, m->n, a, r); break;
      default: k_spmv_csr<MODE, 32><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, m->n, a, r); break;
    }
  }
  count_launch();
}

int launch_spmv(const Matrix *m, SpmvMode mode, const SpmvArgs &a, RedScratch *red) {
  switch (mode) {
    case SP_PLAIN: spmv_dispatch<SP_PLAIN>(m, a, red); break;
    case SP_JACOBI_R0: spmv_dispatch<SP_JACOBI_R0>(m, a, red); break;
    case SP_JACOBI_TT: spmv_dispatch<SP_JACOBI_TT>(m, a, red); break;
    default: spmv_dispatch<SP_RESIDUAL>(m, a, red); break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

// diagonal (sparse.py:44-51: 0 where the row has no diagonal entry), its inverse and the
// number of zero entries (solvers.py:101-103)
__global__ void __launch_bounds__(kThreads) k_diagonal(const int32_t *__restrict__ indptr,
                                                       const int32_t *__restrict__ indices,
                                                       const int32_t *__restrict__ slots,
                                                       const double *__restrict__ data, int64_t n, double *diag,
                                                       double *inv, RedScratch red) {
  double zeros[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    if (slots) {
      d = data[slots[i]];
    } else {
      int lo = indptr[i], hi = indptr[i + 1];
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (indices[mid] < i) lo = mid + 1; else hi = mid;
      }
      if (lo < indptr[i + 1] && indices[lo] == i) d = data[lo];
    }
    diag[i] = d;
    inv[i] = 1.0 / d;
    zeros[0] += (d == 0.0) ? 1.0 : 0.0;
  }
  double tot[1];
  block_partials_and_finish<1>(zeros, red, tot);
}

int launch_diagonal(const Matrix *m, double *diag, double *inv, RedScratch *red, int64_t *n_zero) {
  k_diagonal<<<kRedBlocks, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->diag_slots, m->data, m->n, diag, inv,
                                                     *red);
  count_launch();
  if (n_zero) {
    double z = 0.0;
    B200_CUDA(cudaMemcpyAsync(&z, red->result, sizeof(double), cudaMemcpyDeviceToHost, m->stream));
    B200_CUDA(cudaStreamSynchronize(m->stream));
    *n_zero = (int64_t)z;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

}  // namespace b200
