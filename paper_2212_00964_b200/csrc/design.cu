// Design-loop vector kernels: the density filter as a device CSR, the
// filtered sensitivities, and the MMA update (reference inverse.py:186-346).
//
// Density filter (inverse.py:200-228).  Element centroids are the sequential mean of the 8
// vertex coordinates (numpy's reduction order for cell_coords().mean(axis=1)).  Neighbours
// within the radius come from a uniform bin grid (bin edge >= radius, so the 27 surrounding
// bins cover the ball): cells are sorted by bin key once (cub radix sort), each row then
// scans its 27 bins with binary searches, counts (pass 1) and fills (pass 2) its neighbours,
// and sorts them ascending in place.  Weights w = max(r - |c_j - c_i|, 0) with the distance
// summed as numpy does ((0 + dx^2) + dy^2) + dz^2, normalised by numpy's pairwise sum, so
// the CSR matches the reference's cKDTree construction value for value.
//
// Filter application is a row-sequential CSR product (acc += a_k * v_j, no FMA: the
// reference's numba matvec order, kernels.py:21-28) with optional fused elementwise
// pre-multiply and post-division, which is exactly filter_sensitivities (inverse.py:231-234).
//
// MMA (inverse.py:260-346).  All per-variable arithmetic uses explicitly rounded operations
// (no contraction), so x_of(y) reproduces the reference bit for bit for a given multiplier
// y.  The outer dual search (one doubling phase, then 100 bisection steps on y) runs as a
// device state machine: each launch evaluates g(x_of(y)) with a deterministic reduction
// and the last block advances the state, so a whole update is one stream of launches with
// no host round trip.

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.cuh"

namespace b200 {

// ------------------------------------------------------------------ filter
__global__ void k_centroids(const double *__restrict__ X, const int32_t *__restrict__ cells, int64_t n,
                            double *__restrict__ cent) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = cells[e * 8 + k];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double s = X[(int64_t)v[0] * 3 + d];
#pragma unroll
      for (int k = 1; k < 8; ++k) s = __dadd_rn(s, X[(int64_t)v[k] * 3 + d]);
      cent[e * 3 + d] = s / 8.0;
    }
  }
}

__device__ __forceinline__ unsigned long long ord_u(double x) {  // order-preserving bits
  const unsigned long long b = __double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_u(unsigned long long u) {
  return __longlong_as_double((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u);
}

__global__ void k_bbox(const double *__restrict__ cent, int64_t n, unsigned long long *__restrict__ bb) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const unsigned long long u = ord_u(cent[e * 3 + d]);
      lo[d] = min(lo[d], u);
      hi[d] = max(hi[d], u);
    }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    for (int o = 16; o; o >>= 1) {
      lo[d] = min(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = max(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(bb + d, lo[d]);
      atomicMax(bb + 3 + d, hi[d]);
    }
  }
}

static double host_unord(unsigned long long u) {
  const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
  double d;
  memcpy(&d, &b, sizeof(d));
  return d;
}

struct BinGrid {
  double org[3];
  double h;
  int64_t dims[3];
};

__device__ __forceinline__ int64_t bin_coord(double c, double org, double h, int64_t dim) {
  int64_t b = (int64_t)floor((c - org) / h);
  return b < 0 ? 0 : (b >= dim ? dim - 1 : b);
}

__global__ void k_bin_keys(const double *__restrict__ cent, int64_t n, BinGrid g, int64_t *__restrict__ key,
                           int32_t *__restrict__ ids) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) b[d] = bin_coord(cent[e * 3 + d], g.org[d], g.h, g.dims[d]);
    key[e] = (b[2] * g.dims[1] + b[1]) * g.dims[0] + b[0];
    ids[e] = (int32_t)e;
  }
}

__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ int64_t lower_key(const int64_t *__restrict__ k, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (k[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ double cdist(const double *__restrict__ cent, int64_t i, int64_t j) {
  const double dx = cent[j * 3] - cent[i * 3], dy = cent[j * 3 + 1] - cent[i * 3 + 1],
               dz = cent[j * 3 + 2] - cent[i * 3 + 2];
  double s = __dadd_rn(0.0, __dmul_rn(dx, dx));
  s = __dadd_rn(s, __dmul_rn(dy, dy));
  s = __dadd_rn(s, __dmul_rn(dz, dz));
  return sqrt(s);
}

// PASS 0: count neighbours of each cell; PASS 1: write them (unsorted) into the row.
template <int PASS>
__global__ void k_filter_rows(const double *__restrict__ cent, int64_t n, BinGrid g, double r,
                              const int64_t *__restrict__ skey, const int32_t *__restrict__ sid,
                              int32_t *__restrict__ cnt, const int32_t *__restrict__ indptr,
                              int32_t *__restrict__ indices, double *__restrict__ dist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) b[d] = bin_coord(cent[i * 3 + d], g.org[d], g.h, g.dims[d]);
    int c = 0;
    int64_t w = PASS ? indptr[i] : 0;
    for (int64_t bz = imax(b[2] - 1, 0); bz <= imin(b[2] + 1, g.dims[2] - 1); ++bz)
      for (int64_t by = imax(b[1] - 1, 0); by <= imin(b[1] + 1, g.dims[1] - 1); ++by) {
        // the x-range of bins in this (by, bz) row is one contiguous key range
        const int64_t k0 = (bz * g.dims[1] + by) * g.dims[0] + imax(b[0] - 1, 0);
        const int64_t k1 = (bz * g.dims[1] + by) * g.dims[0] + imin(b[0] + 1, g.dims[0] - 1);
        for (int64_t p = lower_key(skey, n, k0); p < n && skey[p] <= k1; ++p) {
          const int32_t j = sid[p];
          const double dd = cdist(cent, i, j);
          if (dd <= r) {
            if (PASS) {
              indices[w] = j;
              dist[w] = dd;
              ++w;
            }
            ++c;
          }
        }
      }
    if (!PASS) cnt[i] = c;
  }
}

// numpy's pairwise summation (umath loops: pairwise_sum, PW_BLOCKSIZE 128) of a[0..n).
__device__ double np_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// sort each row's neighbours ascending (insertion sort: rows are short), then weights.
__global__ void k_filter_finish(int64_t n, double r, const int32_t *__restrict__ indptr, int32_t *__restrict__ indices,
                                double *__restrict__ dist, double *__restrict__ data) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = indptr[i], b = indptr[i + 1];
    for (int64_t p = a + 1; p < b; ++p) {
      const int32_t kj = indices[p];
      const double kd = dist[p];
      int64_t q = p - 1;
      while (q >= a && indices[q] > kj) {
        indices[q + 1] = indices[q];
        dist[q + 1] = dist[q];
        --q;
      }
      indices[q + 1] = kj;
      dist[q + 1] = kd;
    }
    for (int64_t p = a; p < b; ++p) {
      const double w = r - dist[p];
      data[p] = w > 0.0 ? w : 0.0;
    }
    const double total = np_pairwise_sum(data + a, b - a);
    for (int64_t p = a; p < b; ++p) data[p] = data[p] / total;
  }
}

// y_i = (sum_k a_k (v_j [* m_j])) [/ max(dv_i, floor)], row-sequential, no contraction.
__global__ void k_filter_apply(int64_t n, const int32_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                               const double *__restrict__ data, const double *__restrict__ v,
                               const double *__restrict__ m, const double *__restrict__ dv, double floor_v,
                               double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = indptr[i], k1 = indptr[i + 1]; k < k1; ++k) {
      const int j = indices[k];
      const double xv = m ? __dmul_rn(v[j], m[j]) : v[j];
      acc = __dadd_rn(acc, __dmul_rn(data[k], xv));
    }
    if (dv) {
      const double t = dv[i];
      acc = acc / (t > floor_v ? t : floor_v);
    }
    y[i] = acc;
  }
}

struct Filter {
  int64_t n = 0, nnz = 0;
  double radius = 0.0;
  cudaStream_t stream = nullptr;
  int32_t *indptr = nullptr, *indices = nullptr;
  double *data = nullptr;
};

static int grid_n(int64_t items) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (items + kThreads - 1) / kThreads));
}

// ------------------------------------------------------------------ MMA
struct MmaCtl {
  int stage;  // 0: test y=0, 1: doubling, 2: bisection, 3: done
  int k;      // bisection steps taken
  double y_lo, y_hi, y_final, g_value;
  unsigned long long absmax;  // ordered bits of max |dj|
};

__global__ void k_mma_absmax(int64_t n, const double *__restrict__ dj, MmaCtl *ctl) {
  unsigned long long m = 0ull;  // ord_u(+0.0) > ord_u of any negative; |dj| >= 0
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, ord_u(fabs(dj[i])));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&ctl->absmax, m);
}

struct MmaArgs {
  const double *x, *dj, *c, *lb, *ub, *xp, *xpp;
  double *low, *upp, *alpha, *beta, *p0, *q0, *xnew;
  double asym_init, asym_expand, asym_shrink, move_limit;
  int use_hist;
};

__global__ void k_mma_prep(int64_t n, MmaArgs a, const MmaCtl *ctl) {
  const double mx = n > 0 ? unord_u(ctl->absmax) : 0.0;
  const double eps = __dmul_rn(1e-9, mx > 1.0 ? mx : 1.0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a.x[i], lb = a.lb[i], ub = a.ub[i];
    const double rng = __dsub_rn(ub, lb);
    double low, upp;
    if (!a.use_hist) {
      low = __dsub_rn(x, __dmul_rn(a.asym_init, rng));
      upp = __dadd_rn(x, __dmul_rn(a.asym_init, rng));
    } else {
      const double xp = a.xp[i], xpp = a.xpp[i];
      const double osc = __dmul_rn(__dsub_rn(x, xp), __dsub_rn(xp, xpp));
      const double sc = osc < 0.0 ? a.asym_shrink : (osc > 0.0 ? a.asym_expand : 1.0);
      low = __dsub_rn(x, __dmul_rn(sc, __dsub_rn(xp, a.low[i])));
      upp = __dadd_rn(x, __dmul_rn(sc, __dsub_rn(a.upp[i], xp)));
      const double l0 = __dsub_rn(x, __dmul_rn(10.0, rng)), l1 = __dsub_rn(x, __dmul_rn(0.01, rng));
      const double u0 = __dadd_rn(x, __dmul_rn(0.01, rng)), u1 = __dadd_rn(x, __dmul_rn(10.0, rng));
      low = fmin(fmax(low, l0), l1);  // np.clip(low, l0, l1)
      upp = fmin(fmax(upp, u0), u1);
    }
    const double mv = __dmul_rn(a.move_limit, rng);
    double al = fmax(fmax(lb, __dadd_rn(low, __dmul_rn(0.1, __dsub_rn(x, low)))), __dsub_rn(x, mv));
    double be = fmin(fmin(ub, __dsub_rn(upp, __dmul_rn(0.1, __dsub_rn(upp, x)))), __dadd_rn(x, mv));
    const double ux = __dsub_rn(upp, x), xl = __dsub_rn(x, low);
    const double dj = a.dj[i];
    a.p0[i] = __dmul_rn(__dmul_rn(ux, ux), __dadd_rn(dj > 0.0 ? dj : 0.0, eps));
    a.q0[i] = __dmul_rn(__dmul_rn(xl, xl), __dadd_rn(-dj > 0.0 ? -dj : 0.0, eps));
    a.low[i] = low;
    a.upp[i] = upp;
    a.alpha[i] = al;
    a.beta[i] = be;
  }
}

__device__ __forceinline__ double mma_phi(double t, double p0, double q0, double low, double upp, double y, double c) {
  const double u = __dsub_rn(upp, t), l = __dsub_rn(t, low);
  return __dadd_rn(__dsub_rn(p0 / __dmul_rn(u, u), q0 / __dmul_rn(l, l)), __dmul_rn(y, c));
}

__device__ __forceinline__ double mma_x_of(double y, double al, double be, double p0, double q0, double low,
                                           double upp, double c) {
  if (mma_phi(al, p0, q0, low, upp, y, c) >= 0.0) return al;
  const bool at_hi = mma_phi(be, p0, q0, low, upp, y, c) <= 0.0;
  double lo = al, hi = be;
  for (int it = 0; it < 80; ++it) {
    const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
    if (mma_phi(mid, p0, q0, low, upp, y, c) < 0.0) lo = mid;
    else hi = mid;
  }
  return at_hi ? be : __dmul_rn(0.5, __dadd_rn(lo, hi));
}

// One dual evaluation: g(x_of(y)) = g_value + c . (x_of(y) - x); the last block advances the
// state machine.  FINAL: write x_of(y_final).
template <bool FINAL>
__global__ void __launch_bounds__(kThreads) k_mma_eval(int64_t n, MmaArgs a, MmaCtl *ctl, RedScratch red) {
  const int stage = ctl->stage;
  if (FINAL ? stage != 3 : stage == 3) return;
  const double y = FINAL ? ctl->y_final
                         : stage == 0 ? 0.0 : stage == 1 ? ctl->y_hi : __dmul_rn(0.5, __dadd_rn(ctl->y_lo, ctl->y_hi));
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double c = a.c[i];
    const double xv = mma_x_of(y, a.alpha[i], a.beta[i], a.p0[i], a.q0[i], a.low[i], a.upp[i], c);
    if (FINAL) a.xnew[i] = xv;
    else acc[0] = __dadd_rn(acc[0], __dmul_rn(c, __dsub_rn(xv, a.x[i])));
  }
  if (FINAL) return;
  double tot[1];
  if (!block_partials_and_finish<1>(acc, red, tot) || threadIdx.x != 0) return;
  const double g = __dadd_rn(ctl->g_value, tot[0]);
  if (stage == 0) {
    if (g <= 0.0) ctl->stage = 3, ctl->y_final = 0.0;
    else ctl->stage = 1, ctl->y_hi = 1.0;
  } else if (stage == 1) {
    if (g > 0.0 && ctl->y_hi < 1e12) ctl->y_hi = __dmul_rn(ctl->y_hi, 2.0);
    else ctl->stage = 2, ctl->y_lo = 0.0, ctl->k = 0;
  } else {
    if (g > 0.0) ctl->y_lo = y;
    else ctl->y_hi = y;
    if (++ctl->k == 100) ctl->stage = 3, ctl->y_final = ctl->y_hi;
  }
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_filter_create(b200fem_filter **out, int64_t n_cells, const double *coords_dev, const int32_t *cells_dev,
                          double radius, void *stream) {
  if (!out || n_cells <= 0 || !(radius > 0.0) || n_cells >= (int64_t)INT32_MAX) return B200FEM_E_INVALID;
  *out = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  Filter *f = new Filter();
  f->n = n_cells;
  f->radius = radius;
  f->stream = s;
  const int64_t n = n_cells;
  double *cent = nullptr, *dist = nullptr;
  int64_t *key = nullptr, *skey = nullptr;
  int32_t *ids = nullptr, *sid = nullptr, *cnt = nullptr;
  unsigned long long *bb = nullptr;
  void *tmp = nullptr;
  int st = B200FEM_E_CUDA;
  do {
    if (dalloc(&cent, 3 * n) || dalloc(&key, n) || dalloc(&skey, n) || dalloc(&ids, n) || dalloc(&sid, n) ||
        dalloc(&cnt, n + 1) || dalloc(&bb, 6) || dalloc(&f->indptr, n + 1))
      break;
    k_centroids<<<grid_n(n), kThreads, 0, s>>>(coords_dev, cells_dev, n, cent);
    cudaMemsetAsync(bb, 0xff, 3 * sizeof(unsigned long long), s);
    cudaMemsetAsync(bb + 3, 0, 3 * sizeof(unsigned long long), s);
    k_bbox<<<grid_n(n), kThreads, 0, s>>>(cent, n, bb);
    count_launch(2);
    unsigned long long hb[6];  // the grid shape needs the bounding box on the host
    if (cudaMemcpyAsync(hb, bb, sizeof(hb), cudaMemcpyDeviceToHost, s) || cudaStreamSynchronize(s)) break;
    BinGrid g{};
    double hi[3];
    for (int d = 0; d < 3; ++d) g.org[d] = host_unord(hb[d]), hi[d] = host_unord(hb[3 + d]);
    // bin edge >= radius; coarsen so the grid has at most ~2 bins per cell
    g.h = radius;
    for (;;) {
      int64_t tot = 1;
      for (int d = 0; d < 3; ++d) {
        g.dims[d] = std::max<int64_t>(1, (int64_t)std::floor((hi[d] - g.org[d]) / g.h) + 1);
        tot *= g.dims[d];
      }
      if (tot <= 2 * n + 27) break;
      g.h *= 1.5;
    }
    k_bin_keys<<<grid_n(n), kThreads, 0, s>>>(cent, n, g, key, ids);
    size_t sort_bytes = 0, scan_bytes = 0;
    int end_bit = 1;
    {
      const int64_t nb = g.dims[0] * g.dims[1] * g.dims[2];
      while (end_bit < 63 && (int64_t(1) << end_bit) < nb) ++end_bit;
    }
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, skey, ids, sid, (int)n, 0, end_bit, s);
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, f->indptr, (int)(n + 1), s);
    if (cudaMalloc(&tmp, std::max(sort_bytes, scan_bytes))) break;
    if (cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, key, skey, ids, sid, (int)n, 0, end_bit, s)) break;
    cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int32_t), s);
    k_filter_rows<0><<<grid_n(n), kThreads, 0, s>>>(cent, n, g, radius, skey, sid, cnt, nullptr, nullptr, nullptr);
    if (cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, cnt, f->indptr, (int)(n + 1), s)) break;
    int32_t nnz32 = 0;
    if (cudaMemcpyAsync(&nnz32, f->indptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s) ||
        cudaStreamSynchronize(s))
      break;
    f->nnz = nnz32;
    if (dalloc(&f->indices, std::max<int64_t>(1, f->nnz)) || dalloc(&f->data, std::max<int64_t>(1, f->nnz)) ||
        dalloc(&dist, std::max<int64_t>(1, f->nnz)))
      break;
    k_filter_rows<1><<<grid_n(n), kThreads, 0, s>>>(cent, n, g, radius, skey, sid, nullptr, f->indptr, f->indices,
                                                     dist);
    k_filter_finish<<<grid_n(n), kThreads, 0, s>>>(n, radius, f->indptr, f->indices, dist, f->data);
    count_launch(4);
    if (cudaStreamSynchronize(s) || cudaGetLastError()) break;
    st = 0;
  } while (false);
  cudaFree(cent);
  cudaFree(dist);
  cudaFree(key);
  cudaFree(skey);
  cudaFree(ids);
  cudaFree(sid);
  cudaFree(cnt);
  cudaFree(bb);
  cudaFree(tmp);
  if (st) {
    cudaFree(f->indptr);
    cudaFree(f->indices);
    cudaFree(f->data);
    delete f;
    return st;
  }
  *out = (b200fem_filter *)f;
  return 0;
}

int b200fem_filter_info(const b200fem_filter *h, int64_t *n, int64_t *nnz) {
  const Filter *f = (const Filter *)h;
  if (!f) return B200FEM_E_INVALID;
  if (n) *n = f->n;
  if (nnz) *nnz = f->nnz;
  return 0;
}

int b200fem_filter_copy(const b200fem_filter *h, int32_t *indptr, int32_t *indices, double *data) {
  const Filter *f = (const Filter *)h;
  if (!f || !indptr || !indices || !data) return B200FEM_E_INVALID;
  cudaStream_t s = f->stream;
  B200_CUDA(cudaMemcpyAsync(indptr, f->indptr, (f->n + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (f->nnz) {
    B200_CUDA(cudaMemcpyAsync(indices, f->indices, f->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    B200_CUDA(cudaMemcpyAsync(data, f->data, f->nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  B200_CUDA(cudaStreamSynchronize(s));
  return 0;
}

int b200fem_filter_apply(const b200fem_filter *h, const double *v, const double *mul, const double *div,
                         double floor_v, double *y) {
  const Filter *f = (const Filter *)h;
  if (!f || !v || !y) return B200FEM_E_INVALID;
  k_filter_apply<<<grid_n(f->n), kThreads, 0, f->stream>>>(f->n, f->indptr, f->indices, f->data, v, mul, div,
                                                            floor_v, y);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int b200fem_filter_destroy(b200fem_filter *h) {
  Filter *f = (Filter *)h;
  if (!f) return 0;
  cudaStreamSynchronize(f->stream);
  cudaFree(f->indptr);
  cudaFree(f->indices);
  cudaFree(f->data);
  delete f;
  return 0;
}

int b200fem_mma_update(int64_t n, const double *x, const double *dj, double g_value, const double *g_grad,
                       const double *lb, const double *ub, double *lower, double *upper, const double *x_prev,
                       const double *x_prev2, int32_t use_history, double asym_init, double asym_expand,
                       double asym_shrink, double move_limit, double *x_new, void *stream) {
  if (n < 0 || !x || !dj || !g_grad || !lb || !ub || !lower || !upper || !x_new) return B200FEM_E_INVALID;
  if (use_history && (!x_prev || !x_prev2)) return B200FEM_E_INVALID;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // grow-only scratch reused across updates (an optimisation loop calls this every step)
  static double *work = nullptr;
  static int64_t work_n = 0;
  static MmaCtl *ctl = nullptr;
  static RedScratch red{};
  if (!ctl && (dalloc(&ctl, 1) || red_alloc(&red))) return B200FEM_E_CUDA;
  if (work_n < n) {
    cudaStreamSynchronize(s);
    cudaFree(work);
    work = nullptr;
    work_n = 0;
    if (dalloc(&work, 4 * n)) return B200FEM_E_CUDA;
    work_n = n;
  }
  MmaCtl h{};
  h.g_value = g_value;
  B200_CUDA(cudaMemcpyAsync(ctl, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  MmaArgs a{x, dj, g_grad, lb, ub, x_prev, x_prev2, lower, upper, work, work + n, work + 2 * n, work + 3 * n,
            x_new, asym_init, asym_expand, asym_shrink, move_limit, use_history};
  const int gv = grid_n(n), gr = std::min(kRedBlocks, gv);
  k_mma_absmax<<<gv, kThreads, 0, s>>>(n, dj, ctl);
  k_mma_prep<<<gv, kThreads, 0, s>>>(n, a, ctl);
  for (int e = 0; e < 1 + 41 + 100; ++e) k_mma_eval<false><<<gr, kThreads, 0, s>>>(n, a, ctl, red);
  k_mma_eval<true><<<gv, kThreads, 0, s>>>(n, a, ctl, red);
  count_launch(2 + 142 + 1);
  B200_CUDA(cudaStreamSynchronize(s));  // h (the control block source) must outlive the copy
  B200_CUDA(cudaGetLastError());
  return 0;
}

}  // extern "C"
