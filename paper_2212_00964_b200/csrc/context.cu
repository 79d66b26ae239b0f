// Context lifecycle, CSR pattern / scatter-position build, boundary data,
// and the small deterministic vector reductions.
//
// Reference being replaced: assembly.workspace() (assembly.py:83-145) and
// sparse.pattern_from_cells() (sparse.py:75-108).  The pattern is built per node
// instead of by a global sort: a DOF row of node n couples exactly the DOFs of the
// nodes sharing a cell with n, so sorting each node's <=8*deg candidates locally gives
// the same sorted unique keys -> bit-identical indptr / indices / dest.

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdarg>
#include <numeric>

#include "internal.cuh"

namespace b200 {

std::atomic<int64_t> g_launches{0};

void set_err(b200fem_error *err, int code, const char *fmt, ...) {
  if (!err) return;
  err->code = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, b200fem_error *err, const char *where) {
  if (err) {
    err->code = B200FEM_E_CUDA;
    snprintf(err->msg, sizeof(err->msg), "CUDA error %s at %s", cudaGetErrorString(e), where);
  } else {
    fprintf(stderr, "[b200fem] CUDA error %s at %s\n", cudaGetErrorString(e), where);
  }
  return B200FEM_E_CUDA;
}

int red_alloc(RedScratch *r) {
  B200_CUDA(dalloc(&r->partials, (size_t)kRedBlocks * kMaxVals));
  B200_CUDA(dalloc(&r->ticket, 1));
  B200_CUDA(cudaMemset(r->ticket, 0, sizeof(unsigned)));
  B200_CUDA(dalloc(&r->result, kMaxVals));
  return 0;
}

void red_free(RedScratch *r) {
  cudaFree(r->partials);
  cudaFree(r->ticket);
  cudaFree(r->result);
  *r = RedScratch{};
}

// ------------------------------------------------------------ pattern kernels
__global__ void k_degree(const int32_t *__restrict__ cells, int64_t n8, int32_t *deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + cells[i], 1);
}

__global__ void k_fill_n2c(const int32_t *__restrict__ cells, int64_t n8, const int32_t *__restrict__ ptr,
                           int32_t *cursor, int32_t *n2c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    int n = cells[i];
    int slot = atomicAdd(cursor + n, 1);
    n2c[ptr[n] + slot] = (int32_t)(i >> 3);
  }
}

// each node's incident cells in ascending cell order (the reference's accumulation order)
__global__ void k_sort_n2c(const int32_t *__restrict__ ptr, int64_t n_nodes, const int32_t *__restrict__ cells,
                           int32_t *n2c, uint8_t *n2c_a, int *max_deg) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int lo = ptr[n], hi = ptr[n + 1];
    for (int i = lo + 1; i < hi; ++i) {
      const int v = n2c[i];
      int j = i - 1;
      while (j >= lo && n2c[j] > v) {
        n2c[j + 1] = n2c[j];
        --j;
      }
      n2c[j + 1] = v;
    }
    // a cell listing the same node twice appears twice: give each copy its own local index
    for (int i = lo; i < hi; ++i) {
      const int64_t e = n2c[i];
      int k = 0, seen = 0;
      for (int t = lo; t < i; ++t) seen += (n2c[t] == e);
      for (int q = 0; q < 8; ++q)
        if (cells[e * 8 + q] == n) {
          if (seen == 0) {
            k = q;
            break;
          }
          --seen;
        }
      n2c_a[i] = (uint8_t)k;
    }
    atomicMax(max_deg, hi - lo);
  }
}

constexpr int kMaxCand = 512;  // <= 64 cells per node
constexpr int kNbrWarps = 4;

// Warp per node: unique-sort the nodes of all incident cells.  mode 0: write counts,
// mode 1: write the sorted list at out_ptr[n].
__global__ void __launch_bounds__(kNbrWarps * 32) k_neighbors(
    const int32_t *__restrict__ cells, const int32_t *__restrict__ n2c_ptr, const int32_t *__restrict__ n2c,
    int64_t n_nodes, int mode, int32_t *cnt, const int32_t *__restrict__ out_ptr, int32_t *out, int *overflow) {
  __shared__ int32_t cand[kNbrWarps][kMaxCand];
  __shared__ uint8_t first[kNbrWarps][kMaxCand];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t n = blockIdx.x * (int64_t)kNbrWarps + w; n < n_nodes; n += (int64_t)gridDim.x * kNbrWarps) {
    const int c0 = n2c_ptr[n], deg = n2c_ptr[n + 1] - c0;
    const int C = deg * 8;
    if (C > kMaxCand) {
      if (lane == 0) atomicExch(overflow, 1);
      continue;
    }
    for (int j = lane; j < C; j += 32) cand[w][j] = cells[(int64_t)n2c[c0 + (j >> 3)] * 8 + (j & 7)];
    __syncwarp();
    for (int j = lane; j < C; j += 32) {
      int v = cand[w][j];
      bool f = true;
      for (int i = 0; i < j; ++i) f &= (cand[w][i] != v);
      first[w][j] = f;
    }
    __syncwarp();
    int mine = 0;
    for (int j = lane; j < C; j += 32) {
      if (!first[w][j]) continue;
      ++mine;
      if (mode == 1) {
        int v = cand[w][j], rank = 0;
        for (int i = 0; i < C; ++i) rank += (first[w][i] && cand[w][i] < v);
        out[out_ptr[n] + rank] = v;
      }
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (mode == 0 && lane == 0) cnt[n] = mine;
    __syncwarp();
  }
}

__global__ void k_indptr(const int32_t *__restrict__ nbr_ptr, int64_t n_nodes, int vec, int32_t *indptr) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n <= n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = nbr_ptr[n];
    if (n == n_nodes) {
      indptr[n * vec] = (int32_t)(p * vec * vec);
      continue;
    }
    int64_t cnt = nbr_ptr[n + 1] - p;
    for (int c = 0; c < vec; ++c) indptr[n * vec + c] = (int32_t)(p * vec * vec + c * vec * cnt);
  }
}

__device__ __forceinline__ int find_sorted(const int32_t *__restrict__ a, int len, int v) {
  int lo = 0, hi = len;  // first index with a[i] >= v
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_cpos(const int32_t *__restrict__ cells, int64_t n_cells, const int32_t *__restrict__ nbr_ptr,
                       const int32_t *__restrict__ nbr, uint8_t *cpos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_cells * 64; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = i >> 6;
    int a = (i >> 3) & 7, b = i & 7;
    int na = cells[e * 8 + a], nb = cells[e * 8 + b];
    int p0 = nbr_ptr[na];
    cpos[i] = (uint8_t)find_sorted(nbr + p0, nbr_ptr[na + 1] - p0, nb);
  }
}

__global__ void k_diag_slots(const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr,
                             const int32_t *__restrict__ indptr, int64_t n_nodes, int vec, int32_t *diag) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    int p0 = nbr_ptr[n];
    int pos = find_sorted(nbr + p0, nbr_ptr[n + 1] - p0, (int)n);
    for (int c = 0; c < vec; ++c) diag[n * vec + c] = indptr[n * vec + c] + vec * pos + c;
  }
}

// symmetric storage maps: upper-block counts per node, then the block index of every
// lower coupling (m < n) inside m's upper list
__global__ void k_sym_count(const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr, int64_t n_nodes,
                            int32_t *ucnt) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int p0 = nbr_ptr[n], cnt = nbr_ptr[n + 1] - p0;
    ucnt[n] = cnt - find_sorted(nbr + p0, cnt, (int)n);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ucnt[n_nodes] = 0;
}

__global__ void k_sym_lower(const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr,
                            const int32_t *__restrict__ up_ptr, int64_t n_nodes, int32_t *lo_blk) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    const int p0 = nbr_ptr[n], cnt = nbr_ptr[n + 1] - p0;
    for (int j = 0; j < cnt; ++j) {
      const int m = nbr[p0 + j];
      if (m >= n) break;
      const int q0 = nbr_ptr[m], qc = nbr_ptr[m + 1] - q0;
      const int self_m = qc - (up_ptr[m + 1] - up_ptr[m]);
      const int pos = find_sorted(nbr + q0, qc, (int)n);
      lo_blk[p0 + j] = up_ptr[m] + (pos - self_m);
    }
  }
}

__global__ void k_indices(const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr,
                          const int32_t *__restrict__ indptr, int64_t n_nodes, int vec, int32_t *indices) {
  const int lane = threadIdx.x & 31;
  for (int64_t n = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; n < n_nodes;
       n += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int p0 = nbr_ptr[n], cnt = nbr_ptr[n + 1] - p0;
    for (int c = 0; c < vec; ++c) {
      int64_t base = indptr[n * vec + c];
      for (int e = lane; e < cnt * vec; e += 32) indices[base + e] = nbr[p0 + e / vec] * vec + e % vec;
    }
  }
}

__global__ void k_dest(const int32_t *__restrict__ cells, const uint8_t *__restrict__ cpos,
                       const int32_t *__restrict__ indptr, int64_t lo, int64_t hi, int vec, int32_t *dest) {
  const int nd = 8 * vec;
  const int64_t total = (hi - lo) * nd * nd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = lo + i / (nd * nd);
    int A = (int)((i / nd) % nd), B = (int)(i % nd);
    int a = A / vec, ci = A % vec, b = B / vec, ck = B % vec;
    int na = cells[e * 8 + a];
    dest[i] = indptr[(int64_t)na * vec + ci] + vec * cpos[e * 64 + a * 8 + b] + ck;
  }
}

static int grid_for(int64_t n, int threads = kThreads) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

static void free_ctx(Ctx *c) {
  if (!c) return;
  void *ptrs[] = {c->coords, c->cells, c->nbr_ptr, c->nbr, c->indptr, c->cpos, c->diag,
                  c->dir_dofs, c->dir_vals, c->f_neumann, c->f_body, c->theta, c->eps_prev, c->sig_prev, c->derr,
                  c->n2c_ptr, c->n2c, c->n2c_a, c->dir_flag, c->scratch, c->up_ptr, c->lo_blk};
  for (void *p : ptrs) cudaFree(p);
  if (c->indices && c->indices != c->nbr) cudaFree(c->indices);
  red_free(&c->red);
  if (c->pinned) cudaFreeHost(c->pinned);
  delete c;
}

// Host-side restatement of the det J formula for the InvertedElementError message.
static double host_detJ(const double *X /*8x3*/, int q) {
  const double g = 1.0 / std::sqrt(3.0);
  const double s[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                          {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
  double xi[3] = {(q & 1) ? g : -g, (q & 2) ? g : -g, (q & 4) ? g : -g};
  double J[3][3] = {};
  for (int k = 0; k < 8; ++k) {
    double t[3];
    for (int d = 0; d < 3; ++d) t[d] = 1.0 + xi[d] * s[k][d];
    double dn[3] = {s[k][0] * (t[1] * t[2]) / 8.0, s[k][1] * (t[0] * t[2]) / 8.0, s[k][2] * (t[0] * t[1]) / 8.0};
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) J[a][b] += X[k * 3 + a] * dn[b];
  }
  double A = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  double D = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  double G = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  return J[0][0] * A + J[0][1] * D + J[0][2] * G;
}

// GRID3 applies when the connectivity is exactly a z-major box lattice, i.e. the cells of
// generate_box_mesh (mesh.py:152-167; also every z-slab part of one): cell i + nx j + nx ny k
// has vertices base + {0, 1, NX+1, NX, NXY, NXY+1, NXY+NX+1, NXY+NX}, base = i + NX j + NXY k.
static void detect_grid(Ctx *c, const int64_t *cells_h) {
  if (getenv("B200FEM_NO_GRID")) return;
  const int64_t ne = c->n_cells, nn = c->n_nodes;
  const int64_t NX = cells_h[3], NXY = cells_h[4];
  if (NX < 2 || NXY < 2 * NX || NXY % NX || nn % NXY) return;
  const int64_t NY = NXY / NX, NZ = nn / NXY;
  const int64_t nx = NX - 1, ny = NY - 1, nz = NZ - 1;
  if (nz < 1 || nx * ny * nz != ne) return;
  const int64_t pat[8] = {0, 1, NX + 1, NX, NXY, NXY + 1, NXY + NX + 1, NXY + NX};
  for (int64_t e = 0; e < ne; ++e) {
    const int64_t i = e % nx, j = (e / nx) % ny, k = e / (nx * ny);
    const int64_t base = i + NX * j + NXY * k;
    for (int v = 0; v < 8; ++v)
      if (cells_h[8 * e + v] != base + pat[v]) return;
  }
  c->grid_nx = (int)NX;
  c->grid_ny = (int)NY;
  c->grid_nz = (int)NZ;
  c->grid_npad = (nn + 31) & ~31ll;  // whole 32-node tiles (internal.cuh grid_idx)
}

static int build(Ctx *c, const double *coords_h, const int64_t *cells_h, b200fem_error *err) {
  cudaStream_t s = c->stream;
  const int64_t nn = c->n_nodes, ne = c->n_cells;
  // ---- upload mesh (cells as int32: n_nodes < 2^31 is required by the int32 CSR anyway)
  std::vector<int32_t> c32(ne * 8);
  for (int64_t i = 0; i < ne * 8; ++i) c32[i] = (int32_t)cells_h[i];
  B200_CUDA_E(dalloc(&c->coords, nn * 3), err);
  B200_CUDA_E(dalloc(&c->cells, ne * 8), err);
  B200_CUDA_E(cudaMemcpyAsync(c->coords, coords_h, nn * 3 * sizeof(double), cudaMemcpyHostToDevice, s), err);
  B200_CUDA_E(cudaMemcpyAsync(c->cells, c32.data(), ne * 8 * sizeof(int32_t), cudaMemcpyHostToDevice, s), err);
  B200_CUDA_E(dalloc(&c->derr, 1), err);
  B200_CUDA_E(cudaMemsetAsync(c->derr, 0xff, sizeof(DevErr), s), err);
  if (red_alloc(&c->red)) return set_err(err, B200FEM_E_CUDA, "scratch allocation failed"), B200FEM_E_CUDA;
  B200_CUDA_E(cudaMallocHost((void **)&c->pinned, 16 * sizeof(double)), err);

  // ---- geometry check (elements.py:117-131 raises on det <= 0)
  int st = check_geometry(c, err);
  if (st) {
    if (st == B200FEM_E_INVERTED_ELEMENT && err) {
      double X[24];
      for (int k = 0; k < 8; ++k)
        for (int d = 0; d < 3; ++d) X[k * 3 + d] = coords_h[cells_h[err->cell * 8 + k] * 3 + d];
      err->value = host_detJ(X, err->qp);
      snprintf(err->msg, sizeof(err->msg),
               "non-positive Jacobian determinant %.3e (cell %lld of batch, quad point %d)", err->value,
               (long long)err->cell, err->qp);
    }
    return st;
  }

  // ---- node -> cell adjacency
  int32_t *deg = nullptr, *n2c_ptr = nullptr, *n2c = nullptr, *cnt = nullptr, *overflow = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  auto cleanup = [&]() {
    cudaFree(deg); cudaFree(cnt); cudaFree(overflow); cudaFree(tmp);
  };
  B200_CUDA_E(dalloc(&deg, nn + 1), err);
  B200_CUDA_E(dalloc(&n2c_ptr, nn + 1), err);
  B200_CUDA_E(dalloc(&n2c, ne * 8), err);
  B200_CUDA_E(dalloc(&cnt, nn + 1), err);
  B200_CUDA_E(dalloc(&overflow, 1), err);
  B200_CUDA_E(cudaMemsetAsync(deg, 0, (nn + 1) * sizeof(int32_t), s), err);
  B200_CUDA_E(cudaMemsetAsync(overflow, 0, sizeof(int), s), err);
  k_degree<<<grid_for(ne * 8), kThreads, 0, s>>>(c->cells, ne * 8, deg);
  count_launch();
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, deg, n2c_ptr, (int)(nn + 1), s);
  size_t tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, cnt, cnt, (int)(nn + 1), s);
  tmp_bytes = std::max(tmp_bytes, tmp2);
  B200_CUDA_E(cudaMalloc(&tmp, tmp_bytes), err);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, n2c_ptr, (int)(nn + 1), s);
  count_launch();
  B200_CUDA_E(cudaMemsetAsync(deg, 0, (nn + 1) * sizeof(int32_t), s), err);
  k_fill_n2c<<<grid_for(ne * 8), kThreads, 0, s>>>(c->cells, ne * 8, n2c_ptr, deg, n2c);
  count_launch();
  c->n2c_ptr = n2c_ptr;
  c->n2c = n2c;
  B200_CUDA_E(cudaMemsetAsync(overflow, 0, sizeof(int), s), err);
  B200_CUDA_E(dalloc(&c->n2c_a, ne * 8), err);
  k_sort_n2c<<<grid_for(nn), kThreads, 0, s>>>(n2c_ptr, nn, c->cells, n2c, c->n2c_a, overflow);
  count_launch();
  B200_CUDA_E(cudaMemcpyAsync(&c->max_deg, overflow, sizeof(int), cudaMemcpyDeviceToHost, s), err);
  B200_CUDA_E(cudaStreamSynchronize(s), err);
  B200_CUDA_E(cudaMemsetAsync(overflow, 0, sizeof(int), s), err);

  // ---- node adjacency lists (the CSR pattern at node granularity)
  int nb_grid = (int)std::min<int64_t>((nn + kNbrWarps - 1) / kNbrWarps, 148 * 64);
  B200_CUDA_E(cudaMemsetAsync(cnt, 0, (nn + 1) * sizeof(int32_t), s), err);
  k_neighbors<<<nb_grid, kNbrWarps * 32, 0, s>>>(c->cells, n2c_ptr, n2c, nn, 0, cnt, nullptr, nullptr, overflow);
  count_launch();
  B200_CUDA_E(dalloc(&c->nbr_ptr, nn + 1), err);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, c->nbr_ptr, (int)(nn + 1), s);
  count_launch();
  int32_t total = 0, ovf = 0;
  B200_CUDA_E(cudaMemcpyAsync(&total, c->nbr_ptr + nn, sizeof(int32_t), cudaMemcpyDeviceToHost, s), err);
  B200_CUDA_E(cudaMemcpyAsync(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost, s), err);
  B200_CUDA_E(cudaStreamSynchronize(s), err);
  if (ovf) {
    cleanup();
    set_err(err, B200FEM_E_UNSUPPORTED, "a node is shared by more than %d cells", kMaxCand / 8);
    return B200FEM_E_UNSUPPORTED;
  }
  const int64_t nnz = (int64_t)total * c->vec * c->vec;
  if (nnz >= (int64_t)INT32_MAX) {
    cleanup();
    set_err(err, B200FEM_E_UNSUPPORTED, "nnz %lld exceeds the int32 CSR index range", (long long)nnz);
    return B200FEM_E_UNSUPPORTED;
  }
  c->nnz = nnz;
  B200_CUDA_E(dalloc(&c->nbr, total), err);
  k_neighbors<<<nb_grid, kNbrWarps * 32, 0, s>>>(c->cells, n2c_ptr, n2c, nn, 1, nullptr, c->nbr_ptr, c->nbr, overflow);
  count_launch();
  // max neighbours per node (<= 255 so the per-cell positions fit a byte)
  {
    std::vector<int32_t> hp(nn + 1);
    B200_CUDA_E(cudaMemcpyAsync(hp.data(), c->nbr_ptr, (nn + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s), err);
    B200_CUDA_E(cudaStreamSynchronize(s), err);
    int mx = 0;
    for (int64_t n = 0; n < nn; ++n) mx = std::max(mx, hp[n + 1] - hp[n]);
    c->max_nbr = mx;
    if (mx > 255) {
      cleanup();
      set_err(err, B200FEM_E_UNSUPPORTED, "a node couples to %d nodes (> 255)", mx);
      return B200FEM_E_UNSUPPORTED;
    }
  }
  B200_CUDA_E(dalloc(&c->indptr, c->n_dofs + 1), err);
  k_indptr<<<grid_for(nn + 1), kThreads, 0, s>>>(c->nbr_ptr, nn, c->vec, c->indptr);
  count_launch();
  B200_CUDA_E(dalloc(&c->cpos, ne * 64), err);
  k_cpos<<<grid_for(ne * 64), kThreads, 0, s>>>(c->cells, ne, c->nbr_ptr, c->nbr, c->cpos);
  count_launch();
  B200_CUDA_E(dalloc(&c->diag, c->n_dofs), err);
  k_diag_slots<<<grid_for(nn), kThreads, 0, s>>>(c->nbr_ptr, c->nbr, c->indptr, nn, c->vec, c->diag);
  count_launch();
  if (c->vec == 1) c->indices = c->nbr;  // vec 1: the node list IS the column list
  if (c->vec == 3) {  // symmetric node-block storage maps
    int32_t *ucnt = nullptr;
    B200_CUDA_E(dalloc(&ucnt, nn + 1), err);
    B200_CUDA_E(dalloc(&c->up_ptr, nn + 1), err);
    k_sym_count<<<grid_for(nn), kThreads, 0, s>>>(c->nbr_ptr, c->nbr, nn, ucnt);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ucnt, c->up_ptr, (int)(nn + 1), s);
    B200_CUDA_E(dalloc(&c->lo_blk, total), err);
    k_sym_lower<<<grid_for(nn), kThreads, 0, s>>>(c->nbr_ptr, c->nbr, c->up_ptr, nn, c->lo_blk);
    count_launch(3);
    int32_t nb = 0;
    B200_CUDA_E(cudaMemcpyAsync(&nb, c->up_ptr + nn, sizeof(int32_t), cudaMemcpyDeviceToHost, s), err);
    B200_CUDA_E(cudaStreamSynchronize(s), err);
    cudaFree(ucnt);
    c->n_sym_blocks = nb;
  }

  detect_grid(c, cells_h);

  B200_CUDA_E(cudaStreamSynchronize(s), err);
  cleanup();
  B200_CUDA_E(cudaGetLastError(), err);
  return 0;
}

// ------------------------------------------------------------ reductions
template <int MODE>  // 0: dot(x,y), 1: gather-sum x[idx]
__global__ void __launch_bounds__(kThreads) k_reduce(const double *__restrict__ x, const double *__restrict__ y,
                                                     const int64_t *__restrict__ idx, int64_t n, RedScratch red) {
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (MODE == 0) v[0] += x[i] * y[i];
    else v[0] += x[idx[i]];
  }
  double tot[1];
  block_partials_and_finish<1>(v, red, tot);
}

int launch_dot(const double *x, const double *y, int64_t n, RedScratch *r, cudaStream_t s) {
  k_reduce<0><<<kRedBlocks, kThreads, 0, s>>>(x, y, nullptr, n, *r);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int launch_gather_sum(const double *x, const int64_t *idx, int64_t n, RedScratch *r, cudaStream_t s) {
  k_reduce<1><<<kRedBlocks, kThreads, 0, s>>>(x, nullptr, idx, n, *r);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

__global__ void k_axpy(int64_t n, double a, const double *__restrict__ x, double *__restrict__ y, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = mode == 0 ? y[i] + a * x[i] : a * x[i];
}

int launch_axpy(int64_t n, double a, const double *x, double *y, cudaStream_t s) {
  k_axpy<<<grid_for(n), kThreads, 0, s>>>(n, a, x, y, 0);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int launch_scale(int64_t n, double a, const double *x, double *y, cudaStream_t s) {
  k_axpy<<<grid_for(n), kThreads, 0, s>>>(n, a, x, y, 1);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

}  // namespace b200

using namespace b200;

// =====================================================================  C ABI
extern "C" {

int b200fem_version(void) { return 1; }
int64_t b200fem_launch_count(void) { return g_launches.load(); }

int b200fem_stream_sync(void *stream) {
  B200_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

int b200fem_ctx_create(b200fem_ctx **out, int64_t n_nodes, int64_t n_cells, int32_t vec, const double *coords_host,
                       const int64_t *cells_host, int32_t material, const double *params, int32_t flags,
                       void *stream, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (!out || n_nodes <= 0 || n_cells <= 0 || !coords_host || !cells_host || !params || (vec != 1 && vec != 3) ||
      material < 0 || material > 3 || (material == B200FEM_MAT_POISSON) != (vec == 1)) {
    set_err(err, B200FEM_E_INVALID, "invalid context arguments");
    return B200FEM_E_INVALID;
  }
  if (n_nodes * vec >= INT32_MAX) {
    set_err(err, B200FEM_E_UNSUPPORTED, "too many DOFs for int32 CSR");
    return B200FEM_E_UNSUPPORTED;
  }
  for (int64_t i = 0; i < n_cells * 8; ++i)
    if (cells_host[i] < 0 || cells_host[i] >= n_nodes) {
      set_err(err, B200FEM_E_INVALID, "cell connectivity references nodes out of range");
      return B200FEM_E_INVALID;
    }
  element_tables_init();
  Ctx *c = new Ctx();
  cudaGetDevice(&c->device);
  c->stream = (cudaStream_t)stream;
  c->n_nodes = n_nodes;
  c->n_cells = n_cells;
  c->vec = vec;
  c->n_dofs = n_nodes * vec;
  c->material = material;
  c->flags = flags;
  c->mp.alpha = params[0];
  c->mp.lam = params[1];
  c->mp.mu = params[2];
  c->mp.kappa = params[3];
  c->mp.sy = params[4];
  c->mp.penalty = params[5];
  c->mp.simp = (flags & B200FEM_FLAG_SIMP) ? 1 : 0;
  c->mp.design_source = (flags & B200FEM_FLAG_DESIGN_SOURCE) ? 1 : 0;
  int st = build(c, coords_host, cells_host, err);
  if (st) {
    free_ctx(c);
    return st;
  }
  if (material == B200FEM_MAT_J2) {
    size_t n = (size_t)n_cells * 72;
    if (dalloc(&c->eps_prev, n) || dalloc(&c->sig_prev, n) ||
        cudaMemsetAsync(c->eps_prev, 0, n * sizeof(double), c->stream) ||
        cudaMemsetAsync(c->sig_prev, 0, n * sizeof(double), c->stream)) {
      free_ctx(c);
      set_err(err, B200FEM_E_CUDA, "state allocation failed");
      return B200FEM_E_CUDA;
    }
  }
  *out = (b200fem_ctx *)c;
  return 0;
}

int b200fem_ctx_destroy(b200fem_ctx *ctx) {
  Ctx *c = (Ctx *)ctx;
  if (c) cudaStreamSynchronize(c->stream);
  free_ctx(c);
  return 0;
}

int b200fem_ctx_info(const b200fem_ctx *ctx, int64_t *n_dofs, int64_t *nnz, int32_t *max_nbr) {
  const Ctx *c = (const Ctx *)ctx;
  if (!c) return B200FEM_E_INVALID;
  if (n_dofs) *n_dofs = c->n_dofs;
  if (nnz) *nnz = c->nnz;
  if (max_nbr) *max_nbr = c->max_nbr;
  return 0;
}

int b200fem_copy_indptr(b200fem_ctx *ctx, int32_t *out) {
  Ctx *c = (Ctx *)ctx;
  B200_CUDA(cudaMemcpyAsync(out, c->indptr, (c->n_dofs + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
  return 0;
}

int b200fem_copy_indices(b200fem_ctx *ctx, int32_t *out) {
  Ctx *c = (Ctx *)ctx;
  k_indices<<<grid_for(c->n_nodes * 32), kThreads, 0, c->stream>>>(c->nbr_ptr, c->nbr, c->indptr, c->n_nodes, c->vec, out);
  count_launch();
  B200_CUDA(cudaGetLastError());
  return 0;
}

int b200fem_copy_dest(b200fem_ctx *ctx, int64_t lo, int64_t hi, int32_t *out) {
  Ctx *c = (Ctx *)ctx;
  if (lo < 0 || hi > c->n_cells || lo > hi) return B200FEM_E_INVALID;
  if (hi == lo) return 0;
  int64_t total = (hi - lo) * 64 * c->vec * c->vec;
  k_dest<<<grid_for(total), kThreads, 0, c->stream>>>(c->cells, c->cpos, c->indptr, lo, hi, c->vec, out);
  count_launch();
  B200_CUDA(cudaGetLastError());
  return 0;
}

int b200fem_copy_diag_slots(b200fem_ctx *ctx, int32_t *out) {
  Ctx *c = (Ctx *)ctx;
  B200_CUDA(cudaMemcpyAsync(out, c->diag, c->n_dofs * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
  return 0;
}

int b200fem_set_dirichlet(b200fem_ctx *ctx, const int64_t *dofs, const double *vals, int64_t n) {
  Ctx *c = (Ctx *)ctx;
  cudaStreamSynchronize(c->stream);
  cudaFree(c->dir_dofs);
  cudaFree(c->dir_vals);
  c->dir_dofs = nullptr;
  c->dir_vals = nullptr;
  c->n_dir = n;
  if (n <= 0) {
    c->n_dir = 0;
    cudaFree(c->dir_flag);
    c->dir_flag = nullptr;
    return 0;
  }
  std::vector<int32_t> d32(n);
  for (int64_t i = 0; i < n; ++i) {
    if (dofs[i] < 0 || dofs[i] >= c->n_dofs) return B200FEM_E_INVALID;
    d32[i] = (int32_t)dofs[i];
  }
  B200_CUDA(dalloc(&c->dir_dofs, n));
  B200_CUDA(dalloc(&c->dir_vals, n));
  {
    std::vector<uint8_t> flag(c->n_dofs, 0);
    for (int64_t i = 0; i < n; ++i) flag[d32[i]] = 1;
    if (!c->dir_flag) B200_CUDA(dalloc(&c->dir_flag, c->n_dofs));
    B200_CUDA(cudaMemcpy(c->dir_flag, flag.data(), c->n_dofs, cudaMemcpyHostToDevice));
  }
  B200_CUDA(cudaMemcpyAsync(c->dir_dofs, d32.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  B200_CUDA(cudaMemcpyAsync(c->dir_vals, vals, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  B200_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

static int upload_vec(Ctx *c, double **dst, const double *src, int64_t n) {
  if (!src) {
    cudaFree(*dst);
    *dst = nullptr;
    return 0;
  }
  if (!*dst) B200_CUDA(dalloc(dst, n));
  B200_CUDA(cudaMemcpyAsync(*dst, src, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  return 0;
}

int b200fem_set_loads(b200fem_ctx *ctx, const double *fn, const double *fb) {
  Ctx *c = (Ctx *)ctx;
  cudaStreamSynchronize(c->stream);
  int st = upload_vec(c, &c->f_neumann, fn, c->n_dofs);
  if (!st) st = upload_vec(c, &c->f_body, fb, c->n_dofs);
  cudaStreamSynchronize(c->stream);
  return st;
}

int b200fem_set_theta(b200fem_ctx *ctx, const double *theta, int64_t n, int32_t is_host) {
  Ctx *c = (Ctx *)ctx;
  if (c->n_theta != n) {
    cudaStreamSynchronize(c->stream);
    cudaFree(c->theta);
    c->theta = nullptr;
    c->n_theta = n;
    B200_CUDA(dalloc(&c->theta, n));
  }
  B200_CUDA(cudaMemcpyAsync(c->theta, theta, n * sizeof(double),
                            is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream));
  if (is_host) B200_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int b200fem_set_state(b200fem_ctx *ctx, const double *eps, const double *sig, int32_t is_host) {
  Ctx *c = (Ctx *)ctx;
  if (!c->eps_prev) return B200FEM_E_INVALID;
  size_t bytes = (size_t)c->n_cells * 72 * sizeof(double);
  cudaMemcpyKind k = is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  B200_CUDA(cudaMemcpyAsync(c->eps_prev, eps, bytes, k, c->stream));
  B200_CUDA(cudaMemcpyAsync(c->sig_prev, sig, bytes, k, c->stream));
  if (is_host) B200_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int b200fem_get_state(b200fem_ctx *ctx, double *eps, double *sig) {
  Ctx *c = (Ctx *)ctx;
  if (!c->eps_prev) return B200FEM_E_INVALID;
  size_t bytes = (size_t)c->n_cells * 72 * sizeof(double);
  B200_CUDA(cudaMemcpyAsync(eps, c->eps_prev, bytes, cudaMemcpyDeviceToDevice, c->stream));
  B200_CUDA(cudaMemcpyAsync(sig, c->sig_prev, bytes, cudaMemcpyDeviceToDevice, c->stream));
  return 0;
}

int b200fem_norm2(const double *x, int64_t n, double *out_host, void *stream) {
  RedScratch r{};
  if (red_alloc(&r)) return B200FEM_E_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  int st = launch_dot(x, x, n, &r, s);
  double v = 0.0;
  if (!st && cudaMemcpyAsync(&v, r.result, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess) st = B200FEM_E_CUDA;
  if (!st && cudaStreamSynchronize(s) != cudaSuccess) st = B200FEM_E_CUDA;
  red_free(&r);
  *out_host = std::sqrt(v);
  return st;
}

int b200fem_dot(const double *x, const double *y, int64_t n, double *out_host, void *stream) {
  RedScratch r{};
  if (red_alloc(&r)) return B200FEM_E_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  int st = launch_dot(x, y, n, &r, s);
  double v = 0.0;
  if (!st && cudaMemcpyAsync(&v, r.result, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess) st = B200FEM_E_CUDA;
  if (!st && cudaStreamSynchronize(s) != cudaSuccess) st = B200FEM_E_CUDA;
  red_free(&r);
  *out_host = v;
  return st;
}

int b200fem_gather_sum(const double *x, const int64_t *idx, int64_t n, double *out_host, void *stream) {
  RedScratch r{};
  if (red_alloc(&r)) return B200FEM_E_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  int st = launch_gather_sum(x, idx, n, &r, s);
  double v = 0.0;
  if (!st && cudaMemcpyAsync(&v, r.result, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess) st = B200FEM_E_CUDA;
  if (!st && cudaStreamSynchronize(s) != cudaSuccess) st = B200FEM_E_CUDA;
  red_free(&r);
  *out_host = v;
  return st;
}

int b200fem_axpy(int64_t n, double a, const double *x, double *y, void *stream) {
  return launch_axpy(n, a, x, y, (cudaStream_t)stream);
}

int b200fem_scale(int64_t n, double a, const double *x, double *y, void *stream) {
  return launch_scale(n, a, x, y, (cudaStream_t)stream);
}

}  // extern "C"
