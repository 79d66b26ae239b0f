// Internal definitions shared by the libb200fem translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/b200fem.h"

namespace b200 {

// ---------------------------------------------------------------- launch grid
// Reduction kernels use a FIXED grid so that every per-block partial sum, and the
// order in which the last block combines them, is independent of the problem size
// tiling -> results are bit-identical run to run.  148 SMs x 8 blocks of 256 threads.
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRedBlocks = 148 * 8;
constexpr int kMaxVals = 16;  // values reduced per launch

extern std::atomic<int64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// -------------------------------------------------------------- error helpers
void set_err(b200fem_error *err, int code, const char *fmt, ...);
int cuda_status(cudaError_t e, b200fem_error *err, const char *where);
#define B200_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) return cuda_status(_e, nullptr, #call);               \
  } while (0)
#define B200_CUDA_E(call, err)                                                   \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) return cuda_status(_e, err, #call);                   \
  } while (0)

// ---------------------------------------------------- device error reporting
// Keys are cell*8+q (the reference reports the FIRST offender in (cell, qp) order,
// assembly.py:204-213); ULLONG_MAX = none.
struct DevErr {
  unsigned long long inv_def;   // NH det F <= 0
  unsigned long long nonfin_v;  // non-finite flux value
  unsigned long long nonfin_d;  // non-finite tangent
  unsigned long long inv_elem;  // det J <= 0 (geometry)
  unsigned long long min_detF;  // ordered-bits min of det F over offenders
  unsigned long long elem_det;  // ordered-bits det J of ... (min)
};

// ----------------------------------------------------------- scalar workspace
// Device-resident reduction scratch: partials[kRedBlocks * kMaxVals], a ticket for the
// last-block pattern and the reduced results.
struct RedScratch {
  double *partials;
  unsigned int *ticket;
  double *result;  // kMaxVals
};

// Krylov scalars live on the device so the inner loop never waits on the host.
enum : int { KS_RUNNING = 0, KS_CONV_INNER = 1, KS_BREAKDOWN = 2, KS_MAXED = 3 };
struct KrylovScalars {
  double rho, alpha, omega, beta;
  double r0v, tt, ts;
  double res, tol;
  long long mv;
  double r0r0, r0r, rr;
  long long it, max_iters;
  int status, first;
};

struct MatParams {
  double alpha, lam, mu, kappa, sy, penalty;
  int simp, design_source;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n_nodes = 0, n_cells = 0, n_dofs = 0, nnz = 0;
  int vec = 1, material = 0, flags = 0;
  MatParams mp{};
  double *coords = nullptr;   // (n_nodes,3)
  int32_t *cells = nullptr;   // (n_cells,8)
  int32_t *nbr_ptr = nullptr; // (n_nodes+1) node adjacency (includes self)
  int32_t *nbr = nullptr;     // sorted neighbour node ids
  int32_t *indptr = nullptr;  // (n_dofs+1)
  int32_t *indices = nullptr; // lazily materialised (vec==1 aliases nbr)
  uint8_t *cpos = nullptr;    // (n_cells,64) position of node b in node a's neighbour list
  int32_t *diag = nullptr;    // (n_dofs) diagonal slot
  // symmetric node-block storage (vec 3): upper blocks (m >= n) of node n at up_ptr[n],
  // 3x3 row-major; lo_blk[nbr_ptr[n] + j] = block index of (m, n) for the lower neighbours
  int32_t *up_ptr = nullptr;  // (n_nodes+1)
  int32_t *lo_blk = nullptr;  // (total neighbours) only lower entries used
  int64_t n_sym_blocks = 0;
  // GRID3 (vec 3 box lattices, see spmv.cu): nodes per axis (0 = not a lattice) and the
  // padded length of each of the 14 offset arrays of upper node blocks
  int grid_nx = 0, grid_ny = 0, grid_nz = 0;
  int64_t grid_npad = 0;
  int max_nbr = 0;
  int max_deg = 0;              // max cells per node
  int32_t *n2c_ptr = nullptr;   // (n_nodes+1) node -> incident cells, ascending cell id
  int32_t *n2c = nullptr;
  uint8_t *n2c_a = nullptr;     // local index (0..7) of the node in each incident cell
  uint8_t *dir_flag = nullptr;  // (n_dofs) 1 on Dirichlet rows
  double *scratch = nullptr;    // per-cell element blocks (two-phase assembly)
  size_t scratch_len = 0;
  // boundary data
  int64_t n_dir = 0;
  int32_t *dir_dofs = nullptr;
  double *dir_vals = nullptr;
  double *f_neumann = nullptr, *f_body = nullptr;
  double *theta = nullptr;
  int64_t n_theta = 0;
  double *eps_prev = nullptr, *sig_prev = nullptr;
  // scratch
  DevErr *derr = nullptr;
  RedScratch red{};
  double *pinned = nullptr;  // host pinned scratch (8 doubles)
};

struct KrylovWork {
  int64_t n = 0;
  double *r = nullptr, *r0 = nullptr, *p = nullptr, *v = nullptr, *s = nullptr, *t = nullptr;
  double *diag = nullptr, *inv = nullptr;
  KrylovScalars *sc = nullptr;
  KrylovScalars *sc_host = nullptr;  // pinned
  RedScratch red{};
  cudaEvent_t ev[2]{};
};

enum MatKind : int { MK_CSR = 0, MK_FEM3 = 1, MK_SYM3 = 2, MK_GRID3 = 3 };
struct Matrix {
  MatKind kind = MK_CSR;
  int64_t n = 0, nnz = 0;
  const int32_t *indptr = nullptr, *indices = nullptr;  // CSR
  const int32_t *nbr_ptr = nullptr, *nbr = nullptr;     // FEM3
  const int32_t *diag_slots = nullptr;                  // FEM3 (optional fast diagonal)
  const double *data = nullptr;
  cudaStream_t stream = nullptr;
  int lanes = 8;  // CSR sub-warp width
  KrylovWork *kw = nullptr;
  // FEM3 bulk-copy pipeline: node chunks [chunk_node[c], chunk_node[c+1]) sized to a stage
  int32_t *chunk_node = nullptr;
  int n_chunks = 0;
  bool use_tma = false;
  int npw = 2;  // bulk-copy SpMV: nodes per consumer warp (2: half-warp per node; 1: warp per node)
  // rows computed by matvec/Krylov: node range (FEM3) or row range (CSR); -1 = all
  int64_t row_lo = 0, row_hi = -1;
  // Dirichlet identity rows (FEM matrices): PCG starts from x_d = b_d so that the Krylov
  // space stays in {v : v_d = 0}, where the row-replaced K acts as the SPD block K_ff
  const int32_t *dir_dofs = nullptr;
  int64_t n_dir = 0;
  // SYM3: upper node blocks (pre-Dirichlet) + Dirichlet row flags applied on output rows
  const int32_t *up_ptr = nullptr, *lo_blk = nullptr;
  const uint8_t *dir_flag = nullptr;
  // GRID3: lattice nodes per axis and the padded offset-array length (data = 14 arrays)
  int gnx = 0, gny = 0, gnz = 0, gvec = 3;
  int64_t gnpad = 0;
  const float *data32 = nullptr;  // GRID3 vec 3: single-precision copy used by the matvec
};

// ------------------------------------------------------------------ GRID3 offsets
// The 14 lattice offsets (di, dj, dk) with (dk, dj, di) lexicographically >= 0: the self
// block and the 13 "upper" neighbours of a node in a z-major box lattice (node id
// i + NX j + NX NY k, mesh.py:152-158).  Offset k of node n stores the 3x3 block
// K[(n, n + off_k)] in array k (row-major, pre-Dirichlet); the lower block of
// (n, n - off_k) is the transpose of array k's block of node n - off_k.
__host__ __device__ constexpr int grid_di(int k) {
  return k == 0 ? 0 : k == 1 ? 1 : k <= 4 ? k - 3 : (k - 5) % 3 - 1;
}
__host__ __device__ constexpr int grid_dj(int k) { return k <= 1 ? 0 : k <= 4 ? 1 : (k - 5) / 3 - 1; }
__host__ __device__ constexpr int grid_dk(int k) { return k <= 4 ? 0 : 1; }
// index of lattice offset (di, dj, dk) among the 14, or -1 for a "lower" offset
__host__ __device__ inline int grid_index(int di, int dj, int dk) {
  if (dk == 1) return 5 + 3 * (dj + 1) + (di + 1);
  if (dk != 0) return -1;
  if (dj == 1) return 3 + di;
  if (dj != 0) return -1;
  return di == 0 ? 0 : di == 1 ? 1 : -1;
}
// GRID3 value layout (tiled by 32 nodes): value e (0..8, row-major) of the block at offset k
// of node n.  npad = 32 * ceil(n_nodes / 32).  A warp's 32 consecutive nodes read one
// contiguous 256-byte segment per (k, e), and a thread's 9 values sit at +256 B strides.
// (vec 1: one value per block, vv = 1)
__host__ __device__ inline int64_t grid_idx(int k, int e, int64_t n, int64_t npad, int vv = 9) {
  return (((int64_t)k * (npad >> 5) + (n >> 5)) * vv + e) * 32 + (n & 31);
}
int prepare_grid3(Matrix *m);

// allocation helpers
template <class T>
inline cudaError_t dalloc(T **p, size_t n) {
  return cudaMalloc((void **)p, (n ? n : 1) * sizeof(T));
}
int red_alloc(RedScratch *r);
int xr_blocks();  // grid of k_update_xr (krylov.cu)
void red_free(RedScratch *r);

// ---------------------------------------------------------------- launchers
// reductions (deterministic): out_host may be null (result stays in r->result)
int launch_dot(const double *x, const double *y, int64_t n, RedScratch *r, cudaStream_t s);
int launch_gather_sum(const double *x, const int64_t *idx, int64_t n, RedScratch *r, cudaStream_t s);
int launch_axpy(int64_t n, double a, const double *x, double *y, cudaStream_t s);
int launch_scale(int64_t n, double a, const double *x, double *y, cudaStream_t s);

// sparse
enum SpmvMode : int { SP_PLAIN = 0, SP_JACOBI_R0 = 1, SP_JACOBI_TT = 2, SP_RESIDUAL = 3, SP_PQ = 4, SP_CGRES = 5 };
struct SpmvArgs {
  const double *x;   // operand (p, s or x)
  double *y;         // output (v, t or r)
  const double *inv; // inverse diagonal
  const double *dg;  // diagonal (residual mode)
  const double *aux; // r0 (mode 1), b (mode 3)
  double *aux2;      // r0 copy target (mode 3)
  KrylovScalars *sc; // status gate (null -> always run)
  int inline_stage;  // 1: the last block applies the scalar update (one rank);
                     // 0: totals are left in red.result for a cross-rank allreduce
};
int launch_spmv(const Matrix *m, SpmvMode mode, const SpmvArgs &a, RedScratch *red);
int launch_diagonal(const Matrix *m, double *diag, double *inv, RedScratch *red, int64_t *n_zero);
int prepare_fem3_chunks(Matrix *m, int64_t node_lo = 0, int64_t node_hi = -1);
int prepare_sym3_chunks(Matrix *m);

// element kernels
int launch_residual(Ctx *c, const double *U, double *R, double bc_scale, int apply_dirichlet,
                    b200fem_error *err, double *norm_host);
int launch_jacobian(Ctx *c, const double *U, double *data, b200fem_error *err, double *sym = nullptr,
                    double *grid = nullptr);
int launch_qp_flux(Ctx *c, const double *U, double *out, b200fem_error *err);
int launch_volume_average(Ctx *c, const double *U, double *out_host, b200fem_error *err);
int launch_commit(Ctx *c, const double *U);
int check_geometry(Ctx *c, b200fem_error *err);
void element_tables_init();
int fetch_element_errors(Ctx *c, b200fem_error *err, bool jacobian);

// Krylov (krylov.cu)
int ensure_work(Matrix *m);
void free_work(KrylovWork *w);
__global__ void k_begin(KrylovScalars *S);
__global__ void __launch_bounds__(kThreads) k_update_p(int64_t n, const double *__restrict__ r, const double *__restrict__ v,
                           double *__restrict__ p, const KrylovScalars *S);
__global__ void __launch_bounds__(kThreads) k_update_s(int64_t n, const double *__restrict__ r, const double *__restrict__ v,
                           double *__restrict__ s, const KrylovScalars *S);
__global__ void __launch_bounds__(kThreads) k_update_xr(int64_t n, double *__restrict__ x, double *__restrict__ r, const double *__restrict__ p,
                            const double *__restrict__ s, const double *__restrict__ t,
                            const double *__restrict__ r0, const double *__restrict__ dg, KrylovScalars *S,
                            RedScratch red, int inline_stage);
int bicgstab(Matrix *m, const double *b, double *x, int has_x0, double rel_tol, double abs_tol,
             int64_t max_iters, b200fem_solve_info *info, b200fem_error *err);
__global__ void k_begin_cg(KrylovScalars *S);
__global__ void k_set_dirichlet(double *__restrict__ x, const double *__restrict__ b, const int32_t *__restrict__ d,
                                int64_t n);
__global__ void __launch_bounds__(kThreads) k_cg_update_xrz(int64_t n, double *__restrict__ x, double *__restrict__ r,
                                                            const double *__restrict__ p, const double *__restrict__ q,
                                                            const double *__restrict__ inv, double *__restrict__ z,
                                                            KrylovScalars *S, RedScratch red, int inline_stage);
__global__ void __launch_bounds__(kThreads) k_cg_update_p(int64_t n, const double *__restrict__ z,
                                                          double *__restrict__ p, const KrylovScalars *S);

// ------------------------------------------------------ Krylov scalar stages
// BiCGSTAB iteration start (solvers.py:131-139): it += 1, rho_new = r0.r, breakdown test, beta.
__device__ __forceinline__ void iter_start(KrylovScalars *S) {
  if (S->it >= S->max_iters) {
    S->status = KS_MAXED;
    return;
  }
  S->it += 1;
  const double rho_new = S->r0r;
  const double scale = sqrt(S->r0r0) * sqrt(S->rr);
  const bool broke = fabs(rho_new) <= 1e-30 * scale || (!S->first && S->omega == 0.0);
  if (broke) {
    S->status = KS_BREAKDOWN;
    return;
  }
  S->beta = S->first ? 0.0 : (rho_new / S->rho) * (S->alpha / S->omega);
  S->first = 0;
  S->rho = rho_new;
}

enum StageKind : int { ST_R0 = 1, ST_TT = 2, ST_RES = 3, ST_XR = 4, ST_PQ = 5, ST_CGRES = 6, ST_CGXR = 7, ST_TT8 = 8, ST_CONV = 9 };
// Scalar update after a reduction with global totals tot[] (solvers.py:141-167).
__device__ __forceinline__ void apply_stage(int kind, KrylovScalars *S, const double *tot) {
  if (!S || S->status != KS_RUNNING) return;
  if (kind == ST_R0) {
    S->mv += 1;
    S->r0v = tot[0];
    if (tot[0] == 0.0) S->status = KS_BREAKDOWN;
    else S->alpha = S->rho / tot[0];
  } else if (kind == ST_TT) {
    S->mv += 1;
    S->tt = tot[0];
    S->ts = tot[1];
    S->omega = tot[0] > 0.0 ? tot[1] / tot[0] : 0.0;
  } else if (kind == ST_RES) {
    S->mv += 1;
    S->res = sqrt(tot[0]);
    S->r0r0 = S->r0r = S->rr = tot[1];
  } else if (kind == ST_XR) {
    S->res = sqrt(tot[0]);
    S->r0r = tot[1];
    S->rr = tot[2];
    if (S->res <= S->tol) {
      S->status = KS_CONV_INNER;
      return;
    }
    iter_start(S);
  } else if (kind == ST_TT8) {
    // partitioned BiCGSTAB with two allreduces per iteration (>= 4 NCCL ranks): the t-group carries
    // {t.t, t.s, r0.s, r0.t, s.s, |Ds|^2, Ds.Dt, |Dt|^2}; omega as in ST_TT, then the next
    // r = s - omega t enters only through the recurrences r0.r, r.r, |Dr|^2 (clamped at 0)
    S->mv += 1;
    S->tt = tot[0];
    S->ts = tot[1];
    const double om = tot[0] > 0.0 ? tot[1] / tot[0] : 0.0;
    S->omega = om;
    S->r0r = tot[2] - om * tot[3];
    S->rr = fmax(tot[4] - 2.0 * om * tot[1] + om * om * tot[0], 0.0);
    S->res = sqrt(fmax(tot[5] - 2.0 * om * tot[6] + om * om * tot[7], 0.0));
  } else if (kind == ST_CONV) {  // after the x, r update of the ST_TT8 flow: as the end of ST_XR
    if (S->res <= S->tol) {
      S->status = KS_CONV_INNER;
      return;
    }
    iter_start(S);
  } else if (kind == ST_PQ) {  // Jacobi-PCG: alpha = (r.z) / (p.Ap); p.Ap <= 0 -> not SPD
    S->mv += 1;
    S->r0v = tot[0];
    if (!(tot[0] > 0.0)) S->status = KS_BREAKDOWN;
    else S->alpha = S->rho / tot[0];
  } else if (kind == ST_CGRES) {  // explicit residual: ||r||, r.z (p = z)
    S->mv += 1;
    S->res = sqrt(tot[0]);
    S->rho = tot[1];
  } else {  // ST_CGXR: after x += alpha p, r -= alpha q, z = D^-1 r
    S->res = sqrt(tot[0]);
    if (S->res <= S->tol) {
      S->status = KS_CONV_INNER;
      return;
    }
    if (S->it >= S->max_iters) {
      S->status = KS_MAXED;
      return;
    }
    S->it += 1;
    S->beta = tot[1] / S->rho;
    S->rho = tot[1];
  }
}

// ------------------------------------------------------------ device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of NV values per thread; result valid in thread 0.
template <int NV, int NW = kWarps>
__device__ __forceinline__ void block_reduce(double (&v)[NV], double (*sh)[NW]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) sh[j][w] = v[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double a = 0.0;
      for (int k = 0; k < NW; ++k) a += sh[j][k];
      v[j] = a;
    }
  }
}

// Write this block's partials; return true in ALL threads of the last block to finish,
// which then holds the fully reduced values in `tot` (thread 0 valid).
template <int NV, int NW = kWarps>
__device__ __forceinline__ bool block_partials_and_finish(double (&v)[NV], RedScratch red,
                                                          double (&tot)[NV]) {
  __shared__ double sh[NV][NW];
  __shared__ bool last;
  block_reduce<NV, NW>(v, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) red.partials[j * kRedBlocks + blockIdx.x] = v[j];
    __threadfence();
    unsigned t = atomicAdd(red.ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double a = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      a += __ldcg(red.partials + j * kRedBlocks + b);
    acc[j] = a;
  }
  __syncthreads();
  block_reduce<NV, NW>(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      tot[j] = acc[j];
      red.result[j] = acc[j];
    }
    *red.ticket = 0u;
  }
  return true;
}

}  // namespace b200
