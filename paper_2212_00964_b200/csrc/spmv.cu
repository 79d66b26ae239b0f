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

#include <algorithm>
#include <vector>

#include <cstring>

#include "internal.cuh"
#include "spmv_common.cuh"

namespace b200 {

template <int MODE>
__global__ void __launch_bounds__(kThreads, 4) k_spmv_fem3(const int32_t *__restrict__ nbr_ptr,
                                                        const int32_t *__restrict__ nbr,
                                                        const double *__restrict__ data, int64_t node_lo,
                                                        int64_t n_nodes, SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double *__restrict__ x = a.x;
  double red0 = 0.0, red1 = 0.0;
  for (int64_t n = node_lo + warp0; n < n_nodes; n += nwarps) {
    const int p0 = __ldg(nbr_ptr + n);
    const int cnt = __ldg(nbr_ptr + n + 1) - p0;
    const int L = 3 * cnt;
    const double *__restrict__ blk = data + 9 * (int64_t)p0;
    const bool row_lane = (lane & 7) == 0 && lane < 24;
    const int64_t row = 3 * n + (lane >> 3);
    RowPre pre{0.0, 0.0, 0.0, 0.0};
    if (row_lane) pre = spmv_preload<MODE>(row, a);
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int j = lane; j < cnt; j += 32) {
      const int m = __ldg(nbr + p0 + j);
      const double *__restrict__ xm = x + 3 * (int64_t)m;
      const double *__restrict__ r0 = blk + 3 * j;
      const double a00 = __ldcs(r0), a01 = __ldcs(r0 + 1), a02 = __ldcs(r0 + 2);
      const double a10 = __ldcs(r0 + L), a11 = __ldcs(r0 + L + 1), a12 = __ldcs(r0 + L + 2);
      const double a20 = __ldcs(r0 + 2 * L), a21 = __ldcs(r0 + 2 * L + 1), a22 = __ldcs(r0 + 2 * L + 2);
      const double x0 = __ldg(xm), x1 = __ldg(xm + 1), x2 = __ldg(xm + 2);
      y0 = fma(a02, x2, fma(a01, x1, fma(a00, x0, y0)));
      y1 = fma(a12, x2, fma(a11, x1, fma(a10, x0, y1)));
      y2 = fma(a22, x2, fma(a21, x1, fma(a20, x0, y2)));
    }
    const double acc = warp_sum3(y0, y1, y2, lane);
    if (row_lane) spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage) spmv_stage<MODE>(a.sc, tot);
  }
}

// ------------------------------------------------------------------------------------
// SYM3: symmetric node-block operator.  The assembled tangent of every supported law is
// exactly symmetric before the Dirichlet row replacement (K_mn = K_nm^T bit for bit: each
// per-cell block pair is one stored block and its transpose, summed in the same cell order),
// so only the upper blocks (m >= n, 3x3 row-major) are stored: 14 of 27 blocks per interior
// node.  Row n = sum over upper blocks B_nm x_m + sum over lower neighbours B_mn^T x_m; the
// lower blocks were streamed moments earlier as upper blocks of rows m < n and are served
// by L2.  Dirichlet rows act as identity rows (y_d = x_d), exactly the row-replaced K of
// assembly.py:297-299.  DRAM bytes per matvec drop from 8 B/nnz to ~4.2 B/nnz.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 4) k_spmv_sym3(const int32_t *__restrict__ nbr_ptr,
                                                           const int32_t *__restrict__ nbr,
                                                           const int32_t *__restrict__ up_ptr,
                                                           const int32_t *__restrict__ lo_blk,
                                                           const double *__restrict__ sym,
                                                           const uint8_t *__restrict__ dir_flag, int64_t node_lo,
                                                           int64_t n_nodes, SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double *__restrict__ x = a.x;
  double red0 = 0.0, red1 = 0.0;
  // metadata of the warp's next node is prefetched one node ahead so that the block and
  // x loads of a node are issued in a single memory round trip
  int64_t n = node_lo + warp0;
  int nx_p0 = 0, nx_cnt = 0, nx_ub = 0, nx_uc = 0, nx_m = 0, nx_lb = 0;
  auto fetch = [&](int64_t k) {
    nx_p0 = __ldg(nbr_ptr + k);
    nx_cnt = __ldg(nbr_ptr + k + 1) - nx_p0;
    nx_ub = __ldg(up_ptr + k);
    nx_uc = __ldg(up_ptr + k + 1) - nx_ub;
    nx_m = lane < nx_cnt ? __ldg(nbr + nx_p0 + lane) : 0;
    nx_lb = lane < nx_cnt - nx_uc ? __ldg(lo_blk + nx_p0 + lane) : 0;
  };
  if (n < n_nodes) fetch(n);
  for (; n < n_nodes; n += nwarps) {
    const int p0 = nx_p0, cnt = nx_cnt, ub = nx_ub, self = cnt - nx_uc, m0 = nx_m, lb0 = nx_lb;
    const bool row_lane = (lane & 7) == 0 && lane < 24;
    const int64_t row = 3 * n + (lane >> 3);
    RowPre pre{0.0, 0.0, 0.0, 0.0};
    bool dflag = false;
    double xrow = 0.0;
    if (row_lane) {
      pre = spmv_preload<MODE>(row, a);
      dflag = dir_flag && __ldg(dir_flag + row);
      if (dflag) xrow = __ldg(x + row);
    }
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int j = lane; j < cnt; j += 32) {
      const int m = j == lane ? m0 : __ldg(nbr + p0 + j);
      const bool lower = j < self;
      const int blk = lower ? (j == lane ? lb0 : __ldg(lo_blk + p0 + j)) : ub + (j - self);
      const double *__restrict__ B = sym + 9 * (int64_t)blk;
      const double b00 = __ldg(B), b01 = __ldg(B + 1), b02 = __ldg(B + 2);
      const double b10 = __ldg(B + 3), b11 = __ldg(B + 4), b12 = __ldg(B + 5);
      const double b20 = __ldg(B + 6), b21 = __ldg(B + 7), b22 = __ldg(B + 8);
      const double *__restrict__ xm = x + 3 * (int64_t)m;
      const double x0 = __ldg(xm), x1 = __ldg(xm + 1), x2 = __ldg(xm + 2);
      // lower neighbours use the transposed block
      const double a01 = lower ? b10 : b01, a02 = lower ? b20 : b02, a10 = lower ? b01 : b10;
      const double a12 = lower ? b21 : b12, a20 = lower ? b02 : b20, a21 = lower ? b12 : b21;
      y0 = fma(a02, x2, fma(a01, x1, fma(b00, x0, y0)));
      y1 = fma(a12, x2, fma(b11, x1, fma(a10, x0, y1)));
      y2 = fma(b22, x2, fma(a21, x1, fma(a20, x0, y2)));
    }
    if (n + nwarps < n_nodes) fetch(n + nwarps);
    double acc = warp_sum3(y0, y1, y2, lane);
    if (row_lane) {
      if (dflag) acc = xrow;  // identity row
      spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
    }
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage) spmv_stage<MODE>(a.sc, tot);
  }
}

// Two nodes per consumer warp (half-warp per node, two neighbours per lane): the per-node
// bookkeeping (chunk/pointer loads, address math, barrier waits) is shared by two nodes, so
// the warp-instruction count per node roughly halves -- less SM energy per byte, which is
// what limits the kernel once a long solve runs into the board power cap.  16 consumer warps
// keep the same number of gathers in flight as 31 warps with one neighbour per lane.
constexpr int kT2Consumers = 16;
constexpr int kT2Threads = (kT2Consumers + 1) * 32;
constexpr int kT2ExtBytes = 800;  // <= 96 rows + alignment slack
constexpr int kT2StageBytes = kTmaValBytes + kTmaNbrBytes + 3 * kT2ExtBytes;
constexpr int kT2Smem = kTmaStages * kT2StageBytes + 2 * kTmaStages * 8;

// 16-lane reduce-scatter of three row partials: lanes 0, 4, 8 of each half-warp end with
// rows 0, 1, 2 (full-warp shuffles; both halves reduce independently).
__device__ __forceinline__ double half_sum3(double y0, double y1, double y2, int lane) {
  const bool h8 = lane & 8;
  const double s0 = h8 ? y0 : y2, s1 = h8 ? y1 : 0.0;
  double k0 = (h8 ? y2 : y0) + __shfl_xor_sync(0xffffffffu, s0, 8);
  double k1 = (h8 ? 0.0 : y1) + __shfl_xor_sync(0xffffffffu, s1, 8);
  const bool h4 = lane & 4;
  double kk = (h4 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h4 ? k0 : k1, 4);
  kk += __shfl_xor_sync(0xffffffffu, kk, 2);
  kk += __shfl_xor_sync(0xffffffffu, kk, 1);
  return kk;
}

template <int MODE>
__global__ void __launch_bounds__(kT2Threads, 1) k_spmv_fem3_tma2(const int32_t *__restrict__ nbr_ptr,
                                                                 const int32_t *__restrict__ nbr,
                                                                 const double *__restrict__ data,
                                                                 const int32_t *__restrict__ chunk_node, int n_chunks,
                                                                 int64_t total_blocks, int64_t n_rows, SpmvArgs a,
                                                                 RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kTmaStages * kT2StageBytes);
  uint64_t *empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kT2Consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t val_end = (uint64_t)total_blocks * 72, nbr_end = (uint64_t)total_blocks * 4;
  const uint64_t row_end = (uint64_t)n_rows * 8;
  double red0 = 0.0, red1 = 0.0;
  if (warp == kT2Consumers) {
    if (lane == 0) {  // producer
      int it = 0;
      for (int c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
        const int s = it % kTmaStages;
        const uint32_t ph = (it / kTmaStages) & 1;
        mbar_wait(empty + s, ph ^ 1);
        const int64_t cn0 = __ldg(chunk_node + c), cn1 = __ldg(chunk_node + c + 1);
        const int64_t p0 = __ldg(nbr_ptr + cn0), p1 = __ldg(nbr_ptr + cn1);
        const uint64_t vb0 = (72ull * p0) & ~15ull, vb1 = std::min((72ull * p1 + 15) & ~15ull, val_end & ~15ull);
        const uint64_t nb0 = (4ull * p0) & ~15ull, nb1 = std::min((4ull * p1 + 15) & ~15ull, nbr_end & ~15ull);
        const uint64_t eb0 = (24ull * cn0) & ~15ull, eb1 = std::min((24ull * cn1 + 15) & ~15ull, row_end & ~15ull);
        const uint32_t ext_bytes = eb1 > eb0 ? (uint32_t)(eb1 - eb0) : 0u;
        mbar_expect_tx(full + s, (uint32_t)((vb1 - vb0) + (nb1 - nb0)) + n_ext<MODE>() * ext_bytes);
        uint8_t *stage = smem + s * kT2StageBytes;
        if (vb1 > vb0) bulk_g2s(stage, reinterpret_cast<const uint8_t *>(data) + vb0, (uint32_t)(vb1 - vb0), full + s);
        if (nb1 > nb0)
          bulk_g2s(stage + kTmaValBytes, reinterpret_cast<const uint8_t *>(nbr) + nb0, (uint32_t)(nb1 - nb0), full + s);
#pragma unroll
        for (int k = 0; k < n_ext<MODE>(); ++k)
          if (ext_bytes)
            bulk_g2s(stage + kTmaValBytes + kTmaNbrBytes + k * kT2ExtBytes,
                     reinterpret_cast<const uint8_t *>(ext_ptr<MODE>(a, k)) + eb0, ext_bytes, full + s);
      }
    }
    __syncwarp();
  } else {
    const int hl = lane & 15;
    const bool row_lane = (hl & 3) == 0 && hl < 12;
    int it = 0;
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
      const int s = it % kTmaStages;
      const uint32_t ph = (it / kTmaStages) & 1;
      const int n0 = __ldg(chunk_node + c), n1 = __ldg(chunk_node + c + 1);
      const int64_t pc = __ldg(nbr_ptr + n0), pe = __ldg(nbr_ptr + n1);
      const uint64_t vb0 = (72ull * pc) & ~15ull, nb0 = (4ull * pc) & ~15ull;
      const bool tail = (72ull * pe > (val_end & ~15ull)) || (4ull * pe > (nbr_end & ~15ull)) ||
                        (n_ext<MODE>() > 0 && 24ull * n1 > (row_end & ~15ull));
      const uint64_t eb0 = (24ull * n0) & ~15ull;
      const uint8_t *stage = smem + s * kT2StageBytes;
      const int nA = n0 + 2 * warp + (lane >> 4);
      const bool has = nA < n1;
      int64_t pA = 0;
      int cA = 0;
      if (has) {
        pA = __ldg(nbr_ptr + nA);
        cA = __ldg(nbr_ptr + nA + 1) - (int)pA;
      }
      const int64_t row = 3 * (int64_t)nA + (hl >> 2);
      RowPre pre{0.0, 0.0, 0.0, 0.0};
      if (tail && row_lane && has) pre = spmv_preload<MODE>(row, a);
      mbar_wait(full + s, ph);
      if (!tail && row_lane && has && n_ext<MODE>() > 0) {
        const uint8_t *ext = stage + kTmaValBytes + kTmaNbrBytes + (8ull * row - eb0);
        pre = row_pre_from<MODE>(reinterpret_cast<const double *>(ext),
                                 reinterpret_cast<const double *>(ext + kT2ExtBytes),
                                 reinterpret_cast<const double *>(ext + 2 * kT2ExtBytes));
      }
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      if (has) {
        const double *sv = tail ? data + 9 * pA : reinterpret_cast<const double *>(stage + (72ull * pA - vb0));
        const int32_t *sn = tail ? nbr + pA : reinterpret_cast<const int32_t *>(stage + kTmaValBytes + (4ull * pA - nb0));
        const int L = 3 * cA;
        for (int j = hl; j < cA; j += 32) {  // both neighbours' gathers in flight together
          const int j2 = j + 16;
          const bool two = j2 < cA;
          double x0, x1, x2, z0 = 0.0, z1 = 0.0, z2 = 0.0;
          load_x3<0>(a.x, sn[j], x0, x1, x2);
          if (two) load_x3<0>(a.x, sn[j2], z0, z1, z2);
          const double *r0 = sv + 3 * j;
          y0 = fma(r0[2], x2, fma(r0[1], x1, fma(r0[0], x0, y0)));
          y1 = fma(r0[L + 2], x2, fma(r0[L + 1], x1, fma(r0[L], x0, y1)));
          y2 = fma(r0[2 * L + 2], x2, fma(r0[2 * L + 1], x1, fma(r0[2 * L], x0, y2)));
          if (two) {
            const double *r1 = sv + 3 * j2;
            y0 = fma(r1[2], z2, fma(r1[1], z1, fma(r1[0], z0, y0)));
            y1 = fma(r1[L + 2], z2, fma(r1[L + 1], z1, fma(r1[L], z0, y1)));
            y2 = fma(r1[2 * L + 2], z2, fma(r1[2 * L + 1], z1, fma(r1[2 * L], z0, y2)));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      const double acc = half_sum3(y0, y1, y2, lane);
      if (has && row_lane) spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
    }
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2, kT2Consumers + 1>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage)
      spmv_stage<MODE>(a.sc, tot);
  }
}

static void set_t2_attr() {
  cudaFuncSetAttribute(k_spmv_fem3_tma2<SP_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem);
  cudaFuncSetAttribute(k_spmv_fem3_tma2<SP_JACOBI_R0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem);
  cudaFuncSetAttribute(k_spmv_fem3_tma2<SP_JACOBI_TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem);
  cudaFuncSetAttribute(k_spmv_fem3_tma2<SP_RESIDUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem);
  cudaFuncSetAttribute(k_spmv_fem3_tma2<SP_PQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem);
  cudaFuncSetAttribute(k_spmv_fem3_tma2<SP_CGRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem);
}

static int tma_npw_env() {  // B200FEM_SPMV_NPW=1 selects the warp-per-node kernel (read per matrix)
  const char *e = getenv("B200FEM_SPMV_NPW");
  return (e && !strcmp(e, "1")) ? 1 : 2;
}

// Pack consecutive nodes into chunks whose values + neighbour ids fit one stage
// (with 16-byte alignment slack), at most one node per consumer warp.
int prepare_fem3_chunks(Matrix *m, int64_t lo, int64_t hi) {
  const int64_t nn = m->n / 3;
  if (hi < 0) hi = nn;
  std::vector<int32_t> ptr(nn + 1);
  if (cudaMemcpy(ptr.data(), m->nbr_ptr, (nn + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return B200FEM_E_CUDA;
  cudaFree(m->chunk_node);
  m->chunk_node = nullptr;
  m->use_tma = false;
  m->npw = tma_npw_env();
  std::vector<int32_t> ch{(int32_t)lo};
  int64_t start = lo;
  for (int64_t n = lo; n < hi; ++n) {
    const int64_t nb = ptr[n + 1] - ptr[start];
    const int max_nodes = m->npw == 2 ? 2 * kT2Consumers : kTmaConsumers;
    const bool fits = 72 * nb + 32 <= kTmaValBytes && 4 * nb + 32 <= kTmaNbrBytes && (n + 1 - start) <= max_nodes;
    if (!fits) {
      if (n == start) return 0;  // a single node does not fit a stage: keep the LDG kernel
      ch.push_back((int32_t)n);
      start = n;
    }
  }
  ch.push_back((int32_t)hi);
  m->n_chunks = (int)ch.size() - 1;
  if (dalloc(&m->chunk_node, ch.size()) != cudaSuccess) return B200FEM_E_CUDA;
  if (cudaMemcpy(m->chunk_node, ch.data(), ch.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess)
    return B200FEM_E_CUDA;
  static bool attr = false;
  if (!attr) {
    set_fem3_tma_npw1_attr();  // spmv_alt.cu
    set_t2_attr();
    attr = true;
  }
  m->use_tma = true;
  return 0;
}

// ------------------------------------------------------------------------------------
// GRID3: symmetric storage for z-major box lattices (generate_box_mesh, mesh.py:134-168).
//
// The tangent is symmetric outside the Dirichlet rows (which the reference replaces by
// identity rows, assembly.py:297-299), and the node coupling of a lattice is the 27-point
// stencil.  Only the self block and the 13 upper-offset blocks of every node are stored,
// pre-Dirichlet, as 126 element streams tiled by 32 nodes: value e (0..8, row-major) of the
// block K[(n, n + off_k)] sits at grid[grid_idx(k, e, n)] (offsets k = 0..13, internal.cuh).
// Row block a is
//     y_a = sum_k B_k[a] x_{a + off_k}  +  sum_{k >= 1} B_k[a - off_k]^T x_{a - off_k}
// With a thread per node, every value load of a warp is one contiguous 256-byte segment,
// for the upper blocks (index a) and for the lower ones alike (index a - off_k): no column
// indices, no gather.  The lower values were streamed as upper values of node a - off_k at
// most one lattice plane earlier (~19 MB at config 3) and are re-read from L2; the grid-stride
// chunk order keeps all warps on one wavefront so they still are (ncu: 2.73 GB of DRAM reads
// per launch against 2.66 GB algorithmic).
// DRAM per matvec: 14*72 B per node + x + y = 2.72 GB at config 3 (FEM3 CSR: 5.33 GB).
// Dirichlet rows give y = x (identity rows).  Summation order is fixed -> deterministic.
constexpr int kGThreads = 256;
constexpr int kGMinBlocks = 1;  // 255 registers: ILP per thread beats more warps (2/SM: +41 %)
#ifndef GRID32_MIN_BLOCKS
#define GRID32_MIN_BLOCKS 2
#endif
constexpr int kGMinBlocks32 = GRID32_MIN_BLOCKS;  // FP32 copy: 2 CTAs/SM at 128 registers, 328 us vs 389 us at 1 (3: 333 us)

struct GridDims {
  int nx, ny, nz, nxy, nn;  // nodes per axis, per plane, total
  int64_t npad;             // element-array length
  int slab;                 // rows per slab of the slab-major traversal (0: plain node order)
};

struct LatticePos {  // which faces of the lattice node a lies on
  bool i0, iN, j0, jN, k0, kN;
};
// Lattice coordinates of node a = c0 + t from those of the chunk start (the divisions are
// warp-uniform) plus a carry walk.
__device__ __forceinline__ LatticePos lattice_pos(int a, int c0, const GridDims &g) {
  int k = c0 / g.nxy, rem = c0 - k * g.nxy, j = rem / g.nx, i = rem - j * g.nx;
  i += a - c0;
  while (i >= g.nx) {
    i -= g.nx;
    if (++j == g.ny) j = 0, ++k;
  }
  return {i == 0, i == g.nx - 1, j == 0, j == g.ny - 1, k == 0, k == g.nz - 1};
}
// lattice neighbour (di, dj, dk) exists (compile-time offsets fold to predicate logic)
__device__ __forceinline__ bool grid_has(const LatticePos &p, int di, int dj, int dk) {
  return !((di < 0 && p.i0) || (di > 0 && p.iN) || (dj < 0 && p.j0) || (dj > 0 && p.jN) || (dk < 0 && p.k0) ||
           (dk > 0 && p.kN));
}

// Traversal order of the GRID3 matvec.  Every upper block of node m is read a second time,
// transposed, by node m + off as one of its lower blocks; in plain node order 9 of the 13
// offsets span a whole lattice plane, so that second read comes one plane (+ one wave of
// 148 x 256 nodes) later and misses L2 once the plane outgrows it (ncu DRAM bytes over the
// algorithmic bytes: +3 % at 136^3, +18 % at 160^3, +40 % at 200^3).  Slab-major order walks
// slabs of `slab` rows through all planes (for s: for k: rows [s*slab, (s+1)*slab) of plane
// k), which bounds the reuse distance by slab * nx nodes for any lattice size; only the
// first / last row of a slab re-reads across the slab boundary.  Work item w is a (slab,
// plane) segment and a chunk slot in it; a chunk straddling two segments is visited by both,
// each lane keeping only its own segment's nodes.
struct SlabWalk {
  int64_t n_work;
  int per_seg, nk, klo;
  __device__ __forceinline__ int chunk(int64_t w, const GridDims &g, int node_lo, int node_hi, int &lo,
                                       int &hi) const {
    if (g.slab == 0) {  // plain order: chunk c_lo + w over [node_lo, node_hi)
      lo = node_lo, hi = node_hi;
      return (node_lo >> 5) + (int)w;
    }
    const int seg = (int)(w / per_seg), slot = (int)(w - (int64_t)seg * per_seg);
    const int s = seg / nk, k = klo + (seg - s * nk);
    const int row0 = s * g.slab, row1 = min(row0 + g.slab, g.ny);
    lo = max(node_lo, k * g.nxy + row0 * g.nx);
    hi = min(node_hi, k * g.nxy + row1 * g.nx);
    const int c = (lo >> 5) + slot;
    if (lo >= hi || c > ((hi - 1) >> 5)) hi = lo;  // empty slot: no lane passes the range test
    return c;
  }
};
__device__ __forceinline__ SlabWalk slab_walk(const GridDims &g, int node_lo, int node_hi) {
  SlabWalk sw{};
  if (g.slab == 0) {
    sw.n_work = ((node_hi + 31) >> 5) - (node_lo >> 5);
    return sw;
  }
  sw.klo = node_lo / g.nxy;
  sw.nk = (node_hi - 1) / g.nxy + 1 - sw.klo;
  sw.per_seg = (g.slab * g.nx + 31) / 32 + 1;
  sw.n_work = (int64_t)((g.ny + g.slab - 1) / g.slab) * sw.nk * sw.per_seg;
  return sw;
}

// A lattice block's 9 values (value e at +32 e) in FP64, or in the FP32 copy written by
// b200fem_grid_to_f32.  `tile` = (offset, 32-node tile).
__device__ __forceinline__ void grid_block(const double *__restrict__ grid, int64_t tile, int lane, bool ok,
                                           double (&b)[9]) {
  const double *B = grid + tile * 288 + lane;
#pragma unroll
  for (int e = 0; e < 9; ++e) b[e] = ok ? __ldg(B + 32 * e) : 0.0;  // normal L2 policy (see below)
}
__device__ __forceinline__ void grid_block(const float *__restrict__ grid, int64_t tile, int lane, bool ok,
                                           float (&b)[9]) {
  // same layout in FP32, kept in FP32 registers until the FP64 FMA that uses it.  Tried: two
  // float4 + one float per lane (3 loads instead of 9): 690-717 us against 391 us for these
  // scalar loads at config 3 (one CTA per SM)
  const float *B = grid + tile * 288 + lane;
#pragma unroll
  for (int e = 0; e < 9; ++e) b[e] = ok ? __ldg(B + 32 * e) : 0.0f;
}

// VT = double: the stored tangent.  VT = float: its single-precision copy (opt-in
// operator "grid32", b200fem_matrix_set_f32): half the value bytes, products and sums in FP64.
template <int MODE, typename VT>
__global__ void __launch_bounds__(kGThreads, sizeof(VT) == 4 ? kGMinBlocks32 : kGMinBlocks) k_spmv_grid3(const VT *__restrict__ grid, GridDims g,
                                                             const uint8_t *__restrict__ dir_flag, int node_lo,
                                                             int node_hi, SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int warp0 = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  const int64_t np = g.npad;
  double red0 = 0.0, red1 = 0.0;
  const int nch = (int)(np >> 5);
  const SlabWalk sw = slab_walk(g, node_lo, node_hi);
  for (int64_t w = warp0; w < sw.n_work; w += nwarps) {
    int lo, hi;
    const int c = sw.chunk(w, g, node_lo, node_hi, lo, hi);
    const int c0 = c << 5, node = c0 + lane;
    if (node < lo || node >= hi) continue;
    const LatticePos p = lattice_pos(node, c0, g);
    const double *__restrict__ x = a.x;
    // the epilogue's row operands (D^-1, r0 / b / x_i, Dirichlet flags) are loaded first so
    // their latency hides behind the 27 block products instead of trailing them
    RowPre pre[3];
    bool dfl[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      pre[r] = spmv_preload<MODE>(3 * (int64_t)node + r, a);
      dfl[r] = dir_flag && __ldg(dir_flag + 3 * (int64_t)node + r);
    }
    double yu[3] = {0.0, 0.0, 0.0}, yl[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 14; ++q) {  // upper: B_q[a] x_{a + off_q}
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      const bool ok = grid_has(p, di, dj, dk);
      const int m = node + di + dj * g.nx + dk * g.nxy;
      VT b[9];
      double xm[3];
      grid_block(grid, (int64_t)q * nch + c, lane, ok, b);  // first use: normal L2 policy
#pragma unroll
      for (int t = 0; t < 3; ++t) xm[t] = ok ? __ldg(x + 3 * (int64_t)m + t) : 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
        yu[r] = fma((double)b[3 * r + 2], xm[2], fma((double)b[3 * r + 1], xm[1], fma((double)b[3 * r], xm[0], yu[r])));
    }
#pragma unroll
    // lower: B_q[a - off_q]^T x_{a - off_q}.  Normal L2 policy, not evict-first: the warp
    // streaming node a - off_q as an upper block runs concurrently in the same wave, so this
    // read may come first; an evict-first line would then be dropped before that second use
    // (ncu DRAM 2.81 -> 2.73 GB, 474 -> 463 us per matvec at config 3).
    for (int q = 1; q < 14; ++q) {
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      const bool ok = grid_has(p, -di, -dj, -dk);
      const int m = node - di - dj * g.nx - dk * g.nxy;
      VT b[9];
      double xm[3];
      grid_block(grid, (int64_t)q * nch + (m >> 5), m & 31, ok, b);  // normal policy (see below)
#pragma unroll
      for (int t = 0; t < 3; ++t) xm[t] = ok ? __ldg(x + 3 * (int64_t)m + t) : 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
        yl[r] = fma((double)b[6 + r], xm[2], fma((double)b[3 + r], xm[1], fma((double)b[r], xm[0], yl[r])));
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int64_t row = 3 * (int64_t)node + r;
      const double acc = dfl[r] ? __ldg(x + row) : yu[r] + yl[r];
      spmv_epilogue<MODE>(row, acc, a, pre[r], red0, red1);
    }
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2, kGThreads / 32>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage)
      spmv_stage<MODE>(a.sc, tot);
  }
}

template <int MODE, typename VT>
__global__ void __launch_bounds__(kGThreads, sizeof(VT) == 4 ? kGMinBlocks32 : kGMinBlocks) k_spmv_grid3_pf(const VT *__restrict__ grid, GridDims g,
                                                             const uint8_t *__restrict__ dir_flag, int node_lo,
                                                             int node_hi, SpmvArgs a, RedScratch red, int ef) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  // Row operands of the epilogue, software-pipelined one chunk ahead: while chunk i is computed,
  // each lane's cp.async copies of ITS OWN three rows of chunk i+1 are in flight into its private
  // shared-memory slots (no registers held, no cross-lane dependency, no __syncwarp); the
  // epilogue of chunk i waits only for the group issued during chunk i-1.
  constexpr int NE = n_ext<MODE>();
  __shared__ double s_pf[2][NE > 0 ? NE : 1][kGThreads * 3];
  const int lane = threadIdx.x & 31;
  const int warp0 = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  const int64_t np = g.npad;
  double red0 = 0.0, red1 = 0.0;
  const int nch = (int)(np >> 5);
  const SlabWalk sw = slab_walk(g, node_lo, node_hi);
  // read-once row operands evict-first, so they do not push out the blocks this matvec
  // re-reads from L2 (ef = 0: normal policy, the A/B switch B200FEM_GRID_PF_NORMAL=1)
  const uint64_t pol = l2_evict_first_policy();
  auto prefetch = [&](int64_t wn, int buf) {  // this lane's rows of work item wn
    if (wn < sw.n_work) {
      int lo2, hi2;
      const int c2 = sw.chunk(wn, g, node_lo, node_hi, lo2, hi2);
      const int node2 = (c2 << 5) + lane;
      if (node2 >= lo2 && node2 < hi2) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const double *src = ext_ptr<MODE>(a, e) + 3 * (int64_t)node2;
          const bool hint = ef && pf_read_once<MODE>(e);
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            if (hint)
              cp_async8_hint(&s_pf[buf][e][3 * threadIdx.x + r], src + r, pol);
            else
              cp_async8(&s_pf[buf][e][3 * threadIdx.x + r], src + r);
          }
        }
      }
    }
    cp_async_commit();  // one group per work item (possibly empty)
  };
  if (NE > 0) prefetch(warp0, 0);
  int buf = 0;
  for (int64_t w = warp0; w < sw.n_work; w += nwarps, buf ^= 1) {
    if (NE > 0) prefetch(w + nwarps, buf ^ 1);
    int lo, hi;
    const int c = sw.chunk(w, g, node_lo, node_hi, lo, hi);
    const int c0 = c << 5, node = c0 + lane;
    if (node < lo || node >= hi) continue;
    const LatticePos p = lattice_pos(node, c0, g);
    const double *__restrict__ x = a.x;
    // the epilogue's row operands (D^-1, r0 / b / x_i, Dirichlet flags) are loaded first so
    // their latency hides behind the 27 block products instead of trailing them
    bool dfl[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) dfl[r] = dir_flag && __ldg(dir_flag + 3 * (int64_t)node + r);
    double yu[3] = {0.0, 0.0, 0.0}, yl[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 14; ++q) {  // upper: B_q[a] x_{a + off_q}
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      const bool ok = grid_has(p, di, dj, dk);
      const int m = node + di + dj * g.nx + dk * g.nxy;
      VT b[9];
      double xm[3];
      grid_block(grid, (int64_t)q * nch + c, lane, ok, b);  // first use: normal L2 policy
#pragma unroll
      for (int t = 0; t < 3; ++t) xm[t] = ok ? __ldg(x + 3 * (int64_t)m + t) : 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
        yu[r] = fma((double)b[3 * r + 2], xm[2], fma((double)b[3 * r + 1], xm[1], fma((double)b[3 * r], xm[0], yu[r])));
    }
#pragma unroll
    // lower: B_q[a - off_q]^T x_{a - off_q}.  Normal L2 policy, not evict-first: the warp
    // streaming node a - off_q as an upper block runs concurrently in the same wave, so this
    // read may come first; an evict-first line would then be dropped before that second use
    // (ncu DRAM 2.81 -> 2.73 GB, 474 -> 463 us per matvec at config 3).
    for (int q = 1; q < 14; ++q) {
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      const bool ok = grid_has(p, -di, -dj, -dk);
      const int m = node - di - dj * g.nx - dk * g.nxy;
      VT b[9];
      double xm[3];
      grid_block(grid, (int64_t)q * nch + (m >> 5), m & 31, ok, b);  // normal policy (see below)
#pragma unroll
      for (int t = 0; t < 3; ++t) xm[t] = ok ? __ldg(x + 3 * (int64_t)m + t) : 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
        yl[r] = fma((double)b[6 + r], xm[2], fma((double)b[3 + r], xm[1], fma((double)b[r], xm[0], yl[r])));
    }
    if (NE > 0) cp_async_wait_1();  // this item's rows (issued one item ago) have landed
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int64_t row = 3 * (int64_t)node + r;
      const double acc = dfl[r] ? __ldg(x + row) : yu[r] + yl[r];
      const int t = 3 * threadIdx.x + r;
      const RowPre pre = row_pre_from<MODE>(&s_pf[buf][0][t], &s_pf[buf][NE > 1 ? 1 : 0][t],
                                            &s_pf[buf][NE > 2 ? 2 : 0][t]);
      spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
    }
  }
  if (NE > 0) cp_async_wait_all();  // no copy may outlive the block
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2, kGThreads / 32>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage)
      spmv_stage<MODE>(a.sc, tot);
  }
}

// Scalar (vec 1, Poisson) GRID: one value per offset; a thread per node, 4 CTAs per SM.
template <int MODE>
__global__ void __launch_bounds__(kGThreads, 4) k_spmv_grid1(const double *__restrict__ grid, GridDims g,
                                                             const uint8_t *__restrict__ dir_flag, int node_lo,
                                                             int node_hi, SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int warp0 = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  const int c_lo = node_lo >> 5, n_chunks = (node_hi + 31) >> 5;
  const int nch = (int)(g.npad >> 5);
  double red0 = 0.0, red1 = 0.0;
  for (int c = c_lo + warp0; c < n_chunks; c += nwarps) {
    const int c0 = c << 5, node = c0 + lane;
    if (node < node_lo || node >= node_hi) continue;
    const LatticePos p = lattice_pos(node, c0, g);
    const double *__restrict__ x = a.x;
    double yu = 0.0, yl = 0.0;
#pragma unroll
    for (int q = 0; q < 14; ++q) {
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      const bool ok = grid_has(p, di, dj, dk);
      const int m = node + di + dj * g.nx + dk * g.nxy;
      const double b = ok ? __ldg(grid + ((int64_t)(q * nch + c) * 32 + lane)) : 0.0;
      const double xm = ok ? __ldg(x + m) : 0.0;
      yu = fma(b, xm, yu);
    }
#pragma unroll
    for (int q = 1; q < 14; ++q) {
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      const bool ok = grid_has(p, -di, -dj, -dk);
      const int m = node - di - dj * g.nx - dk * g.nxy;
      const double b = ok ? __ldg(grid + ((int64_t)(q * nch + (m >> 5)) * 32 + (m & 31))) : 0.0;
      const double xm = ok ? __ldg(x + m) : 0.0;
      yl = fma(b, xm, yl);
    }
    const int64_t row = node;
    const RowPre pre = spmv_preload<MODE>(row, a);
    const double acc = (dir_flag && __ldg(dir_flag + row)) ? __ldg(x + row) : yu + yl;
    spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2, kGThreads / 32>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage)
      spmv_stage<MODE>(a.sc, tot);
  }
}

static GridDims grid_dims(const Matrix *m) {
  GridDims g{};
  g.nx = m->gnx, g.ny = m->gny, g.nz = m->gnz, g.nxy = m->gnx * m->gny, g.nn = (int)(m->n / m->gvec), g.npad = m->gnpad;
  g.slab = 0;
  if (m->gvec == 3) {  // slabs of ~4096 nodes per plane, once a plane of blocks outgrows L2 reuse
    const char *e = getenv("B200FEM_GRID_SLAB");  // per launch: tests switch it in-process
    const int env = e ? atoi(e) : -1;
    // plain order while one plane of blocks (nxy * 1008 B) stays under ~24 MB: its lower-block
    // re-reads still hit L2 there (ncu: +3 % DRAM at 136^3, a plane of 19 MB), and the order
    // of the fused Krylov dots -- hence the rounding of every iterate -- stays the plain one
    const int rows = env >= 0 ? env : (4096 + g.nx - 1) / g.nx;
    const bool big_plane = (int64_t)g.nxy * 1008 > (int64_t)24 << 20;
    if (rows > 0 && (env >= 0 || (big_plane && g.ny >= 4 * rows))) g.slab = std::min(rows, g.ny);
  }
  return g;
}

int prepare_grid3(Matrix *m) {
  m->n_chunks = (int)((m->n / m->gvec + 31) / 32);
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

template <int MODE, int LANES>
__global__ void __launch_bounds__(kThreads) k_spmv_csr(const int32_t *__restrict__ indptr,
                                                       const int32_t *__restrict__ indices,
                                                       const double *__restrict__ data, int64_t row_lo, int64_t n,
                                                       SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LANES, sl = lane % LANES;
  constexpr int kPerWarp = 32 / LANES;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double red0 = 0.0, red1 = 0.0;
  for (int64_t base = row_lo + warp0 * kPerWarp; base < n; base += nwarps * kPerWarp) {
    const int64_t row = base + sub;
    double acc = 0.0;
    RowPre pre{0.0, 0.0, 0.0, 0.0};
    if (row < n && sl == 0) pre = spmv_preload<MODE>(row, a);
    if (row < n) {
      const int k1 = __ldg(indptr + row + 1);
      int k = __ldg(indptr + row) + sl;
      for (; k + 3 * LANES < k1; k += 4 * LANES) {  // 4 independent loads in flight per lane
        const double d0 = __ldcs(data + k), d1 = __ldcs(data + k + LANES), d2 = __ldcs(data + k + 2 * LANES),
                     d3 = __ldcs(data + k + 3 * LANES);
        const int i0 = __ldcs(indices + k), i1 = __ldcs(indices + k + LANES), i2 = __ldcs(indices + k + 2 * LANES),
                  i3 = __ldcs(indices + k + 3 * LANES);
        acc = fma(d0, __ldg(a.x + i0), acc);
        acc = fma(d1, __ldg(a.x + i1), acc);
        acc = fma(d2, __ldg(a.x + i2), acc);
        acc = fma(d3, __ldg(a.x + i3), acc);
      }
      for (; k < k1; k += LANES) acc = fma(__ldcs(data + k), __ldg(a.x + __ldcs(indices + k)), acc);
    }
#pragma unroll
    for (int o = LANES / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < n && sl == 0) spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
  }
  if (MODE != SP_PLAIN) {
    double v[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2>(v, red, tot) && threadIdx.x == 0 && a.inline_stage) spmv_stage<MODE>(a.sc, tot);
  }
}

// Jacobi / residual modes of the FP64 GRID3 matvec use the row-operand prefetch kernel
// (504 / 492 us against 511 / 516 us with register preloads, config 3, profiles/r02_grid_prefetch_ab.jsonl);
// B200FEM_GRID_NO_PREFETCH=1 restores the preload kernel (A/B).
static bool grid_prefetch() {
  static int v = -1;
  if (v < 0) v = getenv("B200FEM_GRID_NO_PREFETCH") ? 0 : 1;
  return v == 1;
}

static int grid_pf_evict_first() {
  static int v = -1;
  if (v < 0) v = getenv("B200FEM_GRID_PF_NORMAL") ? 0 : 1;
  return v;
}

template <int MODE>
static void spmv_dispatch(const Matrix *m, const SpmvArgs &a, RedScratch *red) {
  const int grid = MODE == SP_PLAIN ? (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (m->n + 63) / 64)) : kRedBlocks;
  RedScratch r = red ? *red : RedScratch{};
  const bool full = m->row_hi < 0;
  if (m->kind == MK_GRID3) {  // all nodes, or the owned node range of a partition
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const GridDims g = grid_dims(m);
    const int lo = full ? 0 : (int)m->row_lo, hi = full ? g.nn : (int)m->row_hi;  // node range
    const int nch = ((hi + 31) >> 5) - (lo >> 5);
    if (m->gvec == 1) {
      const int gg = (int)std::max<int64_t>(1, std::min<int64_t>(4 * sms, (nch + 7) / 8));
      k_spmv_grid1<MODE><<<gg, kGThreads, 0, m->stream>>>(m->data, g, m->dir_flag, lo, hi, a, r);
    } else {
      const int gg = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (nch + 7) / 8));
      if (m->data32)
        k_spmv_grid3<MODE, float><<<(int)std::min<int64_t>((int64_t)kGMinBlocks32 * gg, std::max(1, (nch + 7) / 8)),
                                    kGThreads, 0, m->stream>>>(m->data32, g, m->dir_flag, lo, hi, a, r);
      else if (MODE != SP_PLAIN && grid_prefetch())
        k_spmv_grid3_pf<MODE, double><<<gg, kGThreads, 0, m->stream>>>(m->data, g, m->dir_flag, lo, hi, a, r,
                                                                        grid_pf_evict_first());
      else
        k_spmv_grid3<MODE, double><<<gg, kGThreads, 0, m->stream>>>(m->data, g, m->dir_flag, lo, hi, a, r);
    }
  } else if (m->kind == MK_FEM3 && m->use_tma && m->n_chunks > 0) {  // chunks cover the row range
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int g = std::min(sms, m->n_chunks);
    if (m->npw == 2) {
      k_spmv_fem3_tma2<MODE><<<g, kT2Threads, kT2Smem, m->stream>>>(m->nbr_ptr, m->nbr, m->data, m->chunk_node,
                                                                    m->n_chunks, m->nnz / 9, m->n, a, r);
      count_launch();
      return;
    }
    launch_fem3_tma_npw1(m, MODE, a, r, g);  // spmv_alt.cu
  } else if (m->kind == MK_SYM3 && m->use_tma && full) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    launch_sym3_tma(m, MODE, a, r, std::min(sms, m->n_chunks));  // spmv_alt.cu
  } else if (m->kind == MK_SYM3) {
    const int64_t lo = full ? 0 : m->row_lo, hi = full ? m->n / 3 : m->row_hi;
    k_spmv_sym3<MODE><<<grid, kThreads, 0, m->stream>>>(m->nbr_ptr, m->nbr, m->up_ptr, m->lo_blk, m->data,
                                                       m->dir_flag, lo, hi, a, r);
  } else if (m->kind == MK_FEM3) {
    const int64_t lo = full ? 0 : m->row_lo, hi = full ? m->n / 3 : m->row_hi;
    k_spmv_fem3<MODE><<<grid, kThreads, 0, m->stream>>>(m->nbr_ptr, m->nbr, m->data, lo, hi, a, r);
  } else {
    const int64_t lo = full ? 0 : m->row_lo, hi = full ? m->n : m->row_hi;
    switch (m->lanes) {
      case 4: k_spmv_csr<MODE, 4><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, lo, hi, a, r); break;
      case 8: k_spmv_csr<MODE, 8><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, lo, hi, a, r); break;
      case 16: k_spmv_csr<MODE, 16><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, lo, hi, a, r); break;
      default: k_spmv_csr<MODE, 32><<<grid, kThreads, 0, m->stream>>>(m->indptr, m->indices, m->data, lo, hi, a, r); break;
    }
  }
  count_launch();
}

int launch_spmv(const Matrix *m, SpmvMode mode, const SpmvArgs &a, RedScratch *red) {
  switch (mode) {
    case SP_PLAIN: spmv_dispatch<SP_PLAIN>(m, a, red); break;
    case SP_JACOBI_R0: spmv_dispatch<SP_JACOBI_R0>(m, a, red); break;
    case SP_JACOBI_TT: spmv_dispatch<SP_JACOBI_TT>(m, a, red); break;
    case SP_PQ: spmv_dispatch<SP_PQ>(m, a, red); break;
    case SP_CGRES: spmv_dispatch<SP_CGRES>(m, a, red); break;
    default: spmv_dispatch<SP_RESIDUAL>(m, a, red); break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

// diagonal (sparse.py:44-51: 0 where the row has no diagonal entry), its inverse and the
// number of zero entries (solvers.py:101-103)
__global__ void __launch_bounds__(kThreads) k_diagonal(const int32_t *__restrict__ indptr,
                                                       const int32_t *__restrict__ indices,
                                                       const int32_t *__restrict__ slots,
                                                       const int32_t *__restrict__ up_ptr,
                                                       const uint8_t *__restrict__ dflag,
                                                       const double *__restrict__ data, int64_t row_lo, int64_t n,
                                                       double *diag, double *inv, RedScratch red, int64_t grid_npad,
                                                       int gvec) {
  double zeros[1] = {0.0};
  for (int64_t i = row_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    if (grid_npad) {  // GRID3: entry (c,c) of the node's self block (k = 0, element 4c)
      d = (dflag && dflag[i]) ? 1.0
          : gvec == 3 ? data[grid_idx(0, 4 * (i % 3), i / 3, grid_npad)] : data[grid_idx(0, 0, i, grid_npad, 1)];
    } else if (up_ptr) {  // SYM3: entry (c,c) of the node's self block (first upper block)
      d = (dflag && dflag[i]) ? 1.0 : data[9 * (int64_t)up_ptr[i / 3] + 4 * (i % 3)];
    } else if (slots) {
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
  const int rpn = m->kind == MK_CSR ? 1 : m->kind == MK_GRID3 ? m->gvec : 3;  // rows per range unit
  const int64_t lo = m->row_hi < 0 ? 0 : rpn * m->row_lo;
  const int64_t hi = m->row_hi < 0 ? m->n : rpn * m->row_hi;
  const bool sym = m->kind == MK_SYM3 || m->kind == MK_GRID3;
  k_diagonal<<<kRedBlocks, kThreads, 0, m->stream>>>(m->indptr, m->indices, sym ? nullptr : m->diag_slots,
                                                     m->kind == MK_SYM3 ? m->up_ptr : nullptr,
                                                     sym ? m->dir_flag : nullptr, m->data, lo, hi, diag, inv, *red,
                                                     m->kind == MK_GRID3 ? m->gnpad : 0, m->gvec);
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
