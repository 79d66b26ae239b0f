// SpMV variants that were measured and lost, kept as opt-in A/B switches
// so the numbers in profiles/ stay reproducible:
//  * k_spmv_fem3_tma: the warp-per-node bulk-copy CSR kernel (B200FEM_SPMV_NPW=1; bit-identical
//    to the default two-nodes-per-warp kernel k_spmv_fem3_tma2 and to the LDG kernel), with the
//    x-gather variants of B200FEM_SPMV_X (vec: 16-byte pair loads; none: diagnostic, wrong y);
//  * k_spmv_sym3_tma: the bulk-copy SYM3 operator (B200FEM_SYM_TMA=1; 1.64 ms vs 0.85 ms).

#include <algorithm>
#include <cstring>
#include <vector>

#include "spmv_common.cuh"

namespace b200 {

template <int MODE, int XV>
__global__ void __launch_bounds__(kTmaThreads, 1) k_spmv_fem3_tma(const int32_t *__restrict__ nbr_ptr,
                                                                 const int32_t *__restrict__ nbr,
                                                                 const double *__restrict__ data,
                                                                 const int32_t *__restrict__ chunk_node, int n_chunks,
                                                                 int64_t total_blocks, int64_t n_rows, SpmvArgs a,
                                                                 RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kTmaStages * kTmaStageBytes);
  uint64_t *empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kTmaConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // the last chunk's end may not be 16-byte aligned: it is read from global memory instead
  const uint64_t val_end = (uint64_t)total_blocks * 72, nbr_end = (uint64_t)total_blocks * 4;
  const uint64_t row_end = (uint64_t)n_rows * 8;
  double red0 = 0.0, red1 = 0.0;
  if (warp == kTmaConsumers) {
    if (lane == 0) {  // producer
      int it = 0;
      for (int c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
        const int s = it % kTmaStages;
        const uint32_t ph = (it / kTmaStages) & 1;
        mbar_wait(empty + s, ph ^ 1);
        const int64_t p0 = __ldg(nbr_ptr + __ldg(chunk_node + c)), p1 = __ldg(nbr_ptr + __ldg(chunk_node + c + 1));
        const uint64_t vb0 = (72ull * p0) & ~15ull, vb1 = std::min((72ull * p1 + 15) & ~15ull, val_end & ~15ull);
        const uint64_t nb0 = (4ull * p0) & ~15ull, nb1 = std::min((4ull * p1 + 15) & ~15ull, nbr_end & ~15ull);
        const int64_t cn0 = __ldg(chunk_node + c), cn1 = __ldg(chunk_node + c + 1);
        const uint64_t eb0 = (24ull * cn0) & ~15ull, eb1 = std::min((24ull * cn1 + 15) & ~15ull, row_end & ~15ull);
        const uint32_t ext_bytes = eb1 > eb0 ? (uint32_t)(eb1 - eb0) : 0u;
        mbar_expect_tx(full + s, (uint32_t)((vb1 - vb0) + (nb1 - nb0)) + n_ext<MODE>() * ext_bytes);
        uint8_t *stage = smem + s * kTmaStageBytes;
        if (vb1 > vb0) bulk_g2s(stage, reinterpret_cast<const uint8_t *>(data) + vb0, (uint32_t)(vb1 - vb0), full + s);
        if (nb1 > nb0)
          bulk_g2s(stage + kTmaValBytes, reinterpret_cast<const uint8_t *>(nbr) + nb0, (uint32_t)(nb1 - nb0), full + s);
#pragma unroll
        for (int k = 0; k < n_ext<MODE>(); ++k)
          if (ext_bytes)
            bulk_g2s(stage + kTmaValBytes + kTmaNbrBytes + k * kTmaExtBytes,
                     reinterpret_cast<const uint8_t *>(ext_ptr<MODE>(a, k)) + eb0, ext_bytes, full + s);
      }
    }
    __syncwarp();  // reconverge the producer warp before the block-wide reduction barrier
  } else {
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
      const uint8_t *stage = smem + s * kTmaStageBytes;
      const int nA = n0 + warp;
      const bool has = nA < n1;
      int64_t pA = 0;
      int cA = 0;
      if (has) {
        pA = __ldg(nbr_ptr + nA);
        cA = __ldg(nbr_ptr + nA + 1) - (int)pA;
      }
      const bool row_lane = (lane & 7) == 0 && lane < 24;
      const int64_t row = 3 * (int64_t)nA + (lane >> 3);
      RowPre pre{0.0, 0.0, 0.0, 0.0};
      if (tail && row_lane && has) pre = spmv_preload<MODE>(row, a);
      mbar_wait(full + s, ph);
      if (!tail && row_lane && has && n_ext<MODE>() > 0) {
        const uint8_t *ext = stage + kTmaValBytes + kTmaNbrBytes + (8ull * row - eb0);
        pre = row_pre_from<MODE>(reinterpret_cast<const double *>(ext),
                                 reinterpret_cast<const double *>(ext + kTmaExtBytes),
                                 reinterpret_cast<const double *>(ext + 2 * kTmaExtBytes));
      }
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      if (has) {
        if (!tail)
          node_rows<XV>(reinterpret_cast<const double *>(stage + (72ull * pA - vb0)),
                    reinterpret_cast<const int32_t *>(stage + kTmaValBytes + (4ull * pA - nb0)), cA, a.x, lane, y0, y1,
                    y2);
        else
          node_rows<XV>(data + 9 * pA, nbr + pA, cA, a.x, lane, y0, y1, y2);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);  // stage reads done; the producer may refill it
      if (has) {
        const double acc = warp_sum3(y0, y1, y2, lane);
        if (row_lane) spmv_epilogue<MODE>(3 * (int64_t)nA + (lane >> 3), acc, a, pre, red0, red1);
      }
    }
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2, kTmaConsumers + 1>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage)
      spmv_stage<MODE>(a.sc, tot);
  }
}

template <int XV>
static void set_tma_attr() {
  cudaFuncSetAttribute(k_spmv_fem3_tma<SP_PLAIN, XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
  cudaFuncSetAttribute(k_spmv_fem3_tma<SP_JACOBI_R0, XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
  cudaFuncSetAttribute(k_spmv_fem3_tma<SP_JACOBI_TT, XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
  cudaFuncSetAttribute(k_spmv_fem3_tma<SP_RESIDUAL, XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
  cudaFuncSetAttribute(k_spmv_fem3_tma<SP_PQ, XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
  cudaFuncSetAttribute(k_spmv_fem3_tma<SP_CGRES, XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
}

// x-gather variant of the bulk-copy kernel (B200FEM_SPMV_X = "vec" | "none"; "none" is a
// diagnostic that skips the gather and computes wrong results).
static int tma_x_variant() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("B200FEM_SPMV_X");
    v = (e && !strcmp(e, "vec")) ? 1 : (e && !strcmp(e, "none")) ? 2 : 0;
  }
  return v;
}

// ------------------------------------------------------------------------------------
// SYM3 with the bulk-copy pipeline: the chunk's upper blocks, neighbour ids, lower-block
// indices and row operands are contiguous for consecutive nodes and stream into shared
// memory; the consumer warps gather only x and the lower blocks (L2-resident: they were
// streamed as upper blocks of nearby rows moments before).  One memory round trip per node.
constexpr int kSymUpBytes = 40 * 1024;
constexpr int kSymNbrBytes = 4096;
constexpr int kSymStageBytes = kSymUpBytes + 2 * kSymNbrBytes + 3 * kTmaExtBytes;
constexpr int kSymStages = 4;
constexpr int kSymSmem = kSymStages * kSymStageBytes + 2 * kSymStages * 8;

template <int MODE>
__global__ void __launch_bounds__(kTmaThreads, 1) k_spmv_sym3_tma(
    const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr, const int32_t *__restrict__ up_ptr,
    const int32_t *__restrict__ lo_blk, const double *__restrict__ sym, const uint8_t *__restrict__ dir_flag,
    const int32_t *__restrict__ chunk_node, int n_chunks, int64_t n_nodes, SpmvArgs a, RedScratch red) {
  if (a.sc && a.sc->status != KS_RUNNING) return;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kSymStages * kSymStageBytes);
  uint64_t *empty = full + kSymStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSymStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kTmaConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t up_end = (uint64_t)__ldg(up_ptr + n_nodes) * 72, nb_end = (uint64_t)__ldg(nbr_ptr + n_nodes) * 4;
  const uint64_t row_end = (uint64_t)n_nodes * 24;
  double red0 = 0.0, red1 = 0.0;
  if (warp == kTmaConsumers) {
    if (lane == 0) {  // producer
      int it = 0;
      for (int c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
        const int s = it % kSymStages;
        const uint32_t ph = (it / kSymStages) & 1;
        mbar_wait(empty + s, ph ^ 1);
        const int64_t n0 = __ldg(chunk_node + c), n1 = __ldg(chunk_node + c + 1);
        const uint64_t u0 = (72ull * __ldg(up_ptr + n0)) & ~15ull,
                       u1 = std::min((72ull * __ldg(up_ptr + n1) + 15) & ~15ull, up_end & ~15ull);
        const uint64_t b0 = (4ull * __ldg(nbr_ptr + n0)) & ~15ull,
                       b1 = std::min((4ull * __ldg(nbr_ptr + n1) + 15) & ~15ull, nb_end & ~15ull);
        const uint64_t e0 = (24ull * n0) & ~15ull, e1 = std::min((24ull * n1 + 15) & ~15ull, row_end & ~15ull);
        const uint32_t ub = u1 > u0 ? (uint32_t)(u1 - u0) : 0u, nb = b1 > b0 ? (uint32_t)(b1 - b0) : 0u,
                       eb = e1 > e0 ? (uint32_t)(e1 - e0) : 0u;
        mbar_expect_tx(full + s, ub + 2 * nb + n_ext<MODE>() * eb);
        uint8_t *stage = smem + s * kSymStageBytes;
        if (ub) bulk_g2s(stage, reinterpret_cast<const uint8_t *>(sym) + u0, ub, full + s);
        if (nb) {
          bulk_g2s(stage + kSymUpBytes, reinterpret_cast<const uint8_t *>(nbr) + b0, nb, full + s);
          bulk_g2s(stage + kSymUpBytes + kSymNbrBytes, reinterpret_cast<const uint8_t *>(lo_blk) + b0, nb, full + s);
        }
#pragma unroll
        for (int k = 0; k < n_ext<MODE>(); ++k)
          if (eb)
            bulk_g2s(stage + kSymUpBytes + 2 * kSymNbrBytes + k * kTmaExtBytes,
                     reinterpret_cast<const uint8_t *>(ext_ptr<MODE>(a, k)) + e0, eb, full + s);
      }
    }
    __syncwarp();
  } else {
    int it = 0;
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
      const int s = it % kSymStages;
      const uint32_t ph = (it / kSymStages) & 1;
      const int n0 = __ldg(chunk_node + c), n1 = __ldg(chunk_node + c + 1);
      const int64_t u0 = (72ll * __ldg(up_ptr + n0)) & ~15ll, b0 = (4ll * __ldg(nbr_ptr + n0)) & ~15ll;
      const uint64_t e0 = (24ull * n0) & ~15ull;
      const bool tail = (72ull * __ldg(up_ptr + n1) > (up_end & ~15ull)) ||
                        (4ull * __ldg(nbr_ptr + n1) > (nb_end & ~15ull)) ||
                        (n_ext<MODE>() > 0 && 24ull * n1 > (row_end & ~15ull));
      const uint8_t *stage = smem + s * kSymStageBytes;
      const int n = n0 + warp;
      const bool has = n < n1;
      int p0 = 0, cnt = 0, ubn = 0, self = 0;
      if (has) {
        p0 = __ldg(nbr_ptr + n);
        cnt = __ldg(nbr_ptr + n + 1) - p0;
        ubn = __ldg(up_ptr + n);
        self = cnt - (__ldg(up_ptr + n + 1) - ubn);
      }
      const bool row_lane = (lane & 7) == 0 && lane < 24;
      const int64_t row = 3 * (int64_t)n + (lane >> 3);
      RowPre pre{0.0, 0.0, 0.0, 0.0};
      bool dflag = false;
      double xrow = 0.0;
      if (row_lane && has) {
        if (tail) pre = spmv_preload<MODE>(row, a);
        dflag = dir_flag && __ldg(dir_flag + row);
        if (dflag) xrow = __ldg(a.x + row);
      }
      mbar_wait(full + s, ph);
      if (!tail && row_lane && has && n_ext<MODE>() > 0) {
        const uint8_t *ext = stage + kSymUpBytes + 2 * kSymNbrBytes + (8ull * row - e0);
        pre = row_pre_from<MODE>(reinterpret_cast<const double *>(ext),
                                 reinterpret_cast<const double *>(ext + kTmaExtBytes),
                                 reinterpret_cast<const double *>(ext + 2 * kTmaExtBytes));
      }
      double y0 = 0.0, y1 = 0.0, y2 = 0.0;
      if (has) {
        const int32_t *sn = tail ? nbr + p0 : reinterpret_cast<const int32_t *>(stage + kSymUpBytes + (4ll * p0 - b0));
        const int32_t *sl =
            tail ? lo_blk + p0 : reinterpret_cast<const int32_t *>(stage + kSymUpBytes + kSymNbrBytes + (4ll * p0 - b0));
        const double *su = tail ? sym + 9 * (int64_t)ubn : reinterpret_cast<const double *>(stage + (72ll * ubn - u0));
        for (int j = lane; j < cnt; j += 32) {
          const int m = sn[j];
          const bool lower = j < self;
          const double *B = lower ? sym + 9 * (int64_t)sl[j] : su + 9 * (j - self);
          double bb[9];
#pragma unroll
          for (int t = 0; t < 9; ++t) bb[t] = lower ? __ldg(B + t) : B[t];
          const double *__restrict__ xm = a.x + 3 * (int64_t)m;
          const double x0 = __ldg(xm), x1 = __ldg(xm + 1), x2 = __ldg(xm + 2);
          const double a01 = lower ? bb[3] : bb[1], a02 = lower ? bb[6] : bb[2], a10 = lower ? bb[1] : bb[3];
          const double a12 = lower ? bb[7] : bb[5], a20 = lower ? bb[2] : bb[6], a21 = lower ? bb[5] : bb[7];
          y0 = fma(a02, x2, fma(a01, x1, fma(bb[0], x0, y0)));
          y1 = fma(a12, x2, fma(bb[4], x1, fma(a10, x0, y1)));
          y2 = fma(bb[8], x2, fma(a21, x1, fma(a20, x0, y2)));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if (has) {
        double acc = warp_sum3(y0, y1, y2, lane);
        if (row_lane) {
          if (dflag) acc = xrow;
          spmv_epilogue<MODE>(row, acc, a, pre, red0, red1);
        }
      }
    }
  }
  if (MODE != SP_PLAIN) {
    double v2[2] = {red0, red1}, tot[2];
    if (block_partials_and_finish<2, kTmaConsumers + 1>(v2, red, tot) && threadIdx.x == 0 && a.inline_stage)
      spmv_stage<MODE>(a.sc, tot);
  }
}

int prepare_sym3_chunks(Matrix *m) {
  const int64_t nn = m->n / 3;
  std::vector<int32_t> ptr(nn + 1), up(nn + 1);
  if (cudaMemcpy(ptr.data(), m->nbr_ptr, (nn + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(up.data(), m->up_ptr, (nn + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return B200FEM_E_CUDA;
  std::vector<int32_t> ch{0};
  int64_t start = 0;
  for (int64_t n = 0; n < nn; ++n) {
    const int64_t nu = up[n + 1] - up[start], nb = ptr[n + 1] - ptr[start];
    const bool fits = 72 * nu + 32 <= kSymUpBytes && 4 * nb + 32 <= kSymNbrBytes && (n + 1 - start) <= kTmaConsumers;
    if (!fits) {
      if (n == start) return 0;
      ch.push_back((int32_t)n);
      start = n;
    }
  }
  ch.push_back((int32_t)nn);
  m->n_chunks = (int)ch.size() - 1;
  if (dalloc(&m->chunk_node, ch.size()) != cudaSuccess) return B200FEM_E_CUDA;
  if (cudaMemcpy(m->chunk_node, ch.data(), ch.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess)
    return B200FEM_E_CUDA;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmv_sym3_tma<SP_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
    cudaFuncSetAttribute(k_spmv_sym3_tma<SP_JACOBI_R0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
    cudaFuncSetAttribute(k_spmv_sym3_tma<SP_JACOBI_TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
    cudaFuncSetAttribute(k_spmv_sym3_tma<SP_RESIDUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
    cudaFuncSetAttribute(k_spmv_sym3_tma<SP_PQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
    cudaFuncSetAttribute(k_spmv_sym3_tma<SP_CGRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
    attr = true;
  }
  m->use_tma = true;
  return 0;
}



void set_fem3_tma_npw1_attr() {
  set_tma_attr<0>();
  set_tma_attr<1>();
  set_tma_attr<2>();
}

template <int MODE>
static void fem3_npw1(const Matrix *m, const SpmvArgs &a, const RedScratch &r, int g) {
  switch (tma_x_variant()) {
    case 1: k_spmv_fem3_tma<MODE, 1><<<g, kTmaThreads, kTmaSmem, m->stream>>>(m->nbr_ptr, m->nbr, m->data, m->chunk_node,
                                                                              m->n_chunks, m->nnz / 9, m->n, a, r); break;
    case 2: k_spmv_fem3_tma<MODE, 2><<<g, kTmaThreads, kTmaSmem, m->stream>>>(m->nbr_ptr, m->nbr, m->data, m->chunk_node,
                                                                              m->n_chunks, m->nnz / 9, m->n, a, r); break;
    default: k_spmv_fem3_tma<MODE, 0><<<g, kTmaThreads, kTmaSmem, m->stream>>>(m->nbr_ptr, m->nbr, m->data, m->chunk_node,
                                                                               m->n_chunks, m->nnz / 9, m->n, a, r);
  }
}

template <int MODE>
static void sym3_tma(const Matrix *m, const SpmvArgs &a, const RedScratch &r, int g) {
  k_spmv_sym3_tma<MODE><<<g, kTmaThreads, kSymSmem, m->stream>>>(m->nbr_ptr, m->nbr, m->up_ptr, m->lo_blk, m->data,
                                                                m->dir_flag, m->chunk_node, m->n_chunks, m->n / 3, a, r);
}

#define B200_MODE_SWITCH(F)                                          \
  switch (mode) {                                                    \
    case SP_PLAIN: F<SP_PLAIN>(m, a, r, grid); break;                \
    case SP_JACOBI_R0: F<SP_JACOBI_R0>(m, a, r, grid); break;        \
    case SP_JACOBI_TT: F<SP_JACOBI_TT>(m, a, r, grid); break;        \
    case SP_PQ: F<SP_PQ>(m, a, r, grid); break;                      \
    case SP_CGRES: F<SP_CGRES>(m, a, r, grid); break;                \
    default: F<SP_RESIDUAL>(m, a, r, grid); break;                   \
  }

void launch_fem3_tma_npw1(const Matrix *m, int mode, const SpmvArgs &a, const RedScratch &r, int grid) {
  B200_MODE_SWITCH(fem3_npw1)
}

void launch_sym3_tma(const Matrix *m, int mode, const SpmvArgs &a, const RedScratch &r, int grid) {
  B200_MODE_SWITCH(sym3_tma)
}

}  // namespace b200
