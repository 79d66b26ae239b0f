// Device helpers shared by the SpMV translation units (spmv.cu: the kernels the solvers use;
// spmv_alt.cu: the measured-and-rejected bulk-copy variants kept as opt-in A/B switches).
#pragma once

#include "internal.cuh"

namespace b200 {

// Row operands the epilogue needs, loaded at the START of a row's work so their latency
// overlaps the value stream instead of serialising after the reduction.
struct RowPre {
  double inv, aux, dg, xi;
};

template <int MODE>
__device__ __forceinline__ RowPre spmv_preload(int64_t i, const SpmvArgs &a) {
  // row operands are read once per matvec: evict-first (__ldcs) so they do not push the
  // matrix blocks a GRID3 matvec re-reads from L2 (its lower blocks) out of the cache
  RowPre p{0.0, 0.0, 0.0, 0.0};
  if (MODE == SP_JACOBI_R0) {
    p.inv = __ldcs(a.inv + i);
    p.aux = __ldcs(a.aux + i);
  } else if (MODE == SP_JACOBI_TT) {
    p.inv = __ldcs(a.inv + i);
    p.xi = __ldg(a.x + i);
  } else if (MODE == SP_RESIDUAL) {
    p.inv = __ldcs(a.inv + i);
    p.aux = __ldcs(a.aux + i);
    p.dg = __ldcs(a.dg + i);
  } else if (MODE == SP_PQ) {
    p.xi = __ldg(a.x + i);
  } else if (MODE == SP_CGRES) {
    p.inv = __ldcs(a.inv + i);
    p.aux = __ldcs(a.aux + i);
  }
  return p;
}

// Post-process row i's dot-product value `acc` for the mode; accumulate reduction terms.
template <int MODE>
__device__ __forceinline__ void spmv_epilogue(int64_t i, double acc, const SpmvArgs &a, const RowPre &p,
                                              double &red0, double &red1) {
  if (MODE == SP_PLAIN) {
    a.y[i] = acc;
  } else if (MODE == SP_JACOBI_R0) {  // v, t: streaming stores (consumed by the vector kernels
    const double v = p.inv * acc;    // after the whole matrix has streamed through L2)
    __stcs(a.y + i, v);
    red0 = fma(p.aux, v, red0);
  } else if (MODE == SP_JACOBI_TT) {
    const double t = p.inv * acc;
    __stcs(a.y + i, t);
    red0 = fma(t, t, red0);
    red1 = fma(t, p.xi, red1);
  } else if (MODE == SP_RESIDUAL) {
    const double r = p.inv * (p.aux - acc);
    a.y[i] = r;
    a.aux2[i] = r;
    const double dr = p.dg * r;
    red0 = fma(dr, dr, red0);
    red1 = fma(r, r, red1);
  } else if (MODE == SP_PQ) {  // q = A p, p.q
    a.y[i] = acc;
    red0 = fma(p.xi, acc, red0);
  } else {  // SP_CGRES: r = b - A x, p = z = D^-1 r, ||r||^2, r.z
    const double r = p.aux - acc;
    const double z = p.inv * r;
    a.y[i] = r;
    a.aux2[i] = z;
    red0 = fma(r, r, red0);
    red1 = fma(r, z, red1);
  }
}

// Scalar updates performed by the last block of a reduction launch (one rank).
template <int MODE>
__device__ __forceinline__ void spmv_stage(KrylovScalars *S, const double (&tot)[2]) {
  if (MODE == SP_JACOBI_R0) apply_stage(ST_R0, S, tot);
  else if (MODE == SP_JACOBI_TT) apply_stage(ST_TT, S, tot);
  else if (MODE == SP_RESIDUAL) apply_stage(ST_RES, S, tot);
  else if (MODE == SP_PQ) apply_stage(ST_PQ, S, tot);
  else if (MODE == SP_CGRES) apply_stage(ST_CGRES, S, tot);
}

// Sum three per-lane partials over the warp with a reduce-scatter (6 double shuffles
// instead of 3 full butterflies = 15): afterwards lane 0 holds row 0, lane 8 row 1,
// lane 16 row 2.  Fixed tree -> deterministic.
__device__ __forceinline__ double warp_sum3(double y0, double y1, double y2, int lane) {
  const bool h4 = lane & 16;
  const double s0 = h4 ? y0 : y2, s1 = h4 ? y1 : 0.0;
  double k0 = (h4 ? y2 : y0) + __shfl_xor_sync(0xffffffffu, s0, 16);
  double k1 = (h4 ? 0.0 : y1) + __shfl_xor_sync(0xffffffffu, s1, 16);
  const bool h3 = lane & 8;
  double kk = (h3 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h3 ? k0 : k1, 8);
  kk += __shfl_xor_sync(0xffffffffu, kk, 4);
  kk += __shfl_xor_sync(0xffffffffu, kk, 2);
  kk += __shfl_xor_sync(0xffffffffu, kk, 1);
  return kk;
}

// Warp per node, lane per neighbour node j: the lane loads x_m (3 doubles, L2-resident)
// once and the 3x3 block of values A[3n+c, 3m+k] from the three contiguous row segments
// (rows are 3*cnt long; lane j's entries sit at 3j..3j+2 of each row, so a warp load
// instruction covers one row's 27*24 B contiguous span).  12 independent loads per lane,
// ~60 warp instructions per node; values are streamed with an evict-first hint so x stays
// in L2; the 3 row sums use a 6-shuffle reduce-scatter.
// ------------------------------------------------------------------------------------
// FEM3 SpMV, Blackwell bulk-copy pipeline.  One persistent 1024-thread CTA per SM: a
// producer lane streams contiguous node chunks (their CSR values and neighbour lists are
// contiguous in memory for consecutive nodes) into a 3-stage shared-memory ring with
// cp.async.bulk + mbarrier complete_tx; 31 consumer warps take one node each per chunk,
// gather x from L2 and read the values from shared memory.  The copy engine keeps up to
// two 60 KB chunks per SM in flight without spending registers.  Same per-lane arithmetic
// and reduction tree as k_spmv_fem3 -> bit-identical y.
constexpr int kTmaConsumers = 31;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;
constexpr int kTmaStages = 3;
constexpr int kTmaValBytes = 62 * 1024;
constexpr int kTmaNbrBytes = 4096;
constexpr int kTmaExtBytes = 768;  // one row-operand array of a chunk (<= 93 rows + alignment slack)
constexpr int kTmaStageBytes = kTmaValBytes + kTmaNbrBytes + 3 * kTmaExtBytes;
constexpr int kTmaSmem = kTmaStages * kTmaStageBytes + 2 * kTmaStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
constexpr uint32_t kMbarSuspendNs = 20000;
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t ok = 0;
  do {  // suspend-time hint: a waiting warp sleeps instead of re-polling (issue slots, power)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "r"(kMbarSuspendNs)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy below)
__device__ __forceinline__ void cp_async8_hint(void *dst, const void *src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Row operands of the epilogue, streamed into the stage with the values (so the row lanes
// read them from shared memory instead of issuing scattered 8-byte loads).
template <int MODE>
__host__ __device__ constexpr int n_ext() {
  return MODE == SP_JACOBI_R0 ? 2 : MODE == SP_JACOBI_TT ? 2 : MODE == SP_RESIDUAL ? 3 : MODE == SP_PQ ? 1
       : MODE == SP_CGRES ? 2 : 0;
}
template <int MODE>
__device__ __forceinline__ const double *ext_ptr(const SpmvArgs &a, int k) {
  if (MODE == SP_JACOBI_R0) return k == 0 ? a.inv : a.aux;
  if (MODE == SP_JACOBI_TT) return k == 0 ? a.inv : a.x;
  if (MODE == SP_RESIDUAL) return k == 0 ? a.inv : (k == 1 ? a.aux : a.dg);
  if (MODE == SP_PQ) return a.x;
  return k == 0 ? a.inv : a.aux;  // SP_CGRES
}
// operand e is read once per matvec (not the matvec's own input x, which neighbours re-read)
template <int MODE>
__device__ __forceinline__ bool pf_read_once(int k) {
  return !((MODE == SP_JACOBI_TT && k == 1) || MODE == SP_PQ);
}
template <int MODE>
__device__ __forceinline__ RowPre row_pre_from(const double *e0, const double *e1, const double *e2) {
  RowPre p{0.0, 0.0, 0.0, 0.0};
  if (MODE == SP_JACOBI_R0) p.inv = *e0, p.aux = *e1;
  else if (MODE == SP_JACOBI_TT) p.inv = *e0, p.xi = *e1;
  else if (MODE == SP_RESIDUAL) p.inv = *e0, p.aux = *e1, p.dg = *e2;
  else if (MODE == SP_PQ) p.xi = *e0;
  else if (MODE == SP_CGRES) p.inv = *e0, p.aux = *e1;
  return p;
}

// x_m of neighbour node m (3 doubles at 24 m).  XV=0: three 8-byte loads; XV=1: one
// 16-byte load of the aligned pair plus one 8-byte load (x must be 16-byte aligned);
// XV=2 (diagnostic only, wrong results): no gather, to separate its cost.
template <int XV>
__device__ __forceinline__ void load_x3(const double *__restrict__ x, int m, double &x0, double &x1, double &x2) {
  const double *__restrict__ xm = x + 3 * (int64_t)m;
  if (XV == 0) {
    x0 = __ldg(xm), x1 = __ldg(xm + 1), x2 = __ldg(xm + 2);
  } else if (XV == 1) {
    const int odd = m & 1;
    const double2 v = __ldg(reinterpret_cast<const double2 *>(xm + odd));
    const double sc = __ldg(xm + (odd ? 0 : 2));
    x0 = odd ? sc : v.x;
    x1 = odd ? v.x : v.y;
    x2 = odd ? v.y : sc;
  } else {
    x0 = 1.0, x1 = 0.5, x2 = 0.25;
  }
}

// One node's three row sums from a value block `sv` (stage or global) and its neighbour ids.
template <int XV = 0>
__device__ __forceinline__ void node_rows(const double *sv, const int32_t *sn, int cnt, const double *__restrict__ x,
                                          int lane, double &y0, double &y1, double &y2) {
  const int L = 3 * cnt;
  for (int j = lane; j < cnt; j += 32) {
    const int m = sn[j];
    double x0, x1, x2;
    load_x3<XV>(x, m, x0, x1, x2);
    const double *r0 = sv + 3 * j;
    y0 = fma(r0[2], x2, fma(r0[1], x1, fma(r0[0], x0, y0)));
    y1 = fma(r0[L + 2], x2, fma(r0[L + 1], x1, fma(r0[L], x0, y1)));
    y2 = fma(r0[2 * L + 2], x2, fma(r0[2 * L + 1], x1, fma(r0[2 * L], x0, y2)));
  }
}


// spmv_alt.cu launchers (MODE = SpmvMode)
void set_fem3_tma_npw1_attr();
void launch_fem3_tma_npw1(const Matrix *m, int mode, const SpmvArgs &a, const RedScratch &r, int grid);
void launch_sym3_tma(const Matrix *m, int mode, const SpmvArgs &a, const RedScratch &r, int grid);

}  // namespace b200
