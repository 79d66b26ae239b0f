// Per-cell HEX8 weak-form kernels: geometry, constitutive laws, residual, consistent
// tangent (hand-derived), quadrature-point flux, J2 commit.
//
// Reference being replaced (paths relative to gradfem/):
//   elements.py:17-131   reference element tables, map_elements (recomputed per cell here)
//   materials.py:74-131  linear_elastic_flux, neo_hookean_flux (AD of W), j2_return_map
//   problems.py:166-202  SIMP theta^p scaling;  problems.py:319-324 nodal design source
//   assembly.py:176-300  _element_residual, assemble_residual, assemble_jacobian
//   kernels.py:30-34     sequential scatter_add -> ordered per-node gathers
//
// Reduction: per-cell blocks go to a scratch buffer; a per-node gather (or, on box lattices,
// the lattice pull) then sums every R entry / CSR slot over its cells in ascending cell id --
// the reference's sequential scatter order -- with no atomics, so results are bit-identical
// from run to run.

#include <cmath>

#include "internal.cuh"
#include "laws.cuh"

namespace b200 {

__constant__ double c_dN[8][8][3];  // [q][k][d] dphi_k/dxi_d at Gauss point q (x fastest)
__constant__ double c_N[8][8];      // [q][k]    phi_k at Gauss point q
__constant__ int c_pair_a[36], c_pair_b[36];  // symmetric block pairs a <= b
__constant__ int c_pair_idx[8][8];            // (a <= b) -> pair index

void element_tables_init() {
  static bool done = false;
  if (done) return;
  // Same operation order as elements.py:38-77 (terms product / 8).
  const double g = 1.0 / std::sqrt(3.0);
  const double s[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                          {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
  double dN[8][8][3], N[8][8];
  for (int q = 0; q < 8; ++q) {
    double xi[3] = {(q & 1) ? g : -g, (q & 2) ? g : -g, (q & 4) ? g : -g};
    for (int k = 0; k < 8; ++k) {
      double t[3];
      for (int d = 0; d < 3; ++d) t[d] = 1.0 + xi[d] * s[k][d];
      N[q][k] = t[0] * t[1] * t[2] / 8.0;
      dN[q][k][0] = s[k][0] * (t[1] * t[2]) / 8.0;
      dN[q][k][1] = s[k][1] * (t[0] * t[2]) / 8.0;
      dN[q][k][2] = s[k][2] * (t[0] * t[1]) / 8.0;
    }
  }
  cudaMemcpyToSymbol(c_dN, dN, sizeof(dN));
  cudaMemcpyToSymbol(c_N, N, sizeof(N));
  int pa[36], pb[36], pidx[8][8];
  int p = 0;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) pidx[a][b] = -1;
  for (int a = 0; a < 8; ++a)
    for (int b = a; b < 8; ++b) {
      pa[p] = a;
      pb[p] = b;
      pidx[a][b] = p++;
    }
  cudaMemcpyToSymbol(c_pair_a, pa, sizeof(pa));
  cudaMemcpyToSymbol(c_pair_b, pb, sizeof(pb));
  cudaMemcpyToSymbol(c_pair_idx, pidx, sizeof(pidx));
  done = true;
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
static double unord_bits(unsigned long long u) {
  unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
  double d;
  memcpy(&d, &b, sizeof(d));
  return d;
}

// The same with the point's dphi table in shared memory (dNq[k*3 + d]): lanes of one warp
// working on different Gauss points would serialise on divergent __constant__ addresses.
__device__ __forceinline__ double qp_geometry_s(const double (*X)[3], const double *dNq, double (&G)[8][3]) {
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) J[a][b] = fma(X[k][a], dNq[k * 3 + b], J[a][b]);
  const double a = J[0][0], b = J[0][1], c = J[0][2], d = J[1][0], e = J[1][1], f = J[1][2], g = J[2][0],
               h = J[2][1], i = J[2][2];
  const double A = e * i - f * h, B = c * h - b * i, C = b * f - c * e;
  const double D = f * g - d * i, E = a * i - c * g, F = c * d - a * f;
  const double Gc = d * h - e * g, H = b * g - a * h, I = a * e - b * d;
  const double det = a * A + b * D + c * Gc;
  const double r = 1.0 / det;
  const double inv[3][3] = {{A * r, B * r, C * r}, {D * r, E * r, F * r}, {Gc * r, H * r, I * r}};
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int aa = 0; aa < 3; ++aa)
      G[k][aa] = inv[0][aa] * dNq[k * 3] + inv[1][aa] * dNq[k * 3 + 1] + inv[2][aa] * dNq[k * 3 + 2];
  return det;
}

// J = sum_k X_k (x) dphi_k, cofactor inverse, G_k = J^-T dphi_k (elements.py:117-131)
__device__ __forceinline__ double qp_geometry(const double (*X)[3], int q, double (&G)[8][3]) {
  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) J[a][b] = fma(X[k][a], c_dN[q][k][b], J[a][b]);
  const double a = J[0][0], b = J[0][1], c = J[0][2], d = J[1][0], e = J[1][1], f = J[1][2], g = J[2][0],
               h = J[2][1], i = J[2][2];
  const double A = e * i - f * h, B = c * h - b * i, C = b * f - c * e;
  const double D = f * g - d * i, E = a * i - c * g, F = c * d - a * f;
  const double Gc = d * h - e * g, H = b * g - a * h, I = a * e - b * d;
  const double det = a * A + b * D + c * Gc;
  const double r = 1.0 / det;
  const double inv[3][3] = {{A * r, B * r, C * r}, {D * r, E * r, F * r}, {Gc * r, H * r, I * r}};
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int aa = 0; aa < 3; ++aa)
      G[k][aa] = inv[0][aa] * c_dN[q][k][0] + inv[1][aa] * c_dN[q][k][1] + inv[2][aa] * c_dN[q][k][2];
  return det;
}

struct ElemArgs {
  const double *coords;
  const int32_t *cells;
  const double *U;
  const double *theta;
  const double *eps_prev, *sig_prev;
  MatParams mp;
  DevErr *derr;
};

// 8-lane reduce-scatter: lane q of the group ends with the sum over the group of v[q*V..]
template <int V>
__device__ __forceinline__ void reduce_scatter8(double (&r)[8 * V], int q, double (&out)[V]) {
  // step 1: halves by bit 2
  double h1[4 * V];
  const bool lo2 = !(q & 4);
#pragma unroll
  for (int j = 0; j < 4 * V; ++j) {
    double send = lo2 ? r[j + 4 * V] : r[j];
    double keep = lo2 ? r[j] : r[j + 4 * V];
    h1[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  double h2[2 * V];
  const bool lo1 = !(q & 2);
#pragma unroll
  for (int j = 0; j < 2 * V; ++j) {
    double send = lo1 ? h1[j + 2 * V] : h1[j];
    double keep = lo1 ? h1[j] : h1[j + 2 * V];
    h2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  const bool lo0 = !(q & 1);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    double send = lo0 ? h2[j + V] : h2[j];
    double keep = lo0 ? h2[j] : h2[j + V];
    out[j] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
}

__device__ __forceinline__ bool all_finite(const double (&P)[3][3], int vec) {
  bool ok = true;
  for (int i = 0; i < vec; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) ok &= isfinite(P[i][j]);
  return ok;
}

// ------------------------------------------------------------- residual
// 8 lanes per cell (lane q = quadrature point), 4 cells per warp.
template <int MAT>
__global__ void __launch_bounds__(kThreads, 2) k_residual(ElemArgs a, int64_t n, double *__restrict__ Re) {
  constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  __shared__ double sX[kWarps][4][8][3];
  __shared__ double sU[kWarps][4][8][VEC];
  __shared__ double sT[kWarps][4][8];
  __shared__ double sdN[8 * 25];  // [q][k*3 + d], point stride 25 (odd: conflict-free)
  for (int t = threadIdx.x; t < 192; t += blockDim.x) sdN[(t / 24) * 25 + t % 24] = (&c_dN[0][0][0])[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, slot = lane >> 3, q = lane & 7;
  const double *dNq = sdN + q * 25;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp0 * 4; base < n; base += nwarps * 4) {
    const int64_t idx = base + slot;
    const bool valid = idx < n;
    const int64_t e = valid ? idx : base;
    const int node = a.cells[e * 8 + q];
#pragma unroll
    for (int d = 0; d < 3; ++d) sX[w][slot][q][d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
    for (int v = 0; v < VEC; ++v) sU[w][slot][q][v] = a.U[(int64_t)node * VEC + v];
    if (MAT == B200FEM_MAT_POISSON && a.mp.design_source) sT[w][slot][q] = a.theta[node];
    __syncwarp();
    double G[8][3];
    const double jxw = qp_geometry_s(sX[w][slot], dNq, G);
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) gu[v][d] = fma(sU[w][slot][k][v], G[k][d], gu[v][d]);
    const double *ep = nullptr, *sp = nullptr;
    if (MAT == B200FEM_MAT_J2) {
      ep = a.eps_prev + (e * 8 + q) * 9;
      sp = a.sig_prev + (e * 8 + q) * 9;
    }
    double P[3][3], detF = 1.0;
    const bool ok = flux_at<MAT>(gu, a.mp, ep, sp, P, detF);
    double scale = jxw;
    if (a.mp.simp) scale *= pow(a.theta[e], a.mp.penalty);
    if (valid) {
      const unsigned long long key = (unsigned long long)e * 8 + q;
      if (!ok) {
        atomicMin(&a.derr->inv_def, key);
        atomicMin(&a.derr->min_detF, ord_bits(detF));
      } else if (!all_finite(P, VEC)) {
        atomicMin(&a.derr->nonfin_v, key);
      }
    }
    double r[8 * VEC];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v)
        r[k * VEC + v] = scale * (P[v][0] * G[k][0] + P[v][1] * G[k][1] + P[v][2] * G[k][2]);
    if (MAT == B200FEM_MAT_POISSON && a.mp.design_source) {
      double bq = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) bq = fma(sT[w][slot][k], c_N[q][k], bq);
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] -= bq * c_N[q][k] * jxw;
    }
    double mine[VEC];
    reduce_scatter8<VEC>(r, q, mine);
    if (valid) {  // element block R_e[e, q, :] (node q of the cell), coalesced per cell
#pragma unroll
      for (int v = 0; v < VEC; ++v) Re[(e * 8 + q) * VEC + v] = mine[v];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------- design VJP
// out = w_eff^T dR/dtheta (assembly.py:303-341), w_eff = w with the Dirichlet rows zeroed
// (they do not depend on theta).  SIMP (element layout, problems.py:166-170): the flux is
// theta_e^p sigma(grad u), so dR_e/dtheta_e = p theta_e^(p-1) * (unscaled element
// residual) and out[e] = that dotted with w_e.  8 lanes per cell as in k_residual.
template <int MAT>
__global__ void __launch_bounds__(kThreads, 2) k_vjp_simp(ElemArgs a, int64_t n, const double *__restrict__ th,
                                                          const double *__restrict__ w,
                                                          const uint8_t *__restrict__ dflag, double *__restrict__ out) {
  __shared__ double sX[kWarps][4][8][3];
  __shared__ double sU[kWarps][4][8][3];
  __shared__ double sW[kWarps][4][8][3];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, slot = lane >> 3, q = lane & 7;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp0 * 4; base < n; base += nwarps * 4) {
    const int64_t idx = base + slot;
    const bool valid = idx < n;
    const int64_t e = valid ? idx : base;
    const int node = a.cells[e * 8 + q];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t dof = (int64_t)node * 3 + d;
      sX[wp][slot][q][d] = a.coords[dof];
      sU[wp][slot][q][d] = a.U[dof];
      sW[wp][slot][q][d] = (dflag && dflag[dof]) ? 0.0 : w[dof];
    }
    __syncwarp();
    double G[8][3];
    const double jxw = qp_geometry(sX[wp][slot], q, G);
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int v = 0; v < 3; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) gu[v][d] = fma(sU[wp][slot][k][v], G[k][d], gu[v][d]);
    double P[3][3], detF = 1.0;
    const bool ok = flux_at<MAT>(gu, a.mp, nullptr, nullptr, P, detF);
    if (valid) {
      const unsigned long long key = (unsigned long long)e * 8 + q;
      if (!ok) {
        atomicMin(&a.derr->inv_def, key);
        atomicMin(&a.derr->min_detF, ord_bits(detF));
      } else if (!all_finite(P, 3)) {
        atomicMin(&a.derr->nonfin_v, key);
      }
    }
    const double sc = jxw * (a.mp.penalty * pow(th[e], a.mp.penalty - 1.0));
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int v = 0; v < 3; ++v)
        acc = fma(sc * (P[v][0] * G[k][0] + P[v][1] * G[k][1] + P[v][2] * G[k][2]), sW[wp][slot][k][v], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (valid && q == 0) out[e] = acc;
    __syncwarp();
  }
}

// Poisson design source (node layout, problems.py:125-130): b_q = sum_k theta_k N_k(q)
// enters R_e,i as -sum_q b_q N_i(q) JxW_q, so the VJP of cell e at its local node k is
// -sum_q N_k(q) JxW_q (sum_i N_i(q) w_i); written per (cell, local node) for the ordered
// node gather (the reference's scatter_add over cells[sl].ravel()).
__global__ void __launch_bounds__(kThreads, 2) k_vjp_source(ElemArgs a, int64_t n, const double *__restrict__ w,
                                                            const uint8_t *__restrict__ dflag,
                                                            double *__restrict__ Re) {
  __shared__ double sX[kWarps][4][8][3];
  __shared__ double sW[kWarps][4][8];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, slot = lane >> 3, q = lane & 7;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp0 * 4; base < n; base += nwarps * 4) {
    const int64_t idx = base + slot;
    const bool valid = idx < n;
    const int64_t e = valid ? idx : base;
    const int node = a.cells[e * 8 + q];
#pragma unroll
    for (int d = 0; d < 3; ++d) sX[wp][slot][q][d] = a.coords[(int64_t)node * 3 + d];
    sW[wp][slot][q] = (dflag && dflag[node]) ? 0.0 : w[node];
    __syncwarp();
    double G[8][3];
    const double jxw = qp_geometry(sX[wp][slot], q, G);
    double wq = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) wq = fma(c_N[q][k], sW[wp][slot][k], wq);
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = -(c_N[q][k] * wq * jxw);
    double mine[1];
    reduce_scatter8<1>(r, q, mine);
    if (valid) Re[e * 8 + q] = mine[0];
    __syncwarp();
  }
}

// ------------------------------------------------------------- L2 field error
// inverse.py:45-56: per quadrature point d = sum_k N_k(q) u_k for the predicted and true
// nodal fields; sums of (d_p - d_t)^2 JxW and d_t^2 JxW (deterministic block reduction).
__global__ void __launch_bounds__(kThreads) k_l2_error(const double *__restrict__ X, const int32_t *__restrict__ cells,
                                                       int64_t n, const double *__restrict__ up,
                                                       const double *__restrict__ ut, RedScratch red,
                                                       double *__restrict__ out) {
  __shared__ double sX[kWarps][4][8][3];
  __shared__ double sP[kWarps][4][8], sT[kWarps][4][8];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, slot = lane >> 3, q = lane & 7;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[2] = {0.0, 0.0};
  for (int64_t base = warp0 * 4; base < n; base += nwarps * 4) {
    const int64_t idx = base + slot;
    const bool valid = idx < n;
    const int64_t e = valid ? idx : base;
    const int node = cells[e * 8 + q];
#pragma unroll
    for (int d = 0; d < 3; ++d) sX[wp][slot][q][d] = X[(int64_t)node * 3 + d];
    sP[wp][slot][q] = up[node];
    sT[wp][slot][q] = ut[node];
    __syncwarp();
    double G[8][3];
    const double jxw = qp_geometry(sX[wp][slot], q, G);
    double dp = 0.0, dt = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dp = fma(c_N[q][k], sP[wp][slot][k], dp);
      dt = fma(c_N[q][k], sT[wp][slot][k], dt);
    }
    if (valid) {
      const double df = dp - dt;
      acc[0] = fma(df * df, jxw, acc[0]);
      acc[1] = fma(dt * dt, jxw, acc[1]);
    }
    __syncwarp();
  }
  double tot[2];
  if (block_partials_and_finish<2>(acc, red, tot) && threadIdx.x == 0) out[0] = tot[0], out[1] = tot[1];
}

// Ordered gather (assembly.py:256 semantics): R[n] = sum over the node's incident cells in
// ascending cell id of R_e[e, a(n,e)] -- the reference's accumulation order, no atomics.
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_residual_gather(const int32_t *__restrict__ n2c_ptr,
                                                              const int32_t *__restrict__ n2c,
                                                              const uint8_t *__restrict__ n2c_a,
                                                              const double *__restrict__ Re, int64_t n_nodes,
                                                              double s, const double *__restrict__ fN,
                                                              const double *__restrict__ fB, double *__restrict__ R) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_nodes * VEC;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / VEC;
    const int v = (int)(t - n * VEC);
    double acc = 0.0;
    for (int k = __ldg(n2c_ptr + n), k1 = __ldg(n2c_ptr + n + 1); k < k1; ++k)
      acc += __ldg(Re + ((int64_t)__ldg(n2c + k) * 8 + __ldg(n2c_a + k)) * VEC + v);
    if (fN) acc -= s * fN[t];
    if (fB) acc -= fB[t];
    R[t] = acc;
  }
}

__global__ void k_res_finalize(double *__restrict__ R, int64_t n, double s, const double *__restrict__ fN,
                               const double *__restrict__ fB) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double r = R[i];
    if (fN) r -= s * fN[i];
    if (fB) r -= fB[i];
    R[i] = r;
  }
}

__global__ void k_res_dirichlet(double *__restrict__ R, const double *__restrict__ U, const int32_t *__restrict__ dofs,
                                const double *__restrict__ vals, int64_t n, double s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int d = dofs[i];
    R[d] = U[d] - s * vals[i];
  }
}

// ------------------------------------------------------------- jacobian
// Phase A, warp per cell.  Phase 1 uses all 32 lanes: lane (q, part) = (lane>>2, lane&3)
// owns quadrature point q and nodes {part, part+4}; J and grad u are reduced over the 4
// lanes of a point with shuffles, and each lane tabulates its two nodes' vectors in shared
// memory.  The tangent block of pair (a,b) at a point is written in a factored form with
// one FMA per term (coefficients include JxW and theta^p):
//   NH:  K_ik += c1 d_ik (g_a.g_b) + h_a,i w_b,k + z_a,i h_b,k + t_b,i h_a,k
//        h = H g, w = c3 h - c2 F g, z = -c2 F g, t = c4 h,
//        c1 = G a, c2 = 2/3 G a, c3 = 2/9 G a I1 + k J(2J-1), c4 = G/3 a I1 - k J(J-1)
//   J2:  K_ik += c1 d_ik (g_a.g_b) + cl g_a,i g_b,k + cm g_a,k g_b,i + y_a,i (c3 y_b,k),  y = s g
//        c1 = cm = mu - beta/2, cl = lam + beta/3, c3 = -gamma
//   LE:  J2 with beta = gamma = 0;   Poisson: alpha JxW (g_a.g_b)
// (the algebra of SURVEY.md Appendix A; NH/J2 verified against the reference's AD Jacobian).
// Phase 2: lane p computes the symmetric pair p of the 36 pairs a <= b over the 8 points and
// writes the 3x3 block to the per-cell scratch.
constexpr int kJacWarps = 4;

template <int MAT>
#ifndef JAC_NP
#define JAC_NP 9
#endif
struct JacSmem {
  // node dimension padded to JAC_NP: phase 1 stores [q][part + 4t][d] from lane (q, part),
  // whose row stride decides the shared-memory bank conflicts
  double X[8][3];
  double U[8][3];
  double g[8][JAC_NP][3];
  double h[(MAT == B200FEM_MAT_NH || MAT == B200FEM_MAT_J2) ? 8 : 1][JAC_NP][3];  // NH: H g; J2: c3 * s g
  double w[(MAT == B200FEM_MAT_NH || MAT == B200FEM_MAT_J2) ? 8 : 1][JAC_NP][3];  // NH: c3 h - c2 u; J2: s g
  double z[(MAT == B200FEM_MAT_NH) ? 8 : 1][JAC_NP][3];
  double t[(MAT == B200FEM_MAT_NH) ? 8 : 1][JAC_NP][3];
  double coef[8][3];  // c1, cl, cm
};

__device__ __forceinline__ double quad_sum(double v) {  // sum over the 4 lanes of a point
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// Contribution of quadrature point qq to the VEC x VEC block of pair (a0, b), added to K.
template <int MAT, int VEC>
__device__ __forceinline__ void jac_pair_qp(const JacSmem<MAT> &S, int a0, int b, int qq, double (&K)[VEC][VEC]) {
    const double ga[3] = {S.g[qq][a0][0], S.g[qq][a0][1], S.g[qq][a0][2]};
    const double gb[3] = {S.g[qq][b][0], S.g[qq][b][1], S.g[qq][b][2]};
    const double gg = ga[0] * gb[0] + ga[1] * gb[1] + ga[2] * gb[2];
    const double d = S.coef[qq][0] * gg;
    if (MAT == B200FEM_MAT_POISSON) {
      K[0][0] += d;
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i) K[i][i] += d;
      if (MAT == B200FEM_MAT_LE || MAT == B200FEM_MAT_J2) {
        const double cl = S.coef[qq][1], cm = S.coef[qq][2];
        double la[3], ma[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          la[i] = cl * ga[i];
          ma[i] = cm * gb[i];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) K[i][k] = fma(la[i], gb[k], fma(ma[i], ga[k], K[i][k]));
      }
      if (MAT == B200FEM_MAT_J2) {
        const double ya[3] = {S.w[qq][a0][0], S.w[qq][a0][1], S.w[qq][a0][2]};
        const double cyb[3] = {S.h[qq][b][0], S.h[qq][b][1], S.h[qq][b][2]};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) K[i][k] = fma(ya[i], cyb[k], K[i][k]);
      }
      if (MAT == B200FEM_MAT_NH) {
        const double ha[3] = {S.h[qq][a0][0], S.h[qq][a0][1], S.h[qq][a0][2]};
        const double hb[3] = {S.h[qq][b][0], S.h[qq][b][1], S.h[qq][b][2]};
        const double wb[3] = {S.w[qq][b][0], S.w[qq][b][1], S.w[qq][b][2]};
        const double za[3] = {S.z[qq][a0][0], S.z[qq][a0][1], S.z[qq][a0][2]};
        const double tb[3] = {S.t[qq][b][0], S.t[qq][b][1], S.t[qq][b][2]};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) K[i][k] = fma(ha[i], wb[k], fma(za[i], hb[k], fma(tb[i], ha[k], K[i][k])));
      }
    }
}

// Scratch layouts of the 36 symmetric cell blocks: cell-major [cell][pair][VV] for the ordered
// per-node gather of the CSR / SYM3 paths, or element-major [pair][VV][cell] for the lattice
// pull of the GRID path (consecutive nodes read consecutive cells: coalesced).
template <int VEC>
__device__ __forceinline__ void jac_store(double *__restrict__ Ke, int64_t e, int64_t n_cells, int p, int soa,
                                          const double (&K)[VEC][VEC]) {
  constexpr int VV = VEC * VEC;
#pragma unroll
  for (int i = 0; i < VEC; ++i)
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      if (soa) Ke[((int64_t)p * VV + i * VEC + k) * n_cells + e] = K[i][k];
      else Ke[(e * 36 + p) * VV + i * VEC + k] = K[i][k];
    }
}

template <int MAT>
__global__ void __launch_bounds__(kJacWarps * 32, 6) k_jacobian(ElemArgs a, int64_t n, double *__restrict__ Ke,
                                                                 int soa) {
  constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  __shared__ JacSmem<MAT> sm_all[kJacWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  JacSmem<MAT> &S = sm_all[w];
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int q = lane >> 2, part = lane & 3;
  for (int64_t e = warp0; e < n; e += nwarps) {
    if (lane < 8) {
      const int node = a.cells[e * 8 + lane];
#pragma unroll
      for (int d = 0; d < 3; ++d) S.X[lane][d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
      for (int v = 0; v < VEC; ++v) S.U[lane][v] = a.U[(int64_t)node * VEC + v];
    }
    __syncwarp();
    {  // ---- phase 1
      double Jm[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double pj = S.X[part][i] * c_dN[q][part][j] + S.X[part + 4][i] * c_dN[q][part + 4][j];
          Jm[i][j] = quad_sum(pj);
        }
      const double A0 = Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1], B0 = Jm[0][2] * Jm[2][1] - Jm[0][1] * Jm[2][2];
      const double C0 = Jm[0][1] * Jm[1][2] - Jm[0][2] * Jm[1][1], D0 = Jm[1][2] * Jm[2][0] - Jm[1][0] * Jm[2][2];
      const double E0 = Jm[0][0] * Jm[2][2] - Jm[0][2] * Jm[2][0], F0 = Jm[0][2] * Jm[1][0] - Jm[0][0] * Jm[1][2];
      const double G0 = Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0], H0 = Jm[0][1] * Jm[2][0] - Jm[0][0] * Jm[2][1];
      const double I0 = Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0];
      const double jxw = Jm[0][0] * A0 + Jm[0][1] * D0 + Jm[0][2] * G0;
      const double r = 1.0 / jxw;
      const double inv[3][3] = {{A0 * r, B0 * r, C0 * r}, {D0 * r, E0 * r, F0 * r}, {G0 * r, H0 * r, I0 * r}};
      double scale = jxw;
      if (a.mp.simp) scale *= pow(a.theta[e], a.mp.penalty);
      double Gk[2][3];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int k = part + 4 * t;
#pragma unroll
        for (int aa = 0; aa < 3; ++aa)
          Gk[t][aa] = inv[0][aa] * c_dN[q][k][0] + inv[1][aa] * c_dN[q][k][1] + inv[2][aa] * c_dN[q][k][2];
#pragma unroll
        for (int d = 0; d < 3; ++d) S.g[q][k][d] = Gk[t][d];
      }
      bool bad_def = false, fin = true, vfin = true;
      double detF = 1.0;
      if (MAT == B200FEM_MAT_POISSON) {
        if (part == 0) S.coef[q][0] = a.mp.alpha * scale;
        // the flux value alpha grad u must be finite (the reference checks the AD value first,
        // assembly.py:216-233, even though this tangent does not depend on U)
        double gs = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) gs += fabs(quad_sum(S.U[part][0] * Gk[0][d] + S.U[part + 4][0] * Gk[1][d]));
        vfin = isfinite(gs);
      } else {
        double gu[3][3];
        double gs = 0.0;
#pragma unroll
        for (int v = 0; v < 3; ++v)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            gu[v][d] = quad_sum(S.U[part][v] * Gk[0][d] + S.U[part + 4][v] * Gk[1][d]);
            gs += fabs(gu[v][d]);
          }
        vfin = isfinite(gs);
        if (MAT == B200FEM_MAT_LE) {
          if (part == 0) {
            S.coef[q][0] = a.mp.mu * scale;
            S.coef[q][1] = a.mp.lam * scale;
            S.coef[q][2] = a.mp.mu * scale;
          }
        } else if (MAT == B200FEM_MAT_NH) {
          double F[3][3];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) F[i][j] = gu[i][j] + (i == j ? 1.0 : 0.0);
          const double J = det3(F);
          detF = J;
          double H[3][3];
          if (!(J <= 0.0)) {  // NaN: a non-finite value, not an inversion (materials.py:94)
            inv_transpose(F, J, H);
          } else {
            bad_def = true;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int j = 0; j < 3; ++j) H[i][j] = 0.0;
          }
          double I1 = 0.0;
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) I1 += F[i][j] * F[i][j];
          vfin = vfin && isfinite(J) && isfinite(I1);
          const double rc = bad_def ? 0.0 : rcbrt(J);
          const double aa = rc * rc;  // J^{-2/3}
          const double Ga = a.mp.mu * aa;
          const double c1 = Ga * scale, c2 = (2.0 / 3.0) * Ga * scale;
          const double c3 = ((2.0 / 9.0) * Ga * I1 + a.mp.kappa * J * (2.0 * J - 1.0)) * scale;
          const double c4 = ((1.0 / 3.0) * Ga * I1 - a.mp.kappa * J * (J - 1.0)) * scale;
          fin = isfinite(c1) && isfinite(c2) && isfinite(c3) && isfinite(c4);
          if (part == 0) S.coef[q][0] = c1;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int k = part + 4 * t;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              const double uk = F[i][0] * Gk[t][0] + F[i][1] * Gk[t][1] + F[i][2] * Gk[t][2];
              const double hk = H[i][0] * Gk[t][0] + H[i][1] * Gk[t][1] + H[i][2] * Gk[t][2];
              S.h[q][k][i] = hk;
              S.w[q][k][i] = c3 * hk - c2 * uk;
              S.z[q][k][i] = -c2 * uk;
              S.t[q][k][i] = c4 * hk;
            }
          }
        } else {  // J2 consistent tangent (derivative of j2_return_map incl. the s=0 guard)
          const double *ep = a.eps_prev + (e * 8 + q) * 9;
          const double *sp = a.sig_prev + (e * 8 + q) * 9;
          double st[3][3], sd[3][3], seff;
          bool pos;
          j2_trial(gu, ep, sp, a.mp, st, sd, seff, pos);
          const double over = fmax(seff - a.mp.sy, 0.0);
          const double f = over / seff;
          const double active = (seff - a.mp.sy > 0.0) ? 1.0 : 0.0;  // ramp'(0) = 0
          const double gam = pos ? (active / seff - over / (seff * seff)) * 3.0 * a.mp.mu / seff : 0.0;
          const double beta = 2.0 * a.mp.mu * f;
          const double c1 = (a.mp.mu - 0.5 * beta) * scale, cl = (a.mp.lam + beta / 3.0) * scale;
          const double c3 = -gam * scale;
          fin = isfinite(c1) && isfinite(cl) && isfinite(c3);
          vfin = vfin && isfinite(seff) && isfinite(st[0][0] + st[1][1] + st[2][2]);
          if (part == 0) {
            S.coef[q][0] = c1;
            S.coef[q][1] = cl;
            S.coef[q][2] = c1;
          }
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int k = part + 4 * t;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              const double y = sd[i][0] * Gk[t][0] + sd[i][1] * Gk[t][1] + sd[i][2] * Gk[t][2];
              S.w[q][k][i] = y;
              S.h[q][k][i] = c3 * y;
            }
          }
        }
      }
      if (part == 0) {
        const unsigned long long key = (unsigned long long)e * 8 + q;
        if (bad_def) {
          atomicMin(&a.derr->inv_def, key);
          atomicMin(&a.derr->min_detF, ord_bits(detF));
        } else if (!vfin) {  // the flux value itself is non-finite (assembly.py:228-233)
          atomicMin(&a.derr->nonfin_v, key);
        } else if (!fin) {
          atomicMin(&a.derr->nonfin_d, key);
        }
      }
    }
    __syncwarp();
    // ---- phase 2: the 36 symmetric pairs a <= b.  Round 1: lane p = pair p over all 8
    // points.  Round 2: the last 4 pairs split over 8 lanes each (lane = one point), summed
    // by a fixed 3-level shuffle tree -- 1.125 rounds of work instead of 2 (a second round
    // of only 4 busy lanes).
    {
      const int p = lane, a0 = c_pair_a[p], b = c_pair_b[p];
      double K[VEC][VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i)
#pragma unroll
        for (int k = 0; k < VEC; ++k) K[i][k] = 0.0;
#pragma unroll 2
      for (int qq = 0; qq < 8; ++qq) jac_pair_qp<MAT, VEC>(S, a0, b, qq, K);
      jac_store<VEC>(Ke, e, n, p, soa, K);
    }
    {
      const int p = 32 + (lane >> 3), qq = lane & 7, a0 = c_pair_a[p], b = c_pair_b[p];
      double K[VEC][VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i)
#pragma unroll
        for (int k = 0; k < VEC; ++k) K[i][k] = 0.0;
      jac_pair_qp<MAT, VEC>(S, a0, b, qq, K);
#pragma unroll
      for (int i = 0; i < VEC; ++i)
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
          double v = K[i][k];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          K[i][k] = v;
        }
      if (qq == 0) jac_store<VEC>(Ke, e, n, p, soa, K);
    }
    __syncwarp();
  }
}

// ------------------------------------------------- jacobian phase A, node-lane mapping
// Four cells per warp; lane (c, a) = (lane >> 3, lane & 7).
//  1. lane (c, q) -- the same lanes read as (cell, Gauss point) -- computes the geometry, grad u,
//     the law's scalars and the per-node vectors V_a(q) of its point for all 8 nodes a
//     (NH: g, h = H g, u = F g; J2: g, y = s g; LE / Poisson: g) into shared memory;
//  2. lane (c, a) then owns the symmetric pairs (a, (a + d) mod 8), d = 0..3 (and d = 4 for
//     a < 4): 36 pairs over 8 lanes, 4 or 5 blocks in registers, accumulated over the 8 points.
//     Per point a lane reads only the partner vectors V_b (9 doubles for NH: g, h and
//     w = c3 h - c2 u formed once per node in step 1) -- the operands it
//     reuses (V_a, the coefficients) stay in registers -- so shared-memory wavefronts per cell
//     drop ~3x against the pair-per-lane kernel above (its 858 wavefronts/cell made it
//     L1-bound, profiles/r01_ncu_jacobian_nh.json).
// Block algebra (same as above; the own -c2 u_a is recovered as w_a - c3 h_a):
//   NH:  K_ik += c1 d_ik (g_a.g_b) + h_a,i w_b,k - c2 u_a,i h_b,k + c4 h_a,k h_b,i
//   J2:  K_ik += c1 d_ik (g_a.g_b) + cl g_a,i g_b,k + c1 g_a,k g_b,i + c3 y_a,i y_b,k
//   LE:  J2 without the y term;  Poisson: c1 (g_a.g_b)
// Shared-memory strides are padded so that every access pattern is bank-conflict free.
constexpr int kJac2Warps = 4;

template <int MAT>
struct Jac2Cfg {
  static constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  static constexpr int NV = (MAT == B200FEM_MAT_NH) ? 9 : (MAT == B200FEM_MAT_J2) ? 6 : 3;  // vector doubles
  static constexpr int QS = 8 * NV + 1;   // point stride (odd: conflict-free across points)
  static constexpr int CS = 8 * QS;       // cell stride = 64 NV + 8 = 8 (mod 16): two cells 16 banks apart
  static_assert(CS % 16 == 8, "cell stride must be 8 mod 16 doubles");
  // dynamic shared memory (doubles): dN table [q][25] | X,U [w][c][k][7] | V [w][4 CS] | coef [w][160]
  // per-warp V region, also the staging buffer of the element-major scratch stores (36 pairs x
  // VEC^2 entries x 4 cells): the larger of the two
  static constexpr int VW = (4 * CS > 36 * VEC * VEC * 4) ? 4 * CS : 36 * VEC * VEC * 4;
  static constexpr int SM_DN = 8 * 25, SM_XU = kJac2Warps * 4 * 8 * 7, SM_V = kJac2Warps * VW,
                       SM_C = kJac2Warps * 160;
  static constexpr size_t BYTES = sizeof(double) * (SM_DN + SM_XU + SM_V + SM_C);
};

// Phase A of four cells (one per 8-lane group c = lane >> 3; cell e of this lane's group,
// `valid` false for padding lanes): on return lane (c, a) holds in K[d] the block of the pair
// (a, (a + d) mod 8), d = 0..3 (and 4 for a < 4), as K_{(a,i),(b,k)}.  Element errors are
// flagged on the device (DevErr) exactly as the other element kernels do.
template <int MAT, bool LOADED = false>
__device__ __forceinline__ void jac2_cell_blocks(const ElemArgs &a, int64_t e, bool valid, int lane,
                                                 const double *__restrict__ sdN, double (*sXUw)[8][7], double *V,
                                                 double *Cf, double (&K)[5][Jac2Cfg<MAT>::VEC * Jac2Cfg<MAT>::VEC]) {
  using CF = Jac2Cfg<MAT>;
  constexpr int VEC = CF::VEC, NV = CF::NV, QS = CF::QS, CS = CF::CS;
  constexpr int NB = 5, BB = VEC * VEC;
  const int c = lane >> 3, a8 = lane & 7;
  if (!LOADED) {  // node a8 of cell c: coordinates and U (LOADED: the caller staged them)
    const int node = a.cells[e * 8 + a8];
#pragma unroll
    for (int d = 0; d < 3; ++d) sXUw[c][a8][d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
    for (int v = 0; v < VEC; ++v) sXUw[c][a8][3 + v] = a.U[(int64_t)node * VEC + v];
  }
  __syncwarp();
  {  // ---- 1. lane (c, q): point quantities and the per-node vectors
    const int q = a8;
    double Jm[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double d0 = sdN[q * 25 + k * 3], d1 = sdN[q * 25 + k * 3 + 1], d2 = sdN[q * 25 + k * 3 + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double x = sXUw[c][k][i];
        Jm[i][0] = fma(x, d0, Jm[i][0]);
        Jm[i][1] = fma(x, d1, Jm[i][1]);
        Jm[i][2] = fma(x, d2, Jm[i][2]);
      }
    }
    const double A0 = Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1], B0 = Jm[0][2] * Jm[2][1] - Jm[0][1] * Jm[2][2];
    const double C0 = Jm[0][1] * Jm[1][2] - Jm[0][2] * Jm[1][1], D0 = Jm[1][2] * Jm[2][0] - Jm[1][0] * Jm[2][2];
    const double E0 = Jm[0][0] * Jm[2][2] - Jm[0][2] * Jm[2][0], F0 = Jm[0][2] * Jm[1][0] - Jm[0][0] * Jm[1][2];
    const double G0 = Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0], H0 = Jm[0][1] * Jm[2][0] - Jm[0][0] * Jm[2][1];
    const double I0 = Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0];
    const double jxw = Jm[0][0] * A0 + Jm[0][1] * D0 + Jm[0][2] * G0;
    const double r = 1.0 / jxw;
    // G_k[aa] = sum_m inv[m][aa] dphi_k[m]  (elements.py:130)
    const double inv[3][3] = {{A0 * r, B0 * r, C0 * r}, {D0 * r, E0 * r, F0 * r}, {G0 * r, H0 * r, I0 * r}};
    double scale = jxw;
    if (a.mp.simp) scale *= pow(a.theta[e], a.mp.penalty);
    // physical gradients and grad u = sum_k U_k (x) G_k in the residual kernel's operation order
    // (qp_geometry, k_residual): R and K see the same grad u to the last bit, which matters at
    // knife edges such as the J2 yield test f == 0 (reference tests/test_materials.py:199-210)
    double G[8][3];
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double d0 = sdN[q * 25 + k * 3], d1 = sdN[q * 25 + k * 3 + 1], d2 = sdN[q * 25 + k * 3 + 2];
#pragma unroll
      for (int aa = 0; aa < 3; ++aa) G[k][aa] = inv[0][aa] * d0 + inv[1][aa] * d1 + inv[2][aa] * d2;
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) gu[v][d] = fma(sXUw[c][k][3 + v], G[k][d], gu[v][d]);
    }
    double gs = 0.0;
#pragma unroll
    for (int v = 0; v < VEC; ++v)
#pragma unroll
      for (int d = 0; d < 3; ++d) gs += fabs(gu[v][d]);
    bool vfin = isfinite(gs), fin = true, bad_def = false;
    double detF = 1.0;
    double cf[4] = {0.0, 0.0, 0.0, 0.0};
    double M1[3][3], M2[3][3];  // NH: F, H; J2: s (deviator)
    if (MAT == B200FEM_MAT_POISSON) {
      cf[0] = a.mp.alpha * scale;
    } else if (MAT == B200FEM_MAT_LE) {
      cf[0] = a.mp.mu * scale;
      cf[1] = a.mp.lam * scale;
    } else if (MAT == B200FEM_MAT_NH) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) M1[i][j] = gu[i][j] + (i == j ? 1.0 : 0.0);
      const double J = det3(M1);
      detF = J;
      if (!(J <= 0.0)) {
        inv_transpose(M1, J, M2);
      } else {
        bad_def = true;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) M2[i][j] = 0.0;
      }
      double I1 = 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) I1 += M1[i][j] * M1[i][j];
      vfin = vfin && isfinite(J) && isfinite(I1);
      const double rc = bad_def ? 0.0 : rcbrt(J);
      const double Ga = a.mp.mu * (rc * rc);  // G J^{-2/3}
      cf[0] = Ga * scale;
      cf[1] = (2.0 / 3.0) * Ga * scale;
      cf[2] = ((2.0 / 9.0) * Ga * I1 + a.mp.kappa * J * (2.0 * J - 1.0)) * scale;
      cf[3] = ((1.0 / 3.0) * Ga * I1 - a.mp.kappa * J * (J - 1.0)) * scale;
      fin = isfinite(cf[0]) && isfinite(cf[1]) && isfinite(cf[2]) && isfinite(cf[3]);
    } else {  // J2 consistent tangent (derivative of j2_return_map incl. the s = 0 guard)
      const double *ep = a.eps_prev + (e * 8 + q) * 9;
      const double *sp = a.sig_prev + (e * 8 + q) * 9;
      double st[3][3], seff;
      bool pos;
      j2_trial(gu, ep, sp, a.mp, st, M1, seff, pos);
      const double over = fmax(seff - a.mp.sy, 0.0);
      const double f = over / seff;
      const double active = (seff - a.mp.sy > 0.0) ? 1.0 : 0.0;  // ramp'(0) = 0
      const double gam = pos ? (active / seff - over / (seff * seff)) * 3.0 * a.mp.mu / seff : 0.0;
      const double beta = 2.0 * a.mp.mu * f;
      cf[0] = (a.mp.mu - 0.5 * beta) * scale;
      cf[1] = (a.mp.lam + beta / 3.0) * scale;
      cf[2] = -gam * scale;
      fin = isfinite(cf[0]) && isfinite(cf[1]) && isfinite(cf[2]);
      vfin = vfin && isfinite(seff) && isfinite(st[0][0] + st[1][1] + st[2][2]);
    }
    if (valid) {
      const unsigned long long key = (unsigned long long)e * 8 + q;
      if (bad_def) {
        atomicMin(&a.derr->inv_def, key);
        atomicMin(&a.derr->min_detF, ord_bits(detF));
      } else if (!vfin) {
        atomicMin(&a.derr->nonfin_v, key);
      } else if (!fin) {
        atomicMin(&a.derr->nonfin_d, key);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) Cf[c * 40 + q * 5 + j] = cf[j];
    double *Vq = V + c * CS + q * QS;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double g[3] = {G[k][0], G[k][1], G[k][2]};
#pragma unroll
      for (int d = 0; d < 3; ++d) Vq[k * NV + d] = g[d];
      if (MAT == B200FEM_MAT_NH) {  // h = H g (slot 3), w = c3 h - c2 F g (slot 6)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double h = M2[i][0] * g[0] + M2[i][1] * g[1] + M2[i][2] * g[2];
          const double u = M1[i][0] * g[0] + M1[i][1] * g[1] + M1[i][2] * g[2];
          Vq[k * NV + 3 + i] = h;
          Vq[k * NV + 6 + i] = cf[2] * h - cf[1] * u;
        }
      } else if (MAT == B200FEM_MAT_J2) {  // y = s g (slot 3)
#pragma unroll
        for (int i = 0; i < 3; ++i) Vq[k * NV + 3 + i] = M1[i][0] * g[0] + M1[i][1] * g[1] + M1[i][2] * g[2];
      }
    }
  }
  __syncwarp();
  // ---- 2. lane (c, a): pairs (a, a + d mod 8)
#pragma unroll
  for (int d = 0; d < NB; ++d)
#pragma unroll
    for (int t = 0; t < BB; ++t) K[d][t] = 0.0;
  const int ia = a8;
#pragma unroll 1
  for (int q = 0; q < 8; ++q) {
    const double *Vq = V + c * CS + q * QS;
    const double c1 = Cf[c * 40 + q * 5], c2 = Cf[c * 40 + q * 5 + 1], c3 = Cf[c * 40 + q * 5 + 2],
                 c4 = Cf[c * 40 + q * 5 + 3];
    double va[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) va[j] = Vq[ia * NV + j];
    // a-side operands (registers): NH: h_a, -c2 u_a, c4 h_a;  J2: cl g_a, c1 g_a, c3 y_a
    double A1[3], A2[3], A3[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (MAT == B200FEM_MAT_NH) {
        A1[i] = va[3 + i];
        A2[i] = fma(-c3, va[3 + i], va[6 + i]);  // w_a - c3 h_a = -c2 u_a
        A3[i] = c4 * va[3 + i];
      } else {
        A1[i] = c2 * va[i];  // cl g_a (c2 slot holds cl for LE / J2)
        A2[i] = c1 * va[i];
        A3[i] = (MAT == B200FEM_MAT_J2) ? c3 * va[3 + i] : 0.0;
      }
    }
#pragma unroll
    for (int d = 0; d < NB; ++d) {
      if (d == 4 && ia >= 4) break;
      const int b = (ia + d) & 7;
      double vb[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) vb[j] = (d == 0) ? va[j] : Vq[b * NV + j];
      const double gg = va[0] * vb[0] + va[1] * vb[1] + va[2] * vb[2];
      if (MAT == B200FEM_MAT_POISSON) {
        K[d][0] = fma(c1, gg, K[d][0]);
      } else {
        const double dg = c1 * gg;
#pragma unroll
        for (int i = 0; i < 3; ++i) K[d][i * 3 + i] += dg;
        // the self block (d = 0) is symmetric: its upper triangle only, mirrored after the loop
        if (MAT == B200FEM_MAT_NH) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k)
              if (d > 0 || k >= i)
                K[d][i * 3 + k] = fma(A1[i], vb[6 + k], fma(A2[i], vb[3 + k], fma(A3[k], vb[3 + i], K[d][i * 3 + k])));
        } else {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              if (d == 0 && k < i) continue;
              double t = fma(A1[i], vb[k], fma(A2[k], vb[i], K[d][i * 3 + k]));
              if (MAT == B200FEM_MAT_J2) t = fma(A3[i], vb[3 + k], t);
              K[d][i * 3 + k] = t;
            }
        }
      }
    }
  }
  if (VEC == 3) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < i; ++k) K[0][i * 3 + k] = K[0][k * 3 + i];
  }
}

// PF (default; B200FEM_JAC_NO_PF=1 is the A/B): each lane's node of the next batch (id, X, U)
// is loaded into registers while the current batch computes, and staged into shared memory at
// the top of the next iteration -- the batch-start gather latency off the critical path
// (config 3: 6.76 -> 6.59 ms per NH tangent, bit-identical; profiles/r02_jacpf_ab.jsonl).
template <int MAT, bool PF = false>
__global__ void __launch_bounds__(kJac2Warps * 32, 2) k_jacobian_v2(ElemArgs a, int64_t n, double *__restrict__ Ke,
                                                                    int soa) {
  using CF = Jac2Cfg<MAT>;
  constexpr int VEC = CF::VEC, CS = CF::CS;
  constexpr int NB = 5, BB = VEC * VEC;
  extern __shared__ double jac2_sm[];
  double *sdN = jac2_sm;                                                     // [q][k*3 + d], point stride 25
  double(*sXU)[4][8][7] = reinterpret_cast<double(*)[4][8][7]>(jac2_sm + CF::SM_DN);  // [w][c][k][X, U]
  for (int t = threadIdx.x; t < 192; t += blockDim.x) sdN[(t / 24) * 25 + t % 24] = (&c_dN[0][0][0])[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, c = lane >> 3;
  double *V = jac2_sm + CF::SM_DN + CF::SM_XU + w * CF::VW;                  // [c][q][a][NV]
  double *Cf = jac2_sm + CF::SM_DN + CF::SM_XU + CF::SM_V + w * 160;         // [c][q][4], point stride 5
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double px[3] = {0.0, 0.0, 0.0}, pu[3] = {0.0, 0.0, 0.0};
  auto load_node = [&](int64_t b) {  // this lane's node of the batch at b (clamped like e below)
    const int64_t e2 = (b + c < n) ? b + c : n - 1;
    const int node = a.cells[e2 * 8 + (lane & 7)];
#pragma unroll
    for (int d = 0; d < 3; ++d) px[d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
    for (int v = 0; v < VEC; ++v) pu[v] = a.U[(int64_t)node * VEC + v];
  };
  if (PF && warp0 * 4 < n) load_node(warp0 * 4);
  for (int64_t base = warp0 * 4; base < n; base += nwarps * 4) {
    const bool valid = base + c < n;
    const int64_t e = valid ? base + c : n - 1;
    double K[NB][BB];
    if (PF) {
#pragma unroll
      for (int d = 0; d < 3; ++d) sXU[w][c][lane & 7][d] = px[d];
#pragma unroll
      for (int v = 0; v < VEC; ++v) sXU[w][c][lane & 7][3 + v] = pu[v];
      if (base + nwarps * 4 < n) load_node(base + nwarps * 4);
      __syncwarp();
    }
    jac2_cell_blocks<MAT, PF>(a, e, valid, lane, sdN, sXU[w], V, Cf, K);
    const int ia = lane & 7;
    if (soa) {
      // element-major scratch [pair][VV][cell] for the lattice pull: stage the warp's 4 cells
      // in shared memory (the V region is free once the pair loop is done), then write every
      // (pair, entry) as the 4 consecutive cells -- full 32-byte sectors instead of the partial
      // sectors of per-lane 8-byte stores, and coalesced reads for the pull's thread per node
      __syncwarp();
      double *stg = V;  // 36 * BB * 4 doubles <= 4 * CS
#pragma unroll
      for (int d = 0; d < NB; ++d) {
        if (d == 4 && ia >= 4) break;
        const int b = (ia + d) & 7;
        const int lo = ia < b ? ia : b, hi = ia < b ? b : ia;
        const int p = lo * (15 - lo) / 2 + hi;
#pragma unroll
        for (int i = 0; i < VEC; ++i)
#pragma unroll
          for (int k = 0; k < VEC; ++k)
            stg[((p * BB) + i * VEC + k) * 4 + c] = (ia <= b) ? K[d][i * VEC + k] : K[d][k * VEC + i];
      }
      __syncwarp();
      for (int t = lane; t < 36 * BB * 4; t += 32) {
        const int pe = t >> 2, cc = t & 3;
        if (base + cc < n) Ke[(int64_t)pe * n + base + cc] = stg[t];
      }
    } else if (valid) {
#pragma unroll
      for (int d = 0; d < NB; ++d) {
        if (d == 4 && ia >= 4) break;
        const int b = (ia + d) & 7;
        const int lo = ia < b ? ia : b, hi = ia < b ? b : ia;
        const int p = lo * (15 - lo) / 2 + hi;  // upper-triangle index of (lo, hi)
        double Kt[VEC][VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i)
#pragma unroll
          for (int k = 0; k < VEC; ++k) Kt[i][k] = (ia <= b) ? K[d][i * VEC + k] : K[d][k * VEC + i];
        jac_store<VEC>(Ke, e, n, p, soa, Kt);
      }
    }
    __syncwarp();
  }
}

// Warp per node: the node's VEC rows (contiguous in the CSR values) are accumulated in
// shared memory from its incident cells in ascending cell id -- every CSR slot sums its
// contributions in the reference's order (assembly.py:296, kernels.py:30-34) -- then
// Dirichlet rows become identity rows (assembly.py:297-299) and the block is written once.
template <int VEC>
__global__ void __launch_bounds__(kThreads) k_jacobian_gather(
    const int32_t *__restrict__ n2c_ptr, const int32_t *__restrict__ n2c, const uint8_t *__restrict__ n2c_a,
    const uint8_t *__restrict__ cpos, const int32_t *__restrict__ nbr_ptr, const int32_t *__restrict__ nbr,
    const double *__restrict__ Ke, const uint8_t *__restrict__ dir_flag, int64_t n_nodes, int max_nbr,
    double *__restrict__ data, const int32_t *__restrict__ up_ptr, double *__restrict__ sym,
    double *__restrict__ grid = nullptr, int gnx = 0, int gny = 0, int64_t gnpad = 0) {
  extern __shared__ double gsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double *acc = gsm + (size_t)w * VEC * VEC * max_nbr;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t n = warp0; n < n_nodes; n += nwarps) {
    const int p0 = __ldg(nbr_ptr + n), cnt = __ldg(nbr_ptr + n + 1) - p0;
    const int L = VEC * cnt, T = VEC * L;
    for (int t = lane; t < T; t += 32) acc[t] = 0.0;
    __syncwarp();
    int self = 0;
    if (dir_flag || sym || grid) {
      int hi = cnt;  // position of n in its own neighbour list
      while (self < hi) {
        const int mid = (self + hi) >> 1;
        if (__ldg(nbr + p0 + mid) < (int)n) self = mid + 1; else hi = mid;
      }
    }
    // GRID-only assembly (the Newton operator): only the upper blocks (neighbour >= n) are
    // stored, so the lower half of the gather -- half the scratch reads -- is skipped.
    const int min_pos = (grid && !sym && !data) ? self : 0;
    const int k0 = __ldg(n2c_ptr + n), deg = __ldg(n2c_ptr + n + 1) - k0;
    constexpr int ITEMS = 8 * VEC * VEC, PER = (ITEMS + 31) / 32;
    for (int kc = 0; kc < deg; ++kc) {
      const int64_t e = __ldg(n2c + k0 + kc);
      const int a = __ldg(n2c_a + k0 + kc);
      double v[PER];
      int pos[PER];
#pragma unroll
      for (int r = 0; r < PER; ++r) {  // the cell's loads are issued together
        const int it = lane + 32 * r;
        const int b = it / (VEC * VEC), rr = it - b * VEC * VEC, i = rr / VEC, kk = rr - i * VEC;
        const int cp = it < ITEMS ? __ldg(cpos + e * 64 + a * 8 + b) : -1;
        const bool ok = it < ITEMS && cp >= min_pos;
        const int pa = a <= b ? a : b, pb = a <= b ? b : a;
        const int off = a <= b ? i * VEC + kk : kk * VEC + i;
        v[r] = ok ? __ldg(Ke + (e * 36 + c_pair_idx[pa][pb]) * (VEC * VEC) + off) : 0.0;
        pos[r] = ok ? i * L + VEC * cp + kk : -1;
      }
#pragma unroll
      for (int r = 0; r < PER; ++r)
        if (pos[r] >= 0) acc[pos[r]] += v[r];
      __syncwarp();  // ascending cell order per slot
    }
    if (sym) {  // upper node blocks (m >= n), pre-Dirichlet, 3x3 row-major: the SYM3 operator
      double *o = sym + (int64_t)VEC * VEC * __ldg(up_ptr + n);
      const int nu = cnt - self;
      for (int t = lane; t < nu * VEC * VEC; t += 32) {
        const int jb = t / (VEC * VEC), rr = t - jb * VEC * VEC, i = rr / VEC, kk = rr - i * VEC;
        o[t] = acc[i * L + VEC * (self + jb) + kk];
      }
      __syncwarp();
    }
    if (grid) {  // GRID3: upper blocks in the tiled element layout (pre-Dirichlet)
      const int gnxy = gnx * gny;
      const int ni = (int)(n % gnx), nj = (int)((n / gnx) % gny), nk = (int)(n / gnxy);
      const int nu = cnt - self;
      constexpr int VV = VEC * VEC;
      for (int t = lane; t < nu * VV; t += 32) {
        const int jb = t / VV, rr = t - jb * VV, i = rr / VEC, kk = rr - i * VEC;
        const int m = __ldg(nbr + p0 + self + jb);
        const int kx = grid_index(m % gnx - ni, (m / gnx) % gny - nj, m / gnxy - nk);
        grid[grid_idx(kx, rr, n, gnpad, VV)] = acc[i * L + VEC * (self + jb) + kk];
      }
      __syncwarp();
    }
    if (!data) continue;
    if (dir_flag) {
      for (int i = 0; i < VEC; ++i) {
        if (!__ldg(dir_flag + n * VEC + i)) continue;
        for (int t = lane; t < L; t += 32) acc[i * L + t] = (t == VEC * self + i) ? 1.0 : 0.0;
      }
      __syncwarp();
    }
    double *out = data + (int64_t)VEC * VEC * p0;
    for (int t = lane; t < T; t += 32) out[t] = acc[t];
    __syncwarp();
  }
}

__global__ void k_jac_dirichlet(double *__restrict__ data, const int32_t *__restrict__ indptr,
                                const int32_t *__restrict__ diag, const int32_t *__restrict__ dofs, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int d = dofs[i];
    for (int k = indptr[d] + lane; k < indptr[d + 1]; k += 32) data[k] = 0.0;
    __syncwarp();
    if (lane == 0) data[diag[d]] = 1.0;
    __syncwarp();
  }
}

// ---------------------------------------------------------- qp flux / commit
// thread per (cell, qp); MODE 0: write flux, 1: J2 commit, 2: volume-average partials
template <int MAT, int MODE>
__global__ void __launch_bounds__(kThreads) k_qp(ElemArgs a, int64_t n_cells, double *out, double *eps_out,
                                                 double *sig_out, RedScratch red) {
  constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  double acc[10];
#pragma unroll
  for (int j = 0; j < 10; ++j) acc[j] = 0.0;
  const int64_t total = n_cells * 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t e = t >> 3;
    const int q = t & 7;
    double X[8][3], Uk[8][VEC];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int node = a.cells[e * 8 + k];
#pragma unroll
      for (int d = 0; d < 3; ++d) X[k][d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
      for (int v = 0; v < VEC; ++v) Uk[k][v] = a.U[(int64_t)node * VEC + v];
    }
    double G[8][3];
    const double jxw = qp_geometry(X, q, G);
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) gu[v][d] = fma(Uk[k][v], G[k][d], gu[v][d]);
    const double *ep = nullptr, *sp = nullptr;
    if (MAT == B200FEM_MAT_J2) {
      ep = a.eps_prev + t * 9;
      sp = a.sig_prev + t * 9;
    }
    double P[3][3], detF = 1.0;
    const bool ok = flux_at<MAT>(gu, a.mp, ep, sp, P, detF);
    if (!ok) {
      atomicMin(&a.derr->inv_def, (unsigned long long)t);
      atomicMin(&a.derr->min_detF, ord_bits(detF));
    }
    double sc = 1.0;
    if (a.mp.simp) sc = pow(a.theta[e], a.mp.penalty);
    if (MODE == 0) {
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) out[t * VEC * 3 + v * 3 + d] = P[v][d] * sc;
    } else if (MODE == 1) {
      double e9[9], s9[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          e9[i * 3 + j] = 0.5 * (gu[i][j] + gu[j][i]);
          s9[i * 3 + j] = P[i][j];
        }
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        eps_out[t * 9 + j] = e9[j];
        sig_out[t * 9 + j] = s9[j];
      }
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) acc[v * 3 + d] += P[v][d] * sc * jxw;
      acc[9] += jxw;
    }
  }
  if (MODE == 2) {
    double tot[10];
    block_partials_and_finish<10>(acc, red, tot);
  }
}

// ------------------------------------------------- geometry (Workspace fields)
// thread per (cell, qp): phys_grads[e][q][k][:] = J^-T dphi_k, JxW[e][q] = det J (weights 1;
// elements.py:80-131).  Host views only (the kernels recompute geometry per cell).
__global__ void __launch_bounds__(kThreads) k_geometry(const double *__restrict__ coords,
                                                        const int32_t *__restrict__ cells, int64_t n_cells,
                                                        double *__restrict__ pg, double *__restrict__ jxw) {
  const int64_t total = n_cells * 8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t >> 3;
    const int q = t & 7;
    double X[8][3];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int d = 0; d < 3; ++d) X[k][d] = coords[(int64_t)cells[e * 8 + k] * 3 + d];
    double G[8][3];
    const double det = qp_geometry(X, q, G);
    if (jxw) jxw[t] = det;
    if (pg) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) pg[(t * 8 + k) * 3 + d] = G[k][d];
    }
  }
}

// ---------------------------------------------------------- geometry check
__global__ void k_geom_check(const double *__restrict__ coords, const int32_t *__restrict__ cells, int64_t n_cells,
                             DevErr *derr) {
  const int64_t total = n_cells * 8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t >> 3;
    const int q = t & 7;
    double X[8][3];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int node = cells[e * 8 + k];
#pragma unroll
      for (int d = 0; d < 3; ++d) X[k][d] = coords[(int64_t)node * 3 + d];
    }
    double G[8][3];
    const double det = qp_geometry(X, q, G);
    if (!(det > 0.0)) atomicMin(&derr->inv_elem, (unsigned long long)t);
  }
}

// ------------------------------------------------------------ launchers
static int grid_cap(int64_t work_items, int per_block) {
  int64_t g = (work_items + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

static ElemArgs make_args(Ctx *c, const double *U) {
  ElemArgs a;
  a.coords = c->coords;
  a.cells = c->cells;
  a.U = U;
  a.theta = c->theta;
  a.eps_prev = c->eps_prev;
  a.sig_prev = c->sig_prev;
  a.mp = c->mp;
  a.derr = c->derr;
  return a;
}

int check_geometry(Ctx *c, b200fem_error *err) {
  k_geom_check<<<grid_cap(c->n_cells * 8, kThreads), kThreads, 0, c->stream>>>(c->coords, c->cells, c->n_cells,
                                                                              c->derr);
  count_launch();
  DevErr h;
  B200_CUDA_E(cudaMemcpyAsync(&h, c->derr, sizeof(DevErr), cudaMemcpyDeviceToHost, c->stream), err);
  B200_CUDA_E(cudaStreamSynchronize(c->stream), err);
  if (h.inv_elem != ~0ull) {
    if (err) {
      err->code = B200FEM_E_INVERTED_ELEMENT;
      err->cell = (int64_t)(h.inv_elem >> 3);
      err->qp = (int)(h.inv_elem & 7);
    }
    return B200FEM_E_INVERTED_ELEMENT;
  }
  return 0;
}

int fetch_element_errors(Ctx *c, b200fem_error *err, bool jacobian) {
  DevErr h;
  B200_CUDA_E(cudaMemcpyAsync(&h, c->derr, sizeof(DevErr), cudaMemcpyDeviceToHost, c->stream), err);
  B200_CUDA_E(cudaStreamSynchronize(c->stream), err);
  const unsigned long long none = ~0ull;
  if (h.inv_def == none && h.nonfin_v == none && h.nonfin_d == none) return 0;
  B200_CUDA_E(cudaMemsetAsync(c->derr, 0xff, sizeof(DevErr), c->stream), err);
  // earliest offending cell wins (the reference raises in the first failing chunk);
  // det F <= 0 is checked before finiteness on a tie (assembly.py:185-188)
  unsigned long long kd = h.inv_def, kv = h.nonfin_v, kg = h.nonfin_d;
  int code;
  unsigned long long key;
  if (kd != none && (kd >> 3) <= (std::min(kv, kg) >> 3)) {
    code = B200FEM_E_INVERTED_DEFORMATION;
    key = kd;
  } else if (kv <= kg) {
    code = B200FEM_E_NONFINITE_VALUE;
    key = kv;
  } else {
    code = B200FEM_E_NONFINITE_DERIV;
    key = kg;
  }
  if (err) {
    err->code = code;
    err->cell = (int64_t)(key >> 3);
    err->qp = (int)(key & 7);
    if (code == B200FEM_E_INVERTED_DEFORMATION) {
      err->value = unord_bits(h.min_detF);
      snprintf(err->msg, sizeof(err->msg),
               "det(F) <= 0 (min %.3e): element inverted beyond the neo-Hookean domain [element %lld, quad point %d]",
               err->value, (long long)err->cell, err->qp);
    } else if (code == B200FEM_E_NONFINITE_VALUE) {
      snprintf(err->msg, sizeof(err->msg), "non-finite value in flux kernel [element %lld, quad point %d]",
               (long long)err->cell, err->qp);
    } else {
      snprintf(err->msg, sizeof(err->msg), "non-finite derivative in flux kernel [element %lld]",
               (long long)err->cell);
    }
  }
  (void)jacobian;
  return code;
}

static int ensure_scratch(Ctx *c, size_t len, b200fem_error *err) {
  if (c->scratch_len >= len) return 0;
  cudaStreamSynchronize(c->stream);
  cudaFree(c->scratch);
  c->scratch = nullptr;
  c->scratch_len = 0;
  B200_CUDA_E(dalloc(&c->scratch, len), err);
  c->scratch_len = len;
  return 0;
}

// Two-phase residual: (1) per-cell blocks R_e (one launch over all cells), (2) ordered
// per-node gather fused with the load subtraction; Dirichlet rows overwritten last.
int launch_residual(Ctx *c, const double *U, double *R, double bc_scale, int apply_dirichlet, b200fem_error *err,
                    double *norm_host) {
  cudaStream_t s = c->stream;
  if (ensure_scratch(c, (size_t)c->n_cells * 8 * c->vec, err)) return B200FEM_E_CUDA;
  const ElemArgs a = make_args(c, U);
  const int g = grid_cap(c->n_cells, kWarps * 4);
  switch (c->material) {
    case B200FEM_MAT_POISSON: k_residual<B200FEM_MAT_POISSON><<<g, kThreads, 0, s>>>(a, c->n_cells, c->scratch); break;
    case B200FEM_MAT_LE: k_residual<B200FEM_MAT_LE><<<g, kThreads, 0, s>>>(a, c->n_cells, c->scratch); break;
    case B200FEM_MAT_NH: k_residual<B200FEM_MAT_NH><<<g, kThreads, 0, s>>>(a, c->n_cells, c->scratch); break;
    default: k_residual<B200FEM_MAT_J2><<<g, kThreads, 0, s>>>(a, c->n_cells, c->scratch); break;
  }
  const int gg = grid_cap(c->n_dofs, kThreads);
  if (c->vec == 3)
    k_residual_gather<3><<<gg, kThreads, 0, s>>>(c->n2c_ptr, c->n2c, c->n2c_a, c->scratch, c->n_nodes, bc_scale,
                                                 c->f_neumann, c->f_body, R);
  else
    k_residual_gather<1><<<gg, kThreads, 0, s>>>(c->n2c_ptr, c->n2c, c->n2c_a, c->scratch, c->n_nodes, bc_scale,
                                                 c->f_neumann, c->f_body, R);
  count_launch(2);
  if (apply_dirichlet && c->n_dir) {
    k_res_dirichlet<<<grid_cap(c->n_dir, kThreads), kThreads, 0, s>>>(R, U, c->dir_dofs, c->dir_vals, c->n_dir,
                                                                      bc_scale);
    count_launch();
  }
  B200_CUDA_E(cudaGetLastError(), err);
  if (norm_host) {
    if (launch_dot(R, R, c->n_dofs, &c->red, s)) return B200FEM_E_CUDA;
    B200_CUDA_E(cudaMemcpyAsync(c->pinned, c->red.result, sizeof(double), cudaMemcpyDeviceToHost, s), err);
  }
  int st = fetch_element_errors(c, err, false);  // synchronises the stream
  if (st) return st;
  if (norm_host) *norm_host = std::sqrt(c->pinned[0]);
  return 0;
}

// Design VJP (assembly.py:303-341): SIMP -> one value per cell; design source -> per-cell
// local-node values gathered per node in ascending cell order.
int launch_param_vjp(Ctx *c, const double *U, const double *theta, const double *w, double *out,
                     b200fem_error *err) {
  cudaStream_t s = c->stream;
  const ElemArgs a = make_args(c, U);
  const int g = grid_cap(c->n_cells, kWarps * 4);
  if (c->flags & B200FEM_FLAG_SIMP) {
    if (c->vec != 3 || !U) return B200FEM_E_INVALID;
    switch (c->material) {
      case B200FEM_MAT_LE: k_vjp_simp<B200FEM_MAT_LE><<<g, kThreads, 0, s>>>(a, c->n_cells, theta, w, c->dir_flag, out); break;
      case B200FEM_MAT_NH: k_vjp_simp<B200FEM_MAT_NH><<<g, kThreads, 0, s>>>(a, c->n_cells, theta, w, c->dir_flag, out); break;
      default: return B200FEM_E_UNSUPPORTED;
    }
    count_launch();
  } else if (c->flags & B200FEM_FLAG_DESIGN_SOURCE) {
    if (c->vec != 1) return B200FEM_E_INVALID;
    if (ensure_scratch(c, (size_t)c->n_cells * 8, err)) return B200FEM_E_CUDA;
    k_vjp_source<<<g, kThreads, 0, s>>>(a, c->n_cells, w, c->dir_flag, c->scratch);
    k_residual_gather<1><<<grid_cap(c->n_nodes, kThreads), kThreads, 0, s>>>(c->n2c_ptr, c->n2c, c->n2c_a, c->scratch,
                                                                            c->n_nodes, 0.0, nullptr, nullptr, out);
    count_launch(2);
  } else {
    return B200FEM_E_INVALID;
  }
  B200_CUDA_E(cudaGetLastError(), err);
  return fetch_element_errors(c, err, false);  // synchronises the stream
}

// GRID path, lattice pull (box meshes only): thread per node; for every upper lattice offset k
// the 1, 2, 4 or 8 cells shared by node n and n + off_k are known from the lattice, and the
// block is summed from the element-major scratch in ascending cell id -- the same order (and
// the same values) as the per-node gather, without its shared-memory accumulator: every load
// is independent (high memory-level parallelism) and coalesced across consecutive nodes.
__device__ __forceinline__ int vtk_local(int lx, int ly, int lz) {  // HEX8 vertex order, mesh.py:159-167
  return lz * 4 + (ly ? (lx ? 2 : 3) : (lx ? 1 : 0));
}

template <int VEC, bool SOA>
__global__ void __launch_bounds__(kThreads) k_grid_pull(const double *__restrict__ Ke, int64_t n_cells, int NX,
                                                        int NY, int NZ, int64_t gnpad, double *__restrict__ grid) {
  constexpr int VV = VEC * VEC;
  const int64_t nn = (int64_t)NX * NY * NZ;
  const int cx_n = NX - 1, cy_n = NY - 1, cz_n = NZ - 1;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn; n += (int64_t)gridDim.x * blockDim.x) {
    const int kz = (int)(n / ((int64_t)NX * NY)), rem = (int)(n - (int64_t)kz * NX * NY), jy = rem / NX,
              ix = rem - jy * NX;
#pragma unroll 1
    for (int q = 0; q < 14; ++q) {
      const int di = grid_di(q), dj = grid_dj(q), dk = grid_dk(q);
      if ((unsigned)(ix + di) >= (unsigned)NX || (unsigned)(jy + dj) >= (unsigned)NY || (unsigned)(kz + dk) >= (unsigned)NZ)
        continue;  // no such neighbour: the SpMV masks this offset
      double acc[VV];
#pragma unroll
      for (int t = 0; t < VV; ++t) acc[t] = 0.0;
      // corner of a shared cell along an axis: offset 0 -> {x-1, x}; +1 -> x; -1 -> x-1
#pragma unroll
      for (int oz = 0; oz < 2; ++oz) {
        const int cz = (dk == 0) ? kz - 1 + oz : (dk > 0 ? kz : kz - 1);
        if ((dk != 0 && oz) || (unsigned)cz >= (unsigned)cz_n) continue;
#pragma unroll
        for (int oy = 0; oy < 2; ++oy) {
          const int cy = (dj == 0) ? jy - 1 + oy : (dj > 0 ? jy : jy - 1);
          if ((dj != 0 && oy) || (unsigned)cy >= (unsigned)cy_n) continue;
#pragma unroll
          for (int ox = 0; ox < 2; ++ox) {
            const int cx = (di == 0) ? ix - 1 + ox : (di > 0 ? ix : ix - 1);
            if ((di != 0 && ox) || (unsigned)cx >= (unsigned)cx_n) continue;
            const int64_t cell = cx + (int64_t)cx_n * (cy + (int64_t)cy_n * cz);
            const int a = vtk_local(ix - cx, jy - cy, kz - cz);
            const int b = vtk_local(ix + di - cx, jy + dj - cy, kz + dk - cz);
            const int pa = a <= b ? a : b, pb = a <= b ? b : a;
            const int pr = c_pair_idx[pa][pb];
            const double *src = SOA ? Ke + (int64_t)pr * VV * n_cells + cell : Ke + (cell * 36 + pr) * VV;
#pragma unroll
            for (int t = 0; t < VV; ++t) {
              const int i = t / VEC, k = t - i * VEC;
              const int off = a <= b ? t : k * VEC + i;  // block (b, a) is the transpose
              acc[t] += __ldg(src + (SOA ? (int64_t)off * n_cells : off));
            }
          }
        }
      }
#pragma unroll
      for (int t = 0; t < VV; ++t) grid[grid_idx(q, t, n, gnpad, VV)] = acc[t];
    }
  }
}

// The same lattice pull into the reference CSR layout (assemble_jacobian on box meshes): node
// n's VEC rows hold its 27 (or fewer, at the boundary) neighbour blocks in ascending node id,
// i.e. lexicographic (dk, dj, di); Dirichlet rows become identity rows (assembly.py:297-299).
// Same per-slot order (ascending cell id) and values as the per-node gather.
template <int VEC, bool SOA>
__global__ void __launch_bounds__(kThreads) k_csr_pull(const double *__restrict__ Ke, int64_t n_cells, int NX,
                                                       int NY, int NZ, const int32_t *__restrict__ nbr_ptr,
                                                       const uint8_t *__restrict__ dir_flag, double *__restrict__ data) {
  constexpr int VV = VEC * VEC;
  const int64_t nn = (int64_t)NX * NY * NZ;
  const int cx_n = NX - 1, cy_n = NY - 1, cz_n = NZ - 1;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn; n += (int64_t)gridDim.x * blockDim.x) {
    const int kz = (int)(n / ((int64_t)NX * NY)), rem = (int)(n - (int64_t)kz * NX * NY), jy = rem / NX,
              ix = rem - jy * NX;
    const int64_t p0 = __ldg(nbr_ptr + n);
    const int cnt = __ldg(nbr_ptr + n + 1) - (int)p0, L = VEC * cnt;
    double *rows = data + (int64_t)VV * p0;  // row c of the node at rows + c * L
    bool dflag[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) dflag[c] = dir_flag && __ldg(dir_flag + n * VEC + c);
    int j = 0;
#pragma unroll 1
    for (int o = 0; o < 27; ++o) {
      const int dk = o / 9 - 1, dj = (o / 3) % 3 - 1, di = o % 3 - 1;
      if ((unsigned)(ix + di) >= (unsigned)NX || (unsigned)(jy + dj) >= (unsigned)NY || (unsigned)(kz + dk) >= (unsigned)NZ)
        continue;
      double acc[VV];
#pragma unroll
      for (int t = 0; t < VV; ++t) acc[t] = 0.0;
#pragma unroll
      for (int oz = 0; oz < 2; ++oz) {
        const int cz = (dk == 0) ? kz - 1 + oz : (dk > 0 ? kz : kz - 1);
        if ((dk != 0 && oz) || (unsigned)cz >= (unsigned)cz_n) continue;
#pragma unroll
        for (int oy = 0; oy < 2; ++oy) {
          const int cy = (dj == 0) ? jy - 1 + oy : (dj > 0 ? jy : jy - 1);
          if ((dj != 0 && oy) || (unsigned)cy >= (unsigned)cy_n) continue;
#pragma unroll
          for (int ox = 0; ox < 2; ++ox) {
            const int cx = (di == 0) ? ix - 1 + ox : (di > 0 ? ix : ix - 1);
            if ((di != 0 && ox) || (unsigned)cx >= (unsigned)cx_n) continue;
            const int64_t cell = cx + (int64_t)cx_n * (cy + (int64_t)cy_n * cz);
            const int a = vtk_local(ix - cx, jy - cy, kz - cz);
            const int b = vtk_local(ix + di - cx, jy + dj - cy, kz + dk - cz);
            const int pa = a <= b ? a : b, pb = a <= b ? b : a;
            const int pr = c_pair_idx[pa][pb];
            const double *src = SOA ? Ke + (int64_t)pr * VV * n_cells + cell : Ke + (cell * 36 + pr) * VV;
#pragma unroll
            for (int t = 0; t < VV; ++t) {
              const int i = t / VEC, k = t - i * VEC;
              const int off = a <= b ? t : k * VEC + i;
              acc[t] += __ldg(src + (SOA ? (int64_t)off * n_cells : off));
            }
          }
        }
      }
      const bool self = (o == 13);
#pragma unroll
      for (int c = 0; c < VEC; ++c)
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          rows[c * L + VEC * j + k] = dflag[c] ? ((self && k == c) ? 1.0 : 0.0) : acc[c * VEC + k];
      ++j;
    }
  }
}

template <int MAT>
static void launch_jac2(int g, cudaStream_t s, const ElemArgs &a, int64_t n, double *Ke, int soa) {
  static bool attr = false;  // > 48 KB of shared memory is opt-in per kernel
  if (!attr) {
    cudaFuncSetAttribute(k_jacobian_v2<MAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Jac2Cfg<MAT>::BYTES);
    attr = true;
  }
  static int pf = -1;
  if (pf < 0) pf = getenv("B200FEM_JAC_NO_PF") ? 0 : 1;
  if (pf) {
    static bool attr_pf = false;
    if (!attr_pf) {
      cudaFuncSetAttribute(k_jacobian_v2<MAT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)Jac2Cfg<MAT>::BYTES);
      attr_pf = true;
    }
    k_jacobian_v2<MAT, true><<<g, kJac2Warps * 32, Jac2Cfg<MAT>::BYTES, s>>>(a, n, Ke, soa);
    return;
  }
  k_jacobian_v2<MAT><<<g, kJac2Warps * 32, Jac2Cfg<MAT>::BYTES, s>>>(a, n, Ke, soa);
}

// B200FEM_TANGENT = v2 (default: node-lane phase A) | v1 (the r01 pair-per-lane phase A, kept as
// the A/B reference of tools/tangent_ab.py).  A fused lattice column kernel without the per-cell
// scratch was measured at 16.0 ms against 7.1 ms for v2 + pull (one 200 KB CTA of 4 warps per
// SM: latency bound) and removed (profiles/r02_tangent_ab.jsonl).  Read once per process.
static int tangent_variant() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("B200FEM_TANGENT");
    v = (e && !strcmp(e, "v1")) ? 0 : 1;
  }
  return v;
}

// Two-phase Jacobian: (1) the 36 symmetric 3x3 blocks of every cell's Ke into scratch,
// (2) warp-per-node ordered gather writing each CSR row segment exactly once.
int launch_jacobian(Ctx *c, const double *U, double *data, b200fem_error *err, double *sym, double *grid) {
  cudaStream_t s = c->stream;
  const int vv = c->vec * c->vec;
  // GRID-only tangent on a lattice: element-major scratch + lattice pull instead of the gather
  // (element-major scratch for vec 1; vec 3 keeps the cell-major blocks, whose 72-byte rows the
  // pull reads whole -- element-major stores of a warp-per-cell kernel would be partial sectors)
  const bool pull = grid && !data && !sym && c->grid_nx && !getenv("B200FEM_NO_GRID_PULL");
  if (ensure_scratch(c, (size_t)c->n_cells * 36 * vv, err)) return B200FEM_E_CUDA;
  const ElemArgs a = make_args(c, U);
  // reference CSR layout on a scalar lattice: the same pull (assemble_jacobian, operator="csr").
  // Not for vec 3: a thread's 27 blocks land in 3 rows ~2 KB apart from its neighbours' -- the
  // uncoalesced 8-byte stores made it 21 ms against 13.7 ms for the gather (config 3)
  const bool csr_pull = !grid && data && !sym && c->grid_nx && c->vec == 1 && !getenv("B200FEM_NO_GRID_PULL");
  // element-major scratch for the lattice pulls: vec 1 always; vec 3 when the node-lane phase A
  // writes it (staged, full-sector stores; the pair-per-lane v1 kernel keeps cell-major blocks)
  const int soa = ((pull || csr_pull) && (c->vec == 1 || tangent_variant() != 0)) ? 1 : 0;
  if (tangent_variant() == 0) {  // A/B: the pair-per-lane phase A
    const int g = grid_cap(c->n_cells, kJacWarps);
    switch (c->material) {
      case B200FEM_MAT_POISSON: k_jacobian<B200FEM_MAT_POISSON><<<g, kJacWarps * 32, 0, s>>>(a, c->n_cells, c->scratch, soa); break;
      case B200FEM_MAT_LE: k_jacobian<B200FEM_MAT_LE><<<g, kJacWarps * 32, 0, s>>>(a, c->n_cells, c->scratch, soa); break;
      case B200FEM_MAT_NH: k_jacobian<B200FEM_MAT_NH><<<g, kJacWarps * 32, 0, s>>>(a, c->n_cells, c->scratch, soa); break;
      default: k_jacobian<B200FEM_MAT_J2><<<g, kJacWarps * 32, 0, s>>>(a, c->n_cells, c->scratch, soa); break;
    }
  } else {
    const int g = grid_cap(c->n_cells, kJac2Warps * 4);
    switch (c->material) {
      case B200FEM_MAT_POISSON: launch_jac2<B200FEM_MAT_POISSON>(g, s, a, c->n_cells, c->scratch, soa); break;
      case B200FEM_MAT_LE: launch_jac2<B200FEM_MAT_LE>(g, s, a, c->n_cells, c->scratch, soa); break;
      case B200FEM_MAT_NH: launch_jac2<B200FEM_MAT_NH>(g, s, a, c->n_cells, c->scratch, soa); break;
      default: launch_jac2<B200FEM_MAT_J2>(g, s, a, c->n_cells, c->scratch, soa); break;
    }
  }
  if (pull) {
    const int64_t nn = c->n_nodes;
    const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (nn + kThreads - 1) / kThreads));
    if (c->vec == 3 && soa)
      k_grid_pull<3, true><<<gp, kThreads, 0, s>>>(c->scratch, c->n_cells, c->grid_nx, c->grid_ny, c->grid_nz,
                                                   c->grid_npad, grid);
    else if (c->vec == 3)
      k_grid_pull<3, false><<<gp, kThreads, 0, s>>>(c->scratch, c->n_cells, c->grid_nx, c->grid_ny, c->grid_nz,
                                                    c->grid_npad, grid);
    else
      k_grid_pull<1, true><<<gp, kThreads, 0, s>>>(c->scratch, c->n_cells, c->grid_nx, c->grid_ny, c->grid_nz,
                                                   c->grid_npad, grid);
    count_launch(2);
    B200_CUDA_E(cudaGetLastError(), err);
    return fetch_element_errors(c, err, true);
  }
  if (csr_pull) {
    const int64_t nn = c->n_nodes;
    const int gp = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, (nn + kThreads - 1) / kThreads));
    const uint8_t *df = c->n_dir ? c->dir_flag : nullptr;
    k_csr_pull<1, true><<<gp, kThreads, 0, s>>>(c->scratch, c->n_cells, c->grid_nx, c->grid_ny, c->grid_nz,
                                                c->nbr_ptr, df, data);
    count_launch(2);
    B200_CUDA_E(cudaGetLastError(), err);
    return fetch_element_errors(c, err, true);
  }
  int warps = 8;
  while (warps > 1 && (size_t)warps * vv * c->max_nbr * sizeof(double) > 96 * 1024) warps >>= 1;
  const size_t smem = (size_t)warps * vv * c->max_nbr * sizeof(double);
  const int gg = grid_cap(c->n_nodes, warps);
  if (c->vec == 3) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_jacobian_gather<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_jacobian_gather<3><<<gg, warps * 32, smem, s>>>(c->n2c_ptr, c->n2c, c->n2c_a, c->cpos, c->nbr_ptr, c->nbr,
                                                     c->scratch, c->n_dir ? c->dir_flag : nullptr, c->n_nodes,
                                                     c->max_nbr, data, c->up_ptr, sym, grid, c->grid_nx,
                                                     c->grid_ny, c->grid_npad);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_jacobian_gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_jacobian_gather<1><<<gg, warps * 32, smem, s>>>(c->n2c_ptr, c->n2c, c->n2c_a, c->cpos, c->nbr_ptr, c->nbr,
                                                     c->scratch, c->n_dir ? c->dir_flag : nullptr, c->n_nodes,
                                                     c->max_nbr, data, nullptr, nullptr, grid, c->grid_nx, c->grid_ny,
                                                     c->grid_npad);
  }
  count_launch(2);
  B200_CUDA_E(cudaGetLastError(), err);
  return fetch_element_errors(c, err, true);
}

template <int MODE>
static int qp_dispatch(Ctx *c, const ElemArgs &a, double *out, double *eo, double *so) {
  const int g = grid_cap(c->n_cells * 8, kThreads);
  const int gg = MODE == 2 ? kRedBlocks : g;
  switch (c->material) {
    case B200FEM_MAT_POISSON: k_qp<B200FEM_MAT_POISSON, MODE><<<gg, kThreads, 0, c->stream>>>(a, c->n_cells, out, eo, so, c->red); break;
    case B200FEM_MAT_LE: k_qp<B200FEM_MAT_LE, MODE><<<gg, kThreads, 0, c->stream>>>(a, c->n_cells, out, eo, so, c->red); break;
    case B200FEM_MAT_NH: k_qp<B200FEM_MAT_NH, MODE><<<gg, kThreads, 0, c->stream>>>(a, c->n_cells, out, eo, so, c->red); break;
    default: k_qp<B200FEM_MAT_J2, MODE><<<gg, kThreads, 0, c->stream>>>(a, c->n_cells, out, eo, so, c->red); break;
  }
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int launch_qp_flux(Ctx *c, const double *U, double *out, b200fem_error *err) {
  if (qp_dispatch<0>(c, make_args(c, U), out, nullptr, nullptr)) return B200FEM_E_CUDA;
  return fetch_element_errors(c, err, false);
}

int launch_volume_average(Ctx *c, const double *U, double *out_host, b200fem_error *err) {
  if (qp_dispatch<2>(c, make_args(c, U), nullptr, nullptr, nullptr)) return B200FEM_E_CUDA;
  double h[10];
  B200_CUDA_E(cudaMemcpyAsync(h, c->red.result, 10 * sizeof(double), cudaMemcpyDeviceToHost, c->stream), err);
  int st = fetch_element_errors(c, err, false);
  if (st) return st;
  const int nv = c->vec * 3;
  for (int j = 0; j < nv; ++j) out_host[j] = h[j] / h[9];
  return 0;
}

int launch_commit(Ctx *c, const double *U) {
  if (c->material != B200FEM_MAT_J2) return 0;
  // commit writes in place: each (cell, qp) reads and then overwrites only its own state
  return qp_dispatch<1>(c, make_args(c, U), nullptr, c->eps_prev, c->sig_prev);
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_residual(b200fem_ctx *ctx, const double *U, double bc_scale, int32_t apply_dirichlet, double *R,
                     double *norm_host, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  return launch_residual((Ctx *)ctx, U, R, bc_scale, apply_dirichlet, err, norm_host);
}

int b200fem_jacobian(b200fem_ctx *ctx, const double *U, double *data, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  return launch_jacobian((Ctx *)ctx, U, data, err, nullptr);
}

int b200fem_jacobian_sym(b200fem_ctx *ctx, const double *U, double *data, double *sym, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  Ctx *c = (Ctx *)ctx;
  if (c->vec != 3 || !sym) return B200FEM_E_INVALID;
  return launch_jacobian(c, U, data, err, sym);
}

int b200fem_jacobian_grid(b200fem_ctx *ctx, const double *U, double *data, double *grid, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  Ctx *c = (Ctx *)ctx;
  if (!c || !c->grid_nx || !grid) return B200FEM_E_INVALID;
  return launch_jacobian(c, U, data, err, nullptr, grid);
}

int b200fem_param_vjp(b200fem_ctx *ctx, const double *U, const double *theta, const double *w, double *out,
                      b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (!ctx || !theta || !w || !out) return B200FEM_E_INVALID;
  return launch_param_vjp((Ctx *)ctx, U, theta, w, out, err);
}

int b200fem_l2_field_error(int64_t n_cells, const double *coords, const int32_t *cells, const double *up,
                           const double *ut, double *out_host, void *stream) {
  if (n_cells < 0 || !out_host) return B200FEM_E_INVALID;
  out_host[0] = out_host[1] = 0.0;
  if (n_cells == 0) return 0;
  element_tables_init();
  cudaStream_t s = (cudaStream_t)stream;
  RedScratch red{};
  double *d = nullptr;
  int st = B200FEM_E_CUDA;
  if (!red_alloc(&red) && dalloc(&d, 2) == cudaSuccess) {
    const int g = std::min(kRedBlocks, grid_cap(n_cells, kWarps * 4));
    k_l2_error<<<g, kThreads, 0, s>>>(coords, cells, n_cells, up, ut, red, d);
    count_launch();
    if (cudaMemcpyAsync(out_host, d, 2 * sizeof(double), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
        cudaStreamSynchronize(s) == cudaSuccess)
      st = 0;
  }
  cudaFree(d);
  red_free(&red);
  return st;
}

int b200fem_qp_flux(b200fem_ctx *ctx, const double *U, double *out, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  return launch_qp_flux((Ctx *)ctx, U, out, err);
}

int b200fem_volume_average_flux(b200fem_ctx *ctx, const double *U, double *out_host, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  return launch_volume_average((Ctx *)ctx, U, out_host, err);
}

int b200fem_commit_state(b200fem_ctx *ctx, const double *U) { return launch_commit((Ctx *)ctx, U); }

int b200fem_geometry(b200fem_ctx *ctx, double *phys_grads, double *jxw) {
  Ctx *c = (Ctx *)ctx;
  if (!c) return B200FEM_E_INVALID;
  if (c->n_cells == 0 || (!phys_grads && !jxw)) return 0;
  k_geometry<<<grid_cap(c->n_cells * 8, kThreads), kThreads, 0, c->stream>>>(c->coords, c->cells, c->n_cells,
                                                                            phys_grads, jxw);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

}  // extern "C"
