// Per-cell HEX8 weak-form kernels: geometry, constitutive laws, residual, consistent
// tangent (hand-derived), quadrature-point flux, J2 commit.
//
// Reference being replaced (paths relative to gradfem/):
//   elements.py:17-131   reference element tables, map_elements (recomputed per cell here)
//   materials.py:74-131  linear_elastic_flux, neo_hookean_flux (AD of W), j2_return_map
//   problems.py:166-202  SIMP theta^p scaling;  problems.py:319-324 nodal design source
//   assembly.py:176-300  _element_residual, assemble_residual, assemble_jacobian
//   kernels.py:30-34     sequential scatter_add -> colour-ordered deterministic RMW
//
// Reduction: cells are processed colour by colour (colour classes share no node), so
// every R entry / CSR slot is updated by plain read-modify-write with no atomics and a
// fixed order (colour 0 first) -> results are bit-identical from run to run.

#include <cmath>

#include "internal.cuh"

namespace b200 {

__constant__ double c_dN[8][8][3];  // [q][k][d] dphi_k/dxi_d at Gauss point q (x fastest)
__constant__ double c_N[8][8];      // [q][k]    phi_k at Gauss point q

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

__device__ __forceinline__ double det3(const double (&F)[3][3]) {  // autodiff.py:202-206 expansion
  return F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
         F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
}

// H = F^{-T} = cof(F) / J
__device__ __forceinline__ void inv_transpose(const double (&F)[3][3], double J, double (&H)[3][3]) {
  const double r = 1.0 / J;
  H[0][0] = (F[1][1] * F[2][2] - F[1][2] * F[2][1]) * r;
  H[0][1] = (F[1][2] * F[2][0] - F[1][0] * F[2][2]) * r;
  H[0][2] = (F[1][0] * F[2][1] - F[1][1] * F[2][0]) * r;
  H[1][0] = (F[0][2] * F[2][1] - F[0][1] * F[2][2]) * r;
  H[1][1] = (F[0][0] * F[2][2] - F[0][2] * F[2][0]) * r;
  H[1][2] = (F[0][1] * F[2][0] - F[0][0] * F[2][1]) * r;
  H[2][0] = (F[0][1] * F[1][2] - F[0][2] * F[1][1]) * r;
  H[2][1] = (F[0][2] * F[1][0] - F[0][0] * F[1][2]) * r;
  H[2][2] = (F[0][0] * F[1][1] - F[0][1] * F[1][0]) * r;
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

// J2 trial state (materials.py:104-122): returns sig_trial, deviator s, s_eff (guarded),
// and whether ssq > 0.
__device__ __forceinline__ void j2_trial(const double (&gu)[3][3], const double *ep, const double *sp,
                                         const MatParams &mp, double (&st)[3][3], double (&s)[3][3], double &seff,
                                         bool &pos) {
  double de[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) de[i][j] = 0.5 * (gu[i][j] + gu[j][i]) - ep[i * 3 + j];
  const double tr = de[0][0] + de[1][1] + de[2][2];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) st[i][j] = sp[i * 3 + j] + ((i == j) ? mp.lam * tr : 0.0) + 2.0 * mp.mu * de[i][j];
  const double p = (st[0][0] + st[1][1] + st[2][2]) / 3.0;
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      s[i][j] = st[i][j] - (i == j ? p : 0.0);
      ss += s[i][j] * s[i][j];
    }
  const double ssq = 1.5 * ss;
  pos = ssq > 0.0;
  seff = sqrt(pos ? ssq : 1.0);
}

// flux P (vec x 3) at one quadrature point; returns false on det F <= 0 (NH)
template <int MAT>
__device__ __forceinline__ bool flux_at(const double (&gu)[3][3], const MatParams &mp, const double *ep,
                                        const double *sp, double (&P)[3][3], double &detF) {
  if (MAT == B200FEM_MAT_POISSON) {
#pragma unroll
    for (int d = 0; d < 3; ++d) P[0][d] = mp.alpha * gu[0][d];
    return true;
  } else if (MAT == B200FEM_MAT_LE) {
    const double tr = gu[0][0] + gu[1][1] + gu[2][2];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) P[i][j] = (i == j ? mp.lam * tr : 0.0) + mp.mu * (gu[i][j] + gu[j][i]);
    return true;
  } else if (MAT == B200FEM_MAT_NH) {
    // P = G J^{-2/3} (F - I1/3 H) + kappa (J-1) J H  (tests/test_materials.py:71-77 closed
    // form of the reference's AD of W), rewritten in terms of g = grad u so that no O(1)
    // quantities cancel near F = I:
    //   J - 1 = I1(g) + I2(g) + I3(g),  cof F = I + c,  c = tr(g) I - g^T + cof(g)
    //   F - I1/3 H = [ (Jm1 - e) I + (1 + Jm1) g - (1 + e) c ] / J,  e = (2 tr g + |g|^2)/3
    //   kappa (J-1) J H = kappa Jm1 cof F
    const double trg = gu[0][0] + gu[1][1] + gu[2][2];
    double cg[3][3];  // cofactor matrix of g
    cg[0][0] = gu[1][1] * gu[2][2] - gu[1][2] * gu[2][1];
    cg[0][1] = gu[1][2] * gu[2][0] - gu[1][0] * gu[2][2];
    cg[0][2] = gu[1][0] * gu[2][1] - gu[1][1] * gu[2][0];
    cg[1][0] = gu[0][2] * gu[2][1] - gu[0][1] * gu[2][2];
    cg[1][1] = gu[0][0] * gu[2][2] - gu[0][2] * gu[2][0];
    cg[1][2] = gu[0][1] * gu[2][0] - gu[0][0] * gu[2][1];
    cg[2][0] = gu[0][1] * gu[1][2] - gu[0][2] * gu[1][1];
    cg[2][1] = gu[0][2] * gu[1][0] - gu[0][0] * gu[1][2];
    cg[2][2] = gu[0][0] * gu[1][1] - gu[0][1] * gu[1][0];
    const double I2 = cg[0][0] + cg[1][1] + cg[2][2];
    const double I3 = gu[0][0] * cg[0][0] + gu[0][1] * cg[0][1] + gu[0][2] * cg[0][2];
    const double Jm1 = trg + I2 + I3;
    const double J = 1.0 + Jm1;
    detF = J;
    if (!(J > 0.0)) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) P[i][j] = 0.0;
      return false;
    }
    double gg = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) gg += gu[i][j] * gu[i][j];
    const double e = (2.0 * trg + gg) / 3.0;
    const double dI = (Jm1 - e);
    const double Ga = mp.mu * pow(J, -5.0 / 3.0);  // G J^{-2/3} / J
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double c = (i == j ? trg : 0.0) - gu[j][i] + cg[i][j];
        const double dev = (i == j ? dI : 0.0) + (1.0 + Jm1) * gu[i][j] - (1.0 + e) * c;
        P[i][j] = Ga * dev + mp.kappa * Jm1 * ((i == j ? 1.0 : 0.0) + c);
      }
    return true;
  } else {  // J2 perfect plasticity, radial return
    double st[3][3], s[3][3], seff;
    bool pos;
    j2_trial(gu, ep, sp, mp, st, s, seff, pos);
    const double over = fmax(seff - mp.sy, 0.0);
    const double f = over / seff;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) P[i][j] = st[i][j] - s[i][j] * f;
    return true;
  }
}

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
__global__ void __launch_bounds__(kThreads) k_residual(ElemArgs a, const int32_t *__restrict__ list, int64_t n,
                                                       double *__restrict__ R) {
  constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  __shared__ double sX[kWarps][4][8][3];
  __shared__ double sU[kWarps][4][8][VEC];
  __shared__ double sT[kWarps][4][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, slot = lane >> 3, q = lane & 7;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp0 * 4; base < n; base += nwarps * 4) {
    const int64_t idx = base + slot;
    const bool valid = idx < n;
    const int64_t e = list[valid ? idx : base];
    const int node = a.cells[e * 8 + q];
#pragma unroll
    for (int d = 0; d < 3; ++d) sX[w][slot][q][d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
    for (int v = 0; v < VEC; ++v) sU[w][slot][q][v] = a.U[(int64_t)node * VEC + v];
    if (MAT == B200FEM_MAT_POISSON && a.mp.design_source) sT[w][slot][q] = a.theta[node];
    __syncwarp();
    double G[8][3];
    const double jxw = qp_geometry(sX[w][slot], q, G);
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
    if (valid) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) R[(int64_t)node * VEC + v] += mine[v];
    }
    __syncwarp();
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
// Warp per cell.  Lanes 0..7 tabulate per-quadrature-point vectors in shared memory:
//   g_k = G_k, u_k = F g_k, h_k = H g_k (NH) or s g_k (J2), and the scalar coefficients
// of the closed-form block
//   K_ik(a,b) = sum_q [ C1 d_ik (g_a.g_b) + Cl g_a,i g_b,k + Cm g_a,k g_b,i
//                       - C2 (u_a,i h_b,k + h_a,i u_b,k) + C3 h_a,i h_b,k + C4 h_b,i h_a,k ]
// (LE: C1=Cm=mu, Cl=lam; J2: C1=Cm=mu-beta/2, Cl=lam+beta/3, C3=-gamma;
//  NH: C1=G a, C2=2/3 G a, C3=2/9 G a I1 + k(2J^2-J), C4=G/3 a I1 - k(J^2-J); all * JxW * theta^p)
// then all 32 lanes accumulate two (a,b) 3x3 blocks each and RMW them into the CSR values.
constexpr int kJacWarps = 4;

template <int MAT>
struct JacSmem {
  double X[8][3];
  double U[8][3];
  double g[8][8][3];
  double u[(MAT == B200FEM_MAT_NH) ? 8 : 1][8][3];
  double h[(MAT == B200FEM_MAT_NH || MAT == B200FEM_MAT_J2) ? 8 : 1][8][3];
  double coef[8][6];
  int node[8];
};

template <int MAT>
__global__ void __launch_bounds__(kJacWarps * 32) k_jacobian(ElemArgs a, const int32_t *__restrict__ list, int64_t n,
                                                             const uint8_t *__restrict__ cpos,
                                                             const int32_t *__restrict__ indptr,
                                                             double *__restrict__ data) {
  constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  __shared__ JacSmem<MAT> sm_all[kJacWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  JacSmem<MAT> &S = sm_all[w];
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t idx = warp0; idx < n; idx += nwarps) {
    const int64_t e = list[idx];
    if (lane < 8) {
      const int node = a.cells[e * 8 + lane];
      S.node[lane] = node;
#pragma unroll
      for (int d = 0; d < 3; ++d) S.X[lane][d] = a.coords[(int64_t)node * 3 + d];
#pragma unroll
      for (int v = 0; v < VEC; ++v) S.U[lane][v] = a.U[(int64_t)node * VEC + v];
    }
    __syncwarp();
    if (lane < 8) {
      const int q = lane;
      double G[8][3];
      const double jxw = qp_geometry(S.X, q, G);
      double scale = jxw;
      if (a.mp.simp) scale *= pow(a.theta[e], a.mp.penalty);
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) S.g[q][k][d] = G[k][d];
      double C[6] = {0, 0, 0, 0, 0, 0};  // C1, Cl, Cm, C2, C3, C4
      bool bad_def = false;
      double detF = 1.0;
      if (MAT == B200FEM_MAT_POISSON) {
        C[0] = a.mp.alpha * scale;
      } else {
        double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int v = 0; v < 3; ++v)
#pragma unroll
            for (int d = 0; d < 3; ++d) gu[v][d] = fma(S.U[k][v], G[k][d], gu[v][d]);
        if (MAT == B200FEM_MAT_LE) {
          C[0] = a.mp.mu * scale;
          C[1] = a.mp.lam * scale;
          C[2] = a.mp.mu * scale;
        } else if (MAT == B200FEM_MAT_NH) {
          double F[3][3];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) F[i][j] = gu[i][j] + (i == j ? 1.0 : 0.0);
          const double J = det3(F);
          detF = J;
          double H[3][3];
          if (J > 0.0) {
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
          const double aa = bad_def ? 0.0 : pow(J, -2.0 / 3.0);
          const double Ga = a.mp.mu * aa;
          C[0] = Ga * scale;
          C[3] = (2.0 / 3.0) * Ga * scale;
          C[4] = ((2.0 / 9.0) * Ga * I1 + a.mp.kappa * J * (2.0 * J - 1.0)) * scale;
          C[5] = ((1.0 / 3.0) * Ga * I1 - a.mp.kappa * J * (J - 1.0)) * scale;
#pragma unroll
          for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              S.u[q][k][i] = F[i][0] * G[k][0] + F[i][1] * G[k][1] + F[i][2] * G[k][2];
              S.h[q][k][i] = H[i][0] * G[k][0] + H[i][1] * G[k][1] + H[i][2] * G[k][2];
            }
        } else {  // J2 consistent tangent (derivative of j2_return_map incl. the s=0 guard)
          const double *ep = a.eps_prev + (e * 8 + q) * 9;
          const double *sp = a.sig_prev + (e * 8 + q) * 9;
          double st[3][3], s[3][3], seff;
          bool pos;
          j2_trial(gu, ep, sp, a.mp, st, s, seff, pos);
          const double over = fmax(seff - a.mp.sy, 0.0);
          const double f = over / seff;
          const double active = (seff - a.mp.sy > 0.0) ? 1.0 : 0.0;  // ramp'(0) = 0
          const double gam = pos ? (active / seff - over / (seff * seff)) * 3.0 * a.mp.mu / seff : 0.0;
          const double beta = 2.0 * a.mp.mu * f;
          C[0] = (a.mp.mu - 0.5 * beta) * scale;
          C[1] = (a.mp.lam + beta / 3.0) * scale;
          C[2] = C[0];
          C[4] = -gam * scale;
#pragma unroll
          for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int i = 0; i < 3; ++i) S.h[q][k][i] = s[i][0] * G[k][0] + s[i][1] * G[k][1] + s[i][2] * G[k][2];
        }
      }
      bool fin = true;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        S.coef[q][j] = C[j];
        fin &= isfinite(C[j]);
      }
      const unsigned long long key = (unsigned long long)e * 8 + q;
      if (bad_def) {
        atomicMin(&a.derr->inv_def, key);
        atomicMin(&a.derr->min_detF, ord_bits(detF));
      } else if (!fin) {
        atomicMin(&a.derr->nonfin_d, key);
      }
    }
    __syncwarp();
    // ---- accumulate two (a,b) blocks per lane over the 8 quadrature points
    const int b = lane & 7, a0 = lane >> 3, a1 = a0 + 4;
    double K0[VEC][VEC], K1[VEC][VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i)
#pragma unroll
      for (int k = 0; k < VEC; ++k) K0[i][k] = K1[i][k] = 0.0;
#pragma unroll 2
    for (int q = 0; q < 8; ++q) {
      const double c1 = S.coef[q][0];
      const double gb0 = S.g[q][b][0], gb1 = S.g[q][b][1], gb2 = S.g[q][b][2];
      const double ga[2][3] = {{S.g[q][a0][0], S.g[q][a0][1], S.g[q][a0][2]},
                               {S.g[q][a1][0], S.g[q][a1][1], S.g[q][a1][2]}};
      const double gbv[3] = {gb0, gb1, gb2};
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double(&K)[VEC][VEC] = t ? K1 : K0;
        const double gg = ga[t][0] * gb0 + ga[t][1] * gb1 + ga[t][2] * gb2;
        if (MAT == B200FEM_MAT_POISSON) {
          K[0][0] = fma(c1, gg, K[0][0]);
        } else {
          const double d = c1 * gg;
#pragma unroll
          for (int i = 0; i < 3; ++i) K[i][i] += d;
          if (MAT == B200FEM_MAT_LE || MAT == B200FEM_MAT_J2) {
            const double cl = S.coef[q][1], cm = S.coef[q][2];
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int k = 0; k < 3; ++k) K[i][k] += cl * ga[t][i] * gbv[k] + cm * ga[t][k] * gbv[i];
          }
          if (MAT == B200FEM_MAT_J2) {
            const double c3 = S.coef[q][4];
            const int at = t ? a1 : a0;
            const double ha[3] = {S.h[q][at][0], S.h[q][at][1], S.h[q][at][2]};
            const double hb[3] = {S.h[q][b][0], S.h[q][b][1], S.h[q][b][2]};
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int k = 0; k < 3; ++k) K[i][k] = fma(c3 * ha[i], hb[k], K[i][k]);
          }
          if (MAT == B200FEM_MAT_NH) {
            const double c2 = S.coef[q][3], c3 = S.coef[q][4], c4 = S.coef[q][5];
            const int at = t ? a1 : a0;
            const double ha[3] = {S.h[q][at][0], S.h[q][at][1], S.h[q][at][2]};
            const double hb[3] = {S.h[q][b][0], S.h[q][b][1], S.h[q][b][2]};
            const double ua[3] = {S.u[q][at][0], S.u[q][at][1], S.u[q][at][2]};
            const double ub[3] = {S.u[q][b][0], S.u[q][b][1], S.u[q][b][2]};
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
              for (int k = 0; k < 3; ++k)
                K[i][k] += c3 * ha[i] * hb[k] + c4 * hb[i] * ha[k] - c2 * (ua[i] * hb[k] + ha[i] * ub[k]);
          }
        }
      }
    }
    // ---- scatter into the fixed CSR pattern (colour classes are node-disjoint)
    const int nb = S.node[b];
    (void)nb;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int at = t ? a1 : a0;
      const int na = S.node[at];
      const int p = cpos[e * 64 + at * 8 + b];
      double(&K)[VEC][VEC] = t ? K1 : K0;
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        double *row = data + indptr[(int64_t)na * VEC + i] + VEC * p;
#pragma unroll
        for (int k = 0; k < VEC; ++k) row[k] += K[i][k];
      }
    }
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

template <int MAT>
static void residual_colors(Ctx *c, const ElemArgs &a, double *R) {
  for (int col = 0; col < c->n_colors; ++col) {
    const int64_t lo = c->color_off[col], n = c->color_off[col + 1] - lo;
    if (n == 0) continue;
    k_residual<MAT><<<grid_cap(n, kWarps * 4), kThreads, 0, c->stream>>>(a, c->color_cells + lo, n, R);
    count_launch();
  }
}

int launch_residual(Ctx *c, const double *U, double *R, double bc_scale, int apply_dirichlet, b200fem_error *err,
                    double *norm_host) {
  cudaStream_t s = c->stream;
  B200_CUDA_E(cudaMemsetAsync(R, 0, c->n_dofs * sizeof(double), s), err);
  const ElemArgs a = make_args(c, U);
  switch (c->material) {
    case B200FEM_MAT_POISSON: residual_colors<B200FEM_MAT_POISSON>(c, a, R); break;
    case B200FEM_MAT_LE: residual_colors<B200FEM_MAT_LE>(c, a, R); break;
    case B200FEM_MAT_NH: residual_colors<B200FEM_MAT_NH>(c, a, R); break;
    default: residual_colors<B200FEM_MAT_J2>(c, a, R); break;
  }
  if (c->f_neumann || c->f_body) {
    k_res_finalize<<<grid_cap(c->n_dofs, kThreads), kThreads, 0, s>>>(R, c->n_dofs, bc_scale, c->f_neumann, c->f_body);
    count_launch();
  }
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

template <int MAT>
static void jacobian_colors(Ctx *c, const ElemArgs &a, double *data) {
  for (int col = 0; col < c->n_colors; ++col) {
    const int64_t lo = c->color_off[col], n = c->color_off[col + 1] - lo;
    if (n == 0) continue;
    k_jacobian<MAT><<<grid_cap(n, kJacWarps), kJacWarps * 32, 0, c->stream>>>(a, c->color_cells + lo, n, c->cpos,
                                                                               c->indptr, data);
    count_launch();
  }
}

int launch_jacobian(Ctx *c, const double *U, double *data, b200fem_error *err) {
  cudaStream_t s = c->stream;
  B200_CUDA_E(cudaMemsetAsync(data, 0, c->nnz * sizeof(double), s), err);
  const ElemArgs a = make_args(c, U);
  switch (c->material) {
    case B200FEM_MAT_POISSON: jacobian_colors<B200FEM_MAT_POISSON>(c, a, data); break;
    case B200FEM_MAT_LE: jacobian_colors<B200FEM_MAT_LE>(c, a, data); break;
    case B200FEM_MAT_NH: jacobian_colors<B200FEM_MAT_NH>(c, a, data); break;
    default: jacobian_colors<B200FEM_MAT_J2>(c, a, data); break;
  }
  if (c->n_dir) {
    k_jac_dirichlet<<<grid_cap(c->n_dir * 32, kThreads), kThreads, 0, s>>>(data, c->indptr, c->diag, c->dir_dofs,
                                                                           c->n_dir);
    count_launch();
  }
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
  return launch_jacobian((Ctx *)ctx, U, data, err);
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

}  // extern "C"
