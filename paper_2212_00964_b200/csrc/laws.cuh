// Constitutive laws at one quadrature point (device functions shared by the element
// kernels in element.cu and the batch law entry points in material.cu).
//
// Reference (paths relative to gradfem/): materials.py:74-131 -- linear_elastic_flux,
// neo_hookean_energy / neo_hookean_flux (AD of W), j2_return_map, commit_state; the
// consistent tangents are the hand-derived forms of SURVEY.md Appendix A.
#pragma once

#include <cmath>

#include "internal.cuh"

namespace b200 {

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
    if (J <= 0.0) {  // NaN J is not 'inverted' (materials.py:94: np.any(J <= 0)) but a non-finite flux
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
    const double rc = rcbrt(J);
    const double Ga = mp.mu * (rc * rc) / J;  // G J^{-2/3} / J (rcbrt: far cheaper than pow)
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

// Consistent tangent A[iJ][kL] = d flux_iJ / d (grad u)_kL at one point (
// the same factors as the element tangent in element.cu with g_a = e_J, g_b = e_L):
//   NH: A = c1 d_ik d_JL + H_iJ (c3 H_kL - c2 F_kL) - c2 F_iJ H_kL + c4 H_iL H_kJ
//       c1 = G a, c2 = 2/3 G a, c3 = 2/9 G a I1 + k J (2J - 1), c4 = G/3 a I1 - k J (J - 1)
//   J2: A = c1 (d_ik d_JL + d_iL d_kJ) + cl d_iJ d_kL - gamma s_iJ s_kL (c1 = mu - beta/2,
//       cl = lam + beta/3, beta = 2 mu <s_eff - sy>+ / s_eff; gamma from ramp'(0) = 0);
//   LE: J2 with beta = gamma = 0;   Poisson: alpha d_JL.
// Returns false on det F <= 0 (NH; A zeroed).
template <int MAT>
__device__ __forceinline__ bool tangent_at(const double (&gu)[3][3], const MatParams &mp, const double *ep,
                                           const double *sp, double (&A)[9][9]) {
#pragma unroll
  for (int r = 0; r < 9; ++r)
#pragma unroll
    for (int c = 0; c < 9; ++c) A[r][c] = 0.0;
  if (MAT == B200FEM_MAT_POISSON) {
#pragma unroll
    for (int d = 0; d < 3; ++d) A[d][d] = mp.alpha;
    return true;
  }
  if (MAT == B200FEM_MAT_NH) {
    double F[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) F[i][j] = gu[i][j] + (i == j ? 1.0 : 0.0);
    const double J = det3(F);
    if (J <= 0.0) return false;
    double H[3][3];
    inv_transpose(F, J, H);
    double I1 = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) I1 += F[i][j] * F[i][j];
    const double rc = rcbrt(J);
    const double Ga = mp.mu * (rc * rc);
    const double c1 = Ga, c2 = (2.0 / 3.0) * Ga;
    const double c3 = (2.0 / 9.0) * Ga * I1 + mp.kappa * J * (2.0 * J - 1.0);
    const double c4 = (1.0 / 3.0) * Ga * I1 - mp.kappa * J * (J - 1.0);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int Jj = 0; Jj < 3; ++Jj)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int L = 0; L < 3; ++L)
            A[i * 3 + Jj][k * 3 + L] = ((i == k && Jj == L) ? c1 : 0.0) + H[i][Jj] * (c3 * H[k][L] - c2 * F[k][L]) -
                                       c2 * F[i][Jj] * H[k][L] + c4 * H[i][L] * H[k][Jj];
    return true;
  }
  double c1 = mp.mu, cl = mp.lam, gam = 0.0, sd[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  if (MAT == B200FEM_MAT_J2) {
    double st[3][3], seff;
    bool pos;
    j2_trial(gu, ep, sp, mp, st, sd, seff, pos);
    const double over = fmax(seff - mp.sy, 0.0);
    const double active = (seff - mp.sy > 0.0) ? 1.0 : 0.0;  // ramp'(0) = 0 (autodiff.py:177-181)
    gam = pos ? (active / seff - over / (seff * seff)) * 3.0 * mp.mu / seff : 0.0;
    const double beta = 2.0 * mp.mu * (over / seff);
    c1 = mp.mu - 0.5 * beta;
    cl = mp.lam + beta / 3.0;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int Jj = 0; Jj < 3; ++Jj)
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int L = 0; L < 3; ++L)
          A[i * 3 + Jj][k * 3 + L] = ((i == k && Jj == L) ? c1 : 0.0) + ((i == L && k == Jj) ? c1 : 0.0) +
                                     ((i == Jj && k == L) ? cl : 0.0) - gam * sd[i][Jj] * sd[k][L];
  return true;
}

// W(F) = G/2 (J^{-2/3} I1 - 3) + kappa/2 (J - 1)^2 (materials.py:80-85); NaN for J < 0 like
// numpy's J ** (-2/3) of a negative base.
__device__ __forceinline__ double nh_energy(const double (&F)[3][3], const MatParams &mp) {
  const double J = det3(F);
  double I1 = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) I1 += F[i][j] * F[i][j];
  return 0.5 * mp.mu * (pow(J, -2.0 / 3.0) * I1 - 3.0) + 0.5 * mp.kappa * (J - 1.0) * (J - 1.0);
}

}  // namespace b200
