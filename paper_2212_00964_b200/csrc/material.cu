// Constitutive laws over a batch of quadrature points: the device side of the reference's
// material API (gradfem/materials.py:74-194 -- linear_elastic_flux, neo_hookean_energy,
// neo_hookean_flux, j2_return_map, commit_state and Material.flux / J2Plasticity.commit),
// so that host code calling the laws directly (reference tests/test_materials.py) gets the
// same device arithmetic the element kernels use (laws.cuh), not a host restatement.
//
// Thread per point; HBM-bound streaming (9 doubles in, 9 out; 81 out with the tangent).

#include <cmath>

#include "internal.cuh"
#include "laws.cuh"

namespace b200 {

struct LawOut {
  double *flux, *tangent, *eps, *sig, *det;
};

struct BatchErr {
  unsigned long long first_bad;  // smallest point index with det F <= 0
  unsigned long long min_det;    // ordered bits of the smallest such det F
};

__device__ __forceinline__ unsigned long long ord_bits_l(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <int MAT>
__global__ void __launch_bounds__(kThreads) k_law_batch(MatParams mp, int64_t n, const double *__restrict__ gu_in,
                                                         const double *__restrict__ ep, const double *__restrict__ sp,
                                                         LawOut o, BatchErr *be) {
  constexpr int VEC = (MAT == B200FEM_MAT_POISSON) ? 1 : 3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int v = 0; v < VEC; ++v)
#pragma unroll
      for (int d = 0; d < 3; ++d) gu[v][d] = gu_in[t * VEC * 3 + v * 3 + d];
    const double *e9 = (MAT == B200FEM_MAT_J2) ? ep + t * 9 : nullptr;
    const double *s9 = (MAT == B200FEM_MAT_J2) ? sp + t * 9 : nullptr;
    double P[3][3], detF = 1.0;
    const bool ok = flux_at<MAT>(gu, mp, e9, s9, P, detF);
    if (!ok) {
      atomicMin(&be->first_bad, (unsigned long long)t);
      atomicMin(&be->min_det, ord_bits_l(detF));
    }
    if (o.det) o.det[t] = detF;
    if (o.flux) {
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int d = 0; d < 3; ++d) o.flux[t * VEC * 3 + v * 3 + d] = P[v][d];
    }
    if (o.tangent) {
      double A[9][9];
      tangent_at<MAT>(gu, mp, e9, s9, A);
      constexpr int M = VEC * 3;
#pragma unroll
      for (int r = 0; r < M; ++r)
#pragma unroll
        for (int c = 0; c < M; ++c) o.tangent[t * M * M + r * M + c] = A[r][c];
    }
    if (MAT == B200FEM_MAT_J2 && o.eps) {  // commit_state (materials.py:125-131)
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          o.eps[t * 9 + i * 3 + j] = 0.5 * (gu[i][j] + gu[j][i]);
          o.sig[t * 9 + i * 3 + j] = P[i][j];
        }
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_nh_energy(MatParams mp, int64_t n, const double *__restrict__ F9,
                                                         double *__restrict__ W) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double F[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) F[i][j] = F9[t * 9 + i * 3 + j];
    W[t] = nh_energy(F, mp);
  }
}

static MatParams params_from(const double *p) {
  MatParams mp{};
  mp.alpha = p[0];
  mp.lam = p[1];
  mp.mu = p[2];
  mp.kappa = p[3];
  mp.sy = p[4];
  return mp;
}

static int batch_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 16));
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_law_batch(int32_t material_id, const double *params, int64_t n, const double *grad_u,
                      const double *eps_prev, const double *sig_prev, double *flux, double *tangent,
                      double *eps_out, double *sig_out, double *det_f, void *stream, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (!params || n < 0 || (n > 0 && !grad_u) || material_id < B200FEM_MAT_POISSON || material_id > B200FEM_MAT_J2)
    return B200FEM_E_INVALID;
  if (material_id == B200FEM_MAT_J2 && (!eps_prev || !sig_prev || (!eps_out) != (!sig_out)))
    return B200FEM_E_INVALID;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const MatParams mp = params_from(params);
  BatchErr *be = nullptr;
  B200_CUDA_E(cudaMallocAsync((void **)&be, sizeof(BatchErr), s), err);
  B200_CUDA_E(cudaMemsetAsync(be, 0xff, sizeof(BatchErr), s), err);
  const LawOut o{flux, tangent, eps_out, sig_out, det_f};
  const int g = batch_grid(n);
  switch (material_id) {
    case B200FEM_MAT_POISSON: k_law_batch<B200FEM_MAT_POISSON><<<g, kThreads, 0, s>>>(mp, n, grad_u, nullptr, nullptr, o, be); break;
    case B200FEM_MAT_LE: k_law_batch<B200FEM_MAT_LE><<<g, kThreads, 0, s>>>(mp, n, grad_u, nullptr, nullptr, o, be); break;
    case B200FEM_MAT_NH: k_law_batch<B200FEM_MAT_NH><<<g, kThreads, 0, s>>>(mp, n, grad_u, nullptr, nullptr, o, be); break;
    default: k_law_batch<B200FEM_MAT_J2><<<g, kThreads, 0, s>>>(mp, n, grad_u, eps_prev, sig_prev, o, be); break;
  }
  count_launch();
  B200_CUDA_E(cudaGetLastError(), err);
  BatchErr h;
  B200_CUDA_E(cudaMemcpyAsync(&h, be, sizeof(h), cudaMemcpyDeviceToHost, s), err);
  B200_CUDA_E(cudaFreeAsync(be, s), err);
  B200_CUDA_E(cudaStreamSynchronize(s), err);
  if (h.first_bad != ~0ull) {
    unsigned long long u = h.min_det;
    unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    double mn;
    memcpy(&mn, &b, sizeof(mn));
    if (err) {
      err->code = B200FEM_E_INVERTED_DEFORMATION;
      err->cell = (int64_t)h.first_bad;
      err->value = mn;
      snprintf(err->msg, sizeof(err->msg),
               "det(F) <= 0 (min %.3e): element inverted beyond the neo-Hookean domain", mn);
    }
    return B200FEM_E_INVERTED_DEFORMATION;
  }
  return 0;
}

int b200fem_nh_energy_batch(const double *params, int64_t n, const double *F, double *W, void *stream) {
  if (!params || n < 0 || (n > 0 && (!F || !W))) return B200FEM_E_INVALID;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  k_nh_energy<<<batch_grid(n), kThreads, 0, s>>>(params_from(params), n, F, W);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

}  // extern "C"
