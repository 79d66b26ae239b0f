// Partitioned BiCGSTAB: the mesh is split into contiguous node
// ranges ("parts"); each part owns the DOF rows of its nodes and holds a ghost layer of
// cells, so its owned rows assemble locally with no communication.  Per iteration the
// only exchanges are
//   * a halo of the SpMV operand (p, then s): owned values of interface nodes -> the ghost
//     entries of the neighbouring parts (packed, ncclSend/ncclRecv),
//   * three FP64 sum-allreduces of the fused dot groups {r0.v}, {t.t, t.s},
//     {||D r||^2, r0.r, r.r}, after which every part applies the same scalar update -- or
//     two, the third group folded into the second by recurrence, from 4 NCCL ranks
//     (enqueue_dist_iteration_fused) -- (Jacobi-PCG: one halo and two allreduces, {p.Ap},
//     {r.r, r.z}).
// Batches of iterations run as one CUDA graph with the NCCL calls captured on a private
// stream (capture_batch, run_batches).
// Communicators: NCCL across processes (one part per process and GPU), or "local": all
// parts in one process on one device, exchanged by device copies and summed by a kernel
// in part order -- the same algorithm, used to verify partitioning on a single B200.

#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace b200 {

struct Comm {
  int kind = 0;  // 0 local, 1 nccl
  ncclComm_t nccl = nullptr;
  int rank = 0, nranks = 1;
};

struct Part {
  Matrix *m = nullptr;
  int vec = 3;
  int64_t own_lo = 0, own_hi = 0;  // owned local node range
  int n_peers = 0;
  std::vector<int> peer;           // peer part index (local) or rank (nccl)
  std::vector<int64_t> soff, roff; // node offsets into the packed buffers (n_peers + 1)
  int32_t *send_nodes = nullptr, *recv_nodes = nullptr;
  double *sendbuf = nullptr, *recvbuf = nullptr;
  // halo / interior overlap (GRID3 parts): rows of [int_lo, int_hi) touch no ghost node, so
  // their SpMV runs on s2 while the halo is exchanged; the two boundary bands follow it
  bool overlap = false;
  int64_t int_lo = 0, int_hi = 0;
  // every peer's send and recv node list is a contiguous local range (plane-cut lattices):
  // the halo then moves vector slices directly -- no pack / unpack kernels
  bool contiguous = false;
  std::vector<int64_t> s_lo, r_lo;
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_in = nullptr, ev_done = nullptr;
  RedScratch red_in{}, red_lo{}, red_hi{};  // partial dot totals of the three launches
  RedScratch red6{};  // the extra dots of the two-allreduce BiCGSTAB (lazy)
};

// total of the three partial dot groups, in a fixed order (deterministic)
__global__ void k_sum3(const double *a, const double *b, const double *c, double *out, int nv) {
  const int j = threadIdx.x;
  if (j < nv) out[j] = (a[j] + b[j]) + c[j];
}

__global__ void k_pack(const double *__restrict__ v, const int32_t *__restrict__ nodes, int64_t n, int vec,
                       double *__restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * vec; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = v[(int64_t)nodes[i / vec] * vec + i % vec];
}

__global__ void k_unpack(double *__restrict__ v, const int32_t *__restrict__ nodes, int64_t n, int vec,
                         const double *__restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * vec; i += (int64_t)gridDim.x * blockDim.x)
    v[(int64_t)nodes[i / vec] * vec + i % vec] = buf[i];
}

// sum NV values over the parts in part order and broadcast the total back (deterministic)
__global__ void k_sum_parts(double *const *res, int np, int nv) {
  const int j = threadIdx.x;
  if (j >= nv) return;
  double s = 0.0;
  for (int p = 0; p < np; ++p) s += res[p][j];
  for (int p = 0; p < np; ++p) res[p][j] = s;
}

__global__ void k_stage(int kind, KrylovScalars *S, const double *tot) { apply_stage(kind, S, tot); }

// owned-range dot product -> red.result[0]
__global__ void __launch_bounds__(kThreads) k_dot_owned(const double *__restrict__ x, const double *__restrict__ y,
                                                        int64_t n, RedScratch red) {
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[0] = fma(x[i], y[i], v[0]);
  double tot[1];
  block_partials_and_finish<1>(v, red, tot);
}

// {r0.s, r0.t, s.s, |Ds|^2, Ds.Dt, |Dt|^2} over the owned rows; totals land in out[0..5]
__global__ void __launch_bounds__(kThreads) k_dot6(int64_t n, const double *__restrict__ r0,
                                                   const double *__restrict__ s, const double *__restrict__ t,
                                                   const double *__restrict__ dg, const KrylovScalars *S,
                                                   RedScratch red) {
  if (S->status != KS_RUNNING) return;
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double si = s[i], ti = t[i], qi = r0[i], d = dg[i];
    const double ds = d * si, dt = d * ti;
    acc[0] = fma(qi, si, acc[0]);
    acc[1] = fma(qi, ti, acc[1]);
    acc[2] = fma(si, si, acc[2]);
    acc[3] = fma(ds, ds, acc[3]);
    acc[4] = fma(ds, dt, acc[4]);
    acc[5] = fma(dt, dt, acc[5]);
  }
  double tot[6];
  block_partials_and_finish<6>(acc, red, tot);
}

// x += alpha p + omega s, r = s - omega t, without reductions (their dots came by recurrence)
__global__ void __launch_bounds__(kThreads) k_update_xr_nored(int64_t n, double *__restrict__ x,
                                                              double *__restrict__ r, const double *__restrict__ p,
                                                              const double *__restrict__ s,
                                                              const double *__restrict__ t, const KrylovScalars *S) {
  if (S->status != KS_RUNNING) return;
  const double alpha = S->alpha, omega = S->omega;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i] + omega * s[i];
    r[i] = s[i] - omega * t[i];
  }
}

static int grid_n(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + kThreads - 1) / kThreads)); }

struct Dist {
  std::vector<Part *> parts;
  Comm *comm;
  double **res_dev = nullptr;  // device array of the parts' red.result pointers (local comm)

  cudaStream_t stream(int p) const { return parts[p]->m->stream; }

  int allreduce(int nv) {
    if (comm->kind == 1) {
      Part *P = parts[0];
      double *r = P->m->kw->red.result;
      if (ncclAllReduce(r, r, nv, ncclDouble, ncclSum, comm->nccl, stream(0)) != ncclSuccess) return B200FEM_E_CUDA;
      return 0;
    }
    if (parts.size() == 1) return 0;
    k_sum_parts<<<1, 32, 0, stream(0)>>>(res_dev, (int)parts.size(), nv);
    count_launch();
    return 0;
  }

  // ghost entries of vec[p] <- owners' values
  int halo(double *const *vec) {
    for (size_t p = 0; p < parts.size(); ++p) {
      Part *P = parts[p];
      const int64_t ns = P->soff.back();
      if (ns && !P->contiguous) {
        k_pack<<<grid_n(ns * P->vec), kThreads, 0, stream(p)>>>(vec[p], P->send_nodes, ns, P->vec, P->sendbuf);
        count_launch();
      }
    }
    if (comm->kind == 1) {
      Part *P = parts[0];
      if (P->n_peers) {
        ncclGroupStart();
        for (int i = 0; i < P->n_peers; ++i) {
          const int64_t sn = P->soff[i + 1] - P->soff[i], rn = P->roff[i + 1] - P->roff[i];
          const double *sp = P->contiguous ? vec[0] + P->s_lo[i] * P->vec : P->sendbuf + P->soff[i] * P->vec;
          double *rp = P->contiguous ? vec[0] + P->r_lo[i] * P->vec : P->recvbuf + P->roff[i] * P->vec;
          if (sn) ncclSend(sp, sn * P->vec, ncclDouble, P->peer[i], comm->nccl, stream(0));
          if (rn) ncclRecv(rp, rn * P->vec, ncclDouble, P->peer[i], comm->nccl, stream(0));
        }
        if (ncclGroupEnd() != ncclSuccess) return B200FEM_E_CUDA;
      }
    } else {
      for (size_t p = 0; p < parts.size(); ++p) {
        Part *P = parts[p];
        for (int i = 0; i < P->n_peers; ++i) {
          Part *Q = parts[P->peer[i]];
          int j = 0;
          while (j < Q->n_peers && Q->peer[j] != (int)p) ++j;
          if (j == Q->n_peers) return B200FEM_E_INVALID;
          const int64_t rn = P->roff[i + 1] - P->roff[i];
          if (rn != Q->soff[j + 1] - Q->soff[j]) return B200FEM_E_INVALID;
          const double *sp = Q->contiguous ? vec[P->peer[i]] + Q->s_lo[j] * Q->vec : Q->sendbuf + Q->soff[j] * Q->vec;
          double *rp = P->contiguous ? vec[p] + P->r_lo[i] * P->vec : P->recvbuf + P->roff[i] * P->vec;
          if (rn) B200_CUDA(cudaMemcpyAsync(rp, sp, rn * P->vec * sizeof(double), cudaMemcpyDeviceToDevice, stream(p)));
        }
      }
    }
    for (size_t p = 0; p < parts.size(); ++p) {
      Part *P = parts[p];
      const int64_t nr = P->roff.back();
      if (nr && !P->contiguous) {
        k_unpack<<<grid_n(nr * P->vec), kThreads, 0, stream(p)>>>(vec[p], P->recv_nodes, nr, P->vec, P->recvbuf);
        count_launch();
      }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
  }

  // y = op(A) v over the owned rows of every part, partial dot totals left in red.result
  // (inline_stage 0): halo of v first, or overlapped with the interior rows (GRID3 parts)
  int spmv(SpmvMode mode, const std::vector<SpmvArgs> &a, double *const *vec, int nv) {
    for (size_t p = 0; p < parts.size(); ++p) {
      Part *P = parts[p];
      if (!P->overlap) continue;
      Matrix *m = P->m;
      B200_CUDA(cudaEventRecord(P->ev_in, stream(p)));
      B200_CUDA(cudaStreamWaitEvent(P->s2, P->ev_in, 0));
      cudaStream_t ms = m->stream;
      m->stream = P->s2;
      m->row_lo = P->int_lo, m->row_hi = P->int_hi;
      const int st = launch_spmv(m, mode, a[p], &P->red_in);
      m->stream = ms;  // restored on every path
      if (st) return B200FEM_E_CUDA;
      B200_CUDA(cudaEventRecord(P->ev_done, P->s2));
    }
    if (int st = halo(vec)) return st;
    for (size_t p = 0; p < parts.size(); ++p) {
      Part *P = parts[p];
      Matrix *m = P->m;
      KrylovWork *w = m->kw;
      if (!P->overlap) {
        if (launch_spmv(m, mode, a[p], &w->red)) return B200FEM_E_CUDA;
        continue;
      }
      m->row_lo = P->own_lo, m->row_hi = P->int_lo;
      if (launch_spmv(m, mode, a[p], &P->red_lo)) return B200FEM_E_CUDA;
      m->row_lo = P->int_hi, m->row_hi = P->own_hi;
      if (launch_spmv(m, mode, a[p], &P->red_hi)) return B200FEM_E_CUDA;
      m->row_lo = P->own_lo, m->row_hi = P->own_hi;
      B200_CUDA(cudaStreamWaitEvent(stream(p), P->ev_done, 0));
      k_sum3<<<1, 32, 0, stream(p)>>>(P->red_in.result, P->red_lo.result, P->red_hi.result, w->red.result, nv);
      count_launch();
    }
    return 0;
  }

  void stage(int kind) {
    for (size_t p = 0; p < parts.size(); ++p) {
      KrylovWork *w = parts[p]->m->kw;
      k_stage<<<1, 1, 0, stream(p)>>>(kind, w->sc, w->red.result);
      count_launch();
    }
  }

  // owned dot products summed over ranks -> host
  int dot(double *const *x, double *const *y, double *out) {
    for (size_t p = 0; p < parts.size(); ++p) {
      Part *P = parts[p];
      const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
      k_dot_owned<<<kRedBlocks, kThreads, 0, stream(p)>>>(x[p] + lo, y[p] + lo, n, P->m->kw->red);
      count_launch();
    }
    int st = allreduce(1);
    if (st) return st;
    B200_CUDA(cudaMemcpyAsync(out, parts[0]->m->kw->red.result, sizeof(double), cudaMemcpyDeviceToHost, stream(0)));
    B200_CUDA(cudaStreamSynchronize(stream(0)));
    return 0;
  }
};

static int enqueue_dist_iteration(Dist &D, double *const *x) {
  const size_t np = D.parts.size();
  std::vector<double *> pv(np), sv(np);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_update_p<<<grid_n(n), kThreads, 0, D.stream(p)>>>(n, w->r + lo, w->v + lo, w->p + lo, w->sc);
    count_launch();
    pv[p] = w->p;
    sv[p] = w->s;
  }
  std::vector<SpmvArgs> a1(np), a2(np);
  for (size_t p = 0; p < np; ++p) {
    KrylovWork *w = D.parts[p]->m->kw;
    a1[p] = SpmvArgs{w->p, w->v, w->inv, w->diag, w->r0, nullptr, w->sc, 0};
    a2[p] = SpmvArgs{w->s, w->t, w->inv, w->diag, nullptr, nullptr, w->sc, 0};
  }
  int st = D.spmv(SP_JACOBI_R0, a1, pv.data(), 1);
  st |= D.allreduce(1);
  D.stage(ST_R0);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_update_s<<<grid_n(n), kThreads, 0, D.stream(p)>>>(n, w->r + lo, w->v + lo, w->s + lo, w->sc);
    count_launch();
  }
  st |= D.spmv(SP_JACOBI_TT, a2, sv.data(), 2);
  st |= D.allreduce(2);
  D.stage(ST_TT);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_update_xr<<<xr_blocks(), kThreads, 0, D.stream(p)>>>(n, x[p] + lo, w->r + lo, w->p + lo, w->s + lo, w->t + lo,
                                                         w->r0 + lo, w->diag + lo, w->sc, w->red, 0);
    count_launch();
  }
  st |= D.allreduce(3);
  D.stage(ST_XR);
  return st || cudaPeekAtLastError() != cudaSuccess ? B200FEM_E_CUDA : 0;
}

// BiCGSTAB iteration with TWO allreduces (opt-in, B200FEM_DIST_FUSED_DOTS=1): the t-group also
// carries r0.s, r0.t, s.s, |Ds|^2, Ds.Dt, |Dt|^2 (one extra pass over 4 owned vectors), from
// which ST_TT8 forms omega and the next r's r0.r, r.r, |Dr|^2 by the recurrence r = s - omega t;
// x and r are then updated without a reduction.  Same iterates in exact arithmetic; in floating
// point the recurrence norms drift from the explicit ones, so the explicit residual of the
// outer loop (solvers.py:115-118) still decides convergence.  Pays only when an allreduce's
// latency exceeds the extra pass: by default on NCCL communicators of >= 4 ranks
// (DESIGN.md section 5); B200FEM_DIST_FUSED_DOTS=1 / =0 forces it on / off.
static bool dist_fused_dots(const Dist &D) {
  const char *e = getenv("B200FEM_DIST_FUSED_DOTS");
  if (e && *e) return *e != '0';
  return D.comm->kind == 1 && D.comm->nranks >= 4;
}

// k_dot6 in one full wave of resident blocks (42 registers: 5 per SM), as k_update_xr
static int dot6_blocks() {
  static int v = -1;
  if (v < 0) {
    int nb = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    v = (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_dot6, kThreads, 0) == cudaSuccess && nb > 0)
            ? std::min(kRedBlocks, nb * sms)
            : kRedBlocks;
    cudaGetLastError();
  }
  return v;
}

static int enqueue_dist_iteration_fused(Dist &D, double *const *x) {
  const size_t np = D.parts.size();
  std::vector<double *> pv(np), sv(np);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_update_p<<<grid_n(n), kThreads, 0, D.stream(p)>>>(n, w->r + lo, w->v + lo, w->p + lo, w->sc);
    count_launch();
    pv[p] = w->p;
    sv[p] = w->s;
  }
  std::vector<SpmvArgs> a1(np), a2(np);
  for (size_t p = 0; p < np; ++p) {
    KrylovWork *w = D.parts[p]->m->kw;
    a1[p] = SpmvArgs{w->p, w->v, w->inv, w->diag, w->r0, nullptr, w->sc, 0};
    a2[p] = SpmvArgs{w->s, w->t, w->inv, w->diag, nullptr, nullptr, w->sc, 0};
  }
  int st = D.spmv(SP_JACOBI_R0, a1, pv.data(), 1);
  st |= D.allreduce(1);
  D.stage(ST_R0);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_update_s<<<grid_n(n), kThreads, 0, D.stream(p)>>>(n, w->r + lo, w->v + lo, w->s + lo, w->sc);
    count_launch();
  }
  st |= D.spmv(SP_JACOBI_TT, a2, sv.data(), 2);
  for (size_t p = 0; p < np; ++p) {  // the six extra dots into red.result[2..7]
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    RedScratch r6{P->red6.partials, P->red6.ticket, w->red.result + 2};
    k_dot6<<<dot6_blocks(), kThreads, 0, D.stream(p)>>>(n, w->r0 + lo, w->s + lo, w->t + lo, w->diag + lo, w->sc, r6);
    count_launch();
  }
  st |= D.allreduce(8);
  D.stage(ST_TT8);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_update_xr_nored<<<grid_n(n), kThreads, 0, D.stream(p)>>>(n, x[p] + lo, w->r + lo, w->p + lo, w->s + lo,
                                                               w->t + lo, w->sc);
    count_launch();
  }
  D.stage(ST_CONV);
  return st || cudaPeekAtLastError() != cudaSuccess ? B200FEM_E_CUDA : 0;
}

// Jacobi-PCG iteration over the parts (krylov.cu enqueue_cg_iteration with the collectives):
// halo of p + SpMV q = A p with p.Ap -> allreduce -> alpha; x, r, z = D^-1 r with r.r, r.z ->
// allreduce -> beta; p = z + beta p.  Two allreduces and one halo per iteration.
static int enqueue_dist_cg_iteration(Dist &D, double *const *x) {
  const size_t np = D.parts.size();
  std::vector<double *> pv(np);
  std::vector<SpmvArgs> a(np);
  for (size_t p = 0; p < np; ++p) {
    KrylovWork *w = D.parts[p]->m->kw;
    a[p] = SpmvArgs{w->p, w->v, w->inv, w->diag, nullptr, nullptr, w->sc, 0};
    pv[p] = w->p;
  }
  int st = D.spmv(SP_PQ, a, pv.data(), 1);
  st |= D.allreduce(1);
  D.stage(ST_PQ);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_cg_update_xrz<<<kRedBlocks, kThreads, 0, D.stream(p)>>>(n, x[p] + lo, w->r + lo, w->p + lo, w->v + lo,
                                                             w->inv + lo, w->s + lo, w->sc, w->red, 0);
    count_launch();
  }
  st |= D.allreduce(2);
  D.stage(ST_CGXR);
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    KrylovWork *w = P->m->kw;
    const int64_t lo = P->own_lo * P->vec, n = (P->own_hi - P->own_lo) * P->vec;
    k_cg_update_p<<<grid_n(n), kThreads, 0, D.stream(p)>>>(n, w->s + lo, w->p + lo, w->sc);
    count_launch();
  }
  return st || cudaPeekAtLastError() != cudaSuccess ? B200FEM_E_CUDA : 0;
}

// ---- batches of iterations as one CUDA graph (NCCL send/recv and allreduce captured with the
// kernels; the overlap stream joins the capture through its fork/join events).  The graph is
// captured at the first inner loop of a solve and relaunched per batch and per restart; the
// host polls a device status snapshot double-buffered, as the eager loop does.  When the parts
// do not share one stream, or capture fails (an NCCL build without graph support), the solve
// falls back to enqueuing the iterations eagerly.  B200FEM_NO_GRAPH=1 forces the eager loop.
constexpr int kDistGraphBatch = 8;

struct BatchGraph {
  cudaGraphExec_t exec = nullptr;
  bool tried = false;
  int64_t launches = 0;  // library kernels per graph launch
  ~BatchGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

static bool dist_use_graph() {
  static int v = -1;
  if (v < 0) v = getenv("B200FEM_NO_GRAPH") ? 0 : 1;
  return v == 1;
}

template <class F>
static void capture_batch(Dist &D, BatchGraph &g, F &&enqueue_one) {
  g.tried = true;
  cudaStream_t s0 = D.stream(0);
  const bool trace = getenv("B200FEM_KRYLOV_TRACE") != nullptr;
  for (size_t p = 1; p < D.parts.size(); ++p)
    if (D.stream(p) != s0) {
      if (trace) fprintf(stderr, "[dist] batch graph not captured: parts on different streams\n");
      return;
    }
  // capture needs a non-default stream (the parts' stream is usually the legacy one): the body
  // is captured on a private stream (as krylov.cu run_loop_graph does), the graph runs on s0
  static thread_local cudaStream_t cs = nullptr;
  if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const int64_t l0 = g_launches.load();
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    if (trace) fprintf(stderr, "[dist] batch graph not captured: cudaStreamBeginCapture failed\n");
    return;
  }
  for (Part *P : D.parts) P->m->stream = cs;
  int st = 0;
  for (int i = 0; i < kDistGraphBatch; ++i) st |= enqueue_one();
  for (Part *P : D.parts) P->m->stream = s0;
  cudaError_t e = cudaStreamEndCapture(cs, &graph);
  g.launches = g_launches.load() - l0;
  count_launch(-(int)g.launches);  // captured, not launched
  if (st == 0 && e == cudaSuccess && graph) e = cudaGraphInstantiate(&g.exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (st || e != cudaSuccess) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    cudaGetLastError();
  }
  if (getenv("B200FEM_KRYLOV_TRACE"))
    fprintf(stderr, "[dist] batch graph %s (%d iterations, %lld launches)\n", g.exec ? "captured" : "not captured: eager",
            kDistGraphBatch, (long long)g.launches);
}

// Runs iterations until the device status leaves KS_RUNNING; `poll` is the pinned snapshot
// array (3 KrylovScalars) of part 0.  On return poll[0] holds the latest snapshot.
template <class F>
static int run_batches(Dist &D, BatchGraph &g, F &&enqueue_one, KrylovScalars *poll, b200fem_error *err) {
  KrylovWork *w0 = D.parts[0]->m->kw;
  cudaStream_t s0 = D.stream(0);
  if (dist_use_graph() && !g.tried) capture_batch(D, g, enqueue_one);
  int batch = 4, cur = 0;
  auto enqueue_batch = [&](int slot) -> int {
    if (g.exec) {
      if (cudaGraphLaunch(g.exec, s0) != cudaSuccess) return B200FEM_E_CUDA;
      count_launch((int)g.launches);
    } else {
      for (int i = 0; i < batch; ++i)
        if (int st = enqueue_one()) return st;
    }
    B200_CUDA(cudaMemcpyAsync(poll + 1 + slot, w0->sc, sizeof(KrylovScalars), cudaMemcpyDeviceToHost, s0));
    B200_CUDA(cudaEventRecord(w0->ev[slot], s0));
    return 0;
  };
  if (int st = enqueue_batch(cur)) return set_err(err, st, "Krylov iteration enqueue failed"), st;
  for (;;) {
    batch = std::min(batch * 2, 16);
    if (int st = enqueue_batch(cur ^ 1)) return set_err(err, st, "Krylov iteration enqueue failed"), st;
    B200_CUDA_E(cudaEventSynchronize(w0->ev[cur]), err);
    if (poll[1 + cur].status != KS_RUNNING) break;
    cur ^= 1;
  }
  for (size_t p = 0; p < D.parts.size(); ++p) B200_CUDA_E(cudaStreamSynchronize(D.stream(p)), err);
  *poll = poll[1 + (cur ^ 1)];  // latest snapshot (status is sticky)
  B200_CUDA_E(cudaGetLastError(), err);
  return 0;
}

// shared set-up of both distributed Krylov methods: workspaces, the local-comm result table,
// the zero-diagonal check and ||b|| / the global DOF count (collectives)
static int dist_setup(Dist &D, double *const *b, double rel_tol, double abs_tol, int64_t max_iters, double *tol,
                      int64_t *max_it, b200fem_error *err) {
  const size_t np = D.parts.size();
  int64_t n_global_owned = 0;
  for (size_t p = 0; p < np; ++p) {
    Part *P = D.parts[p];
    if (ensure_work(P->m)) return set_err(err, B200FEM_E_CUDA, "Krylov workspace allocation failed"), B200FEM_E_CUDA;
    n_global_owned += (P->own_hi - P->own_lo) * P->vec;
  }
  if (D.comm->kind == 0 && np > 1 && !D.res_dev) {
    std::vector<double *> rp(np);
    for (size_t p = 0; p < np; ++p) rp[p] = D.parts[p]->m->kw->red.result;
    B200_CUDA_E(dalloc(&D.res_dev, np), err);
    B200_CUDA_E(cudaMemcpy(D.res_dev, rp.data(), np * sizeof(double *), cudaMemcpyHostToDevice), err);
  }
  for (size_t p = 0; p < np; ++p) {  // zero-diagonal check on owned rows, summed over ranks
    KrylovWork *w = D.parts[p]->m->kw;
    if (launch_diagonal(D.parts[p]->m, w->diag, w->inv, &w->red, nullptr)) return B200FEM_E_CUDA;
  }
  if (D.allreduce(1)) return B200FEM_E_CUDA;
  double nz = 0.0, bb = 0.0;
  B200_CUDA_E(cudaMemcpyAsync(&nz, D.parts[0]->m->kw->red.result, sizeof(double), cudaMemcpyDeviceToHost, D.stream(0)), err);
  B200_CUDA_E(cudaStreamSynchronize(D.stream(0)), err);
  if (nz > 0.0) {
    set_err(err, B200FEM_E_ZERO_DIAGONAL, "zero diagonal entry; Jacobi preconditioner undefined");
    return B200FEM_E_ZERO_DIAGONAL;
  }
  if (D.dot(b, b, &bb)) return B200FEM_E_CUDA;
  *tol = std::max(rel_tol * std::sqrt(bb), abs_tol);
  if (D.comm->kind == 1) {  // global DOF count for the default max_iters = 10 N
    double cnt = (double)n_global_owned;
    double *slot = D.parts[0]->m->kw->red.result;
    B200_CUDA_E(cudaMemcpyAsync(slot, &cnt, sizeof(double), cudaMemcpyHostToDevice, D.stream(0)), err);
    if (D.allreduce(1)) return B200FEM_E_CUDA;
    B200_CUDA_E(cudaMemcpyAsync(&cnt, slot, sizeof(double), cudaMemcpyDeviceToHost, D.stream(0)), err);
    B200_CUDA_E(cudaStreamSynchronize(D.stream(0)), err);
    n_global_owned = (int64_t)cnt;
  }
  *max_it = max_iters > 0 ? max_iters : 10 * n_global_owned;
  return 0;
}

// Same control flow as the single-GPU bicgstab (krylov.cu) with the collectives inserted.
static int dist_bicgstab(Dist &D, double *const *b, double *const *x, int has_x0, double rel_tol, double abs_tol,
                         int64_t max_iters, b200fem_solve_info *info, b200fem_error *err) {
  const size_t np = D.parts.size();
  double tol = 0.0;
  int64_t max_it = 0;
  if (int st = dist_setup(D, b, rel_tol, abs_tol, max_iters, &tol, &max_it, err)) return st;
  for (size_t p = 0; p < np; ++p) {
    KrylovWork *w = D.parts[p]->m->kw;
    if (!has_x0) B200_CUDA_E(cudaMemsetAsync(x[p], 0, D.parts[p]->m->n * sizeof(double), D.stream(p)), err);
    // ghost rows of the Krylov vectors are never computed: keep them finite
    B200_CUDA_E(cudaMemsetAsync(w->v, 0, D.parts[p]->m->n * sizeof(double), D.stream(p)), err);
  }
  KrylovScalars H{};
  H.tol = tol;
  H.max_iters = max_it;
  long long it = 0, mv = 0, restarts = 0;
  double last_bd = -1.0;
  KrylovScalars *poll = D.parts[0]->m->kw->sc_host;
  BatchGraph graph;  // captured at the first inner loop, relaunched at every restart
  for (;;) {
    H.status = KS_RUNNING;
    H.first = 1;
    H.rho = H.alpha = H.omega = 1.0;
    H.it = it;
    H.mv = mv;
    for (size_t p = 0; p < np; ++p)
      B200_CUDA_E(cudaMemcpyAsync(D.parts[p]->m->kw->sc, &H, sizeof(H), cudaMemcpyHostToDevice, D.stream(p)), err);
    std::vector<SpmvArgs> ar(np);
    for (size_t p = 0; p < np; ++p) {
      KrylovWork *w = D.parts[p]->m->kw;
      ar[p] = SpmvArgs{x[p], w->r, w->inv, w->diag, b[p], w->r0, w->sc, 0};
    }
    if (D.spmv(SP_RESIDUAL, ar, x, 2)) return B200FEM_E_CUDA;
    if (D.allreduce(2)) return B200FEM_E_CUDA;
    D.stage(ST_RES);
    ++restarts;
    B200_CUDA_E(cudaMemcpyAsync(poll, D.parts[0]->m->kw->sc, sizeof(H), cudaMemcpyDeviceToHost, D.stream(0)), err);
    B200_CUDA_E(cudaStreamSynchronize(D.stream(0)), err);
    mv = poll->mv;
    const double res = poll->res;
    if (res <= tol) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, res, tol};
      return 0;
    }
    if (it >= max_it) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, res, tol};
      if (err) err->iterations = it, err->value = res;
      set_err(err, B200FEM_E_LINEAR_SOLVER, "BiCGSTAB did not converge in %lld iterations (residual %.3e, tol %.3e)",
              (long long)max_it, res, tol);
      return B200FEM_E_LINEAR_SOLVER;
    }
    for (size_t p = 0; p < np; ++p) {
      KrylovWork *w = D.parts[p]->m->kw;
      B200_CUDA_E(cudaMemsetAsync(w->p, 0, D.parts[p]->m->n * sizeof(double), D.stream(p)), err);
      B200_CUDA_E(cudaMemsetAsync(w->v, 0, D.parts[p]->m->n * sizeof(double), D.stream(p)), err);
      k_begin<<<1, 1, 0, D.stream(p)>>>(w->sc);
      count_launch();
    }
    const bool fused = dist_fused_dots(D);
    if (fused)  // the fused dot group's scratch, allocated before any capture (no cudaMalloc inside one)
      for (Part *P : D.parts)
        if (!P->red6.partials && red_alloc(&P->red6)) return set_err(err, B200FEM_E_CUDA, "reduction scratch"), B200FEM_E_CUDA;
    (void)xr_blocks();  // occupancy queries of the reducing updates, outside the capture too
    if (fused) (void)dot6_blocks();
    if (int st = run_batches(D, graph, [&] { return fused ? enqueue_dist_iteration_fused(D, x)
                                                           : enqueue_dist_iteration(D, x); }, poll, err))
      return st;
    it = poll->it;
    mv = poll->mv;
    if (poll->status == KS_BREAKDOWN) {
      if (last_bd >= 0.0 && poll->res >= 0.999 * last_bd) {
        if (info) *info = b200fem_solve_info{it, mv, restarts, poll->res, tol};
        if (err) err->iterations = it, err->value = poll->res;
        set_err(err, B200FEM_E_BREAKDOWN, "BiCGSTAB breakdown without progress at iteration %lld (residual %.3e)", it,
                poll->res);
        return B200FEM_E_BREAKDOWN;
      }
      last_bd = poll->res;
    }
  }
}

// Jacobi-PCG over the parts: the single-GPU pcg (krylov.cu) with the collectives inserted.
static int dist_pcg(Dist &D, double *const *b, double *const *x, int has_x0, double rel_tol, double abs_tol,
                    int64_t max_iters, b200fem_solve_info *info, b200fem_error *err) {
  const size_t np = D.parts.size();
  double tol = 0.0;
  int64_t max_it = 0;
  if (int st = dist_setup(D, b, rel_tol, abs_tol, max_iters, &tol, &max_it, err)) return st;
  for (size_t p = 0; p < np; ++p) {
    Matrix *m = D.parts[p]->m;
    KrylovWork *w = m->kw;
    if (!has_x0) B200_CUDA_E(cudaMemsetAsync(x[p], 0, m->n * sizeof(double), D.stream(p)), err);
    B200_CUDA_E(cudaMemsetAsync(w->v, 0, m->n * sizeof(double), D.stream(p)), err);
    B200_CUDA_E(cudaMemsetAsync(w->p, 0, m->n * sizeof(double), D.stream(p)), err);
    if (m->n_dir) {  // x_d = b_d: the Krylov space then lives on the free rows (krylov.cu pcg)
      k_set_dirichlet<<<grid_n(m->n_dir), kThreads, 0, D.stream(p)>>>(x[p], b[p], m->dir_dofs, m->n_dir);
      count_launch();
    }
  }
  KrylovScalars H{};
  H.tol = tol;
  H.max_iters = max_it;
  long long it = 0, mv = 0, restarts = 0;
  KrylovScalars *poll = D.parts[0]->m->kw->sc_host;
  BatchGraph graph;
  for (;;) {
    H.status = KS_RUNNING;
    H.it = it;
    H.mv = mv;
    for (size_t p = 0; p < np; ++p)
      B200_CUDA_E(cudaMemcpyAsync(D.parts[p]->m->kw->sc, &H, sizeof(H), cudaMemcpyHostToDevice, D.stream(p)), err);
    std::vector<SpmvArgs> ar(np);
    for (size_t p = 0; p < np; ++p) {
      KrylovWork *w = D.parts[p]->m->kw;
      ar[p] = SpmvArgs{x[p], w->r, w->inv, w->diag, b[p], w->p, w->sc, 0};  // r = b - A x, p = D^-1 r
    }
    if (D.spmv(SP_CGRES, ar, x, 2)) return B200FEM_E_CUDA;
    if (D.allreduce(2)) return B200FEM_E_CUDA;
    D.stage(ST_CGRES);
    ++restarts;
    B200_CUDA_E(cudaMemcpyAsync(poll, D.parts[0]->m->kw->sc, sizeof(H), cudaMemcpyDeviceToHost, D.stream(0)), err);
    B200_CUDA_E(cudaStreamSynchronize(D.stream(0)), err);
    mv = poll->mv;
    const double res = poll->res;
    if (res <= tol) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, res, tol};
      return 0;
    }
    if (it >= max_it) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, res, tol};
      if (err) err->iterations = it, err->value = res;
      set_err(err, B200FEM_E_LINEAR_SOLVER, "PCG did not converge in %lld iterations (residual %.3e, tol %.3e)",
              (long long)max_it, res, tol);
      return B200FEM_E_LINEAR_SOLVER;
    }
    for (size_t p = 0; p < np; ++p) {
      k_begin_cg<<<1, 1, 0, D.stream(p)>>>(D.parts[p]->m->kw->sc);
      count_launch();
    }
    if (int st = run_batches(D, graph, [&] { return enqueue_dist_cg_iteration(D, x); }, poll, err)) return st;
    it = poll->it;
    mv = poll->mv;
    if (poll->status == KS_BREAKDOWN) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, poll->res, tol};
      if (err) err->iterations = it, err->value = poll->res;
      set_err(err, B200FEM_E_BREAKDOWN, "PCG breakdown at iteration %lld: p.Ap = %.3e <= 0 (operator not SPD)", it,
              poll->r0v);
      return B200FEM_E_BREAKDOWN;
    }
  }
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_comm_unique_id(uint8_t *out) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return B200FEM_E_CUDA;
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int b200fem_comm_create_nccl(b200fem_comm **out, const uint8_t *id_bytes, int32_t nranks, int32_t rank) {
  ncclUniqueId id;
  memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
  Comm *c = new Comm();
  c->kind = 1;
  c->rank = rank;
  c->nranks = nranks;
  if (ncclCommInitRank(&c->nccl, nranks, id, rank) != ncclSuccess) {
    delete c;
    return B200FEM_E_CUDA;
  }
  *out = (b200fem_comm *)c;
  return 0;
}

int b200fem_comm_create_local(b200fem_comm **out) {
  Comm *c = new Comm();
  c->kind = 0;
  *out = (b200fem_comm *)c;
  return 0;
}

int b200fem_comm_destroy(b200fem_comm *cc) {
  Comm *c = (Comm *)cc;
  if (!c) return 0;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return 0;
}

int b200fem_part_create(b200fem_part **out, b200fem_matrix *local, int64_t own_node_lo, int64_t own_node_hi,
                        int32_t n_peers, const int32_t *peers, const int64_t *send_counts, const int32_t *send_nodes,
                        const int64_t *recv_counts, const int32_t *recv_nodes) {
  Matrix *m = (Matrix *)local;
  if (!out || !m || own_node_lo < 0 || own_node_hi < own_node_lo) return B200FEM_E_INVALID;
  Part *P = new Part();
  P->m = m;
  P->vec = m->kind == MK_CSR ? 1 : m->kind == MK_GRID3 ? m->gvec : 3;
  P->own_lo = own_node_lo;
  P->own_hi = own_node_hi;
  m->row_lo = own_node_lo;  // node range (FEM3/SYM3) == row range (vec-1 CSR)
  m->row_hi = own_node_hi;
  if (m->kind == MK_GRID3 && m->gvec == 3 && !getenv("B200FEM_NO_OVERLAP")) {
    const int64_t margin = (int64_t)m->gnx * m->gny + m->gnx + 1;  // largest lattice offset
    P->int_lo = own_node_lo + margin;
    P->int_hi = own_node_hi - margin;
    if (P->int_hi > P->int_lo && n_peers > 0) {
      if (cudaStreamCreateWithFlags(&P->s2, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&P->ev_in, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&P->ev_done, cudaEventDisableTiming) != cudaSuccess || red_alloc(&P->red_in) ||
          red_alloc(&P->red_lo) || red_alloc(&P->red_hi)) {
        delete P;
        return B200FEM_E_CUDA;
      }
      P->overlap = true;
    }
  }
  if (m->kind == MK_FEM3 && m->use_tma) {  // bulk-copy chunks over the owned nodes only
    if (prepare_fem3_chunks(m, own_node_lo, own_node_hi)) {
      delete P;
      return B200FEM_E_CUDA;
    }
  } else {
    m->use_tma = false;
  }
  P->n_peers = n_peers;
  P->peer.assign(peers, peers + n_peers);
  P->soff.assign(n_peers + 1, 0);
  P->roff.assign(n_peers + 1, 0);
  for (int i = 0; i < n_peers; ++i) {
    P->soff[i + 1] = P->soff[i] + send_counts[i];
    P->roff[i + 1] = P->roff[i] + recv_counts[i];
  }
  const int64_t ns = P->soff.back(), nr = P->roff.back();
  if (dalloc(&P->send_nodes, ns) || dalloc(&P->recv_nodes, nr) || dalloc(&P->sendbuf, ns * P->vec) ||
      dalloc(&P->recvbuf, nr * P->vec)) {
    delete P;
    return B200FEM_E_CUDA;
  }
  if (ns) cudaMemcpy(P->send_nodes, send_nodes, ns * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (nr) cudaMemcpy(P->recv_nodes, recv_nodes, nr * sizeof(int32_t), cudaMemcpyHostToDevice);
  // contiguous halo lists (checked on the host lists)
  auto run = [](const int32_t *v, int64_t lo, int64_t hi) {
    for (int64_t t = lo + 1; t < hi; ++t)
      if (v[t] != v[t - 1] + 1) return false;
    return true;
  };
  P->contiguous = !getenv("B200FEM_HALO_PACK");
  for (int i = 0; i < n_peers && P->contiguous; ++i)
    P->contiguous = run(send_nodes, P->soff[i], P->soff[i + 1]) && run(recv_nodes, P->roff[i], P->roff[i + 1]);
  if (P->contiguous)
    for (int i = 0; i < n_peers; ++i) {
      P->s_lo.push_back(P->soff[i + 1] > P->soff[i] ? send_nodes[P->soff[i]] : 0);
      P->r_lo.push_back(P->roff[i + 1] > P->roff[i] ? recv_nodes[P->roff[i]] : 0);
    }
  *out = (b200fem_part *)P;
  return 0;
}

int b200fem_part_destroy(b200fem_part *pp) {
  Part *P = (Part *)pp;
  if (!P) return 0;
  cudaFree(P->send_nodes);
  cudaFree(P->recv_nodes);
  cudaFree(P->sendbuf);
  cudaFree(P->recvbuf);
  if (P->red6.partials) red_free(&P->red6);
  if (P->overlap) {
    cudaStreamSynchronize(P->s2);
    cudaStreamDestroy(P->s2);
    cudaEventDestroy(P->ev_in);
    cudaEventDestroy(P->ev_done);
    red_free(&P->red_in);
    red_free(&P->red_lo);
    red_free(&P->red_hi);
  }
  if (P->m) {
    P->m->row_lo = 0, P->m->row_hi = -1;
    if (P->m->use_tma) prepare_fem3_chunks(P->m);
  }
  delete P;
  return 0;
}

static Dist make_dist(b200fem_part **parts, int32_t np, b200fem_comm *comm) {
  Dist D;
  for (int i = 0; i < np; ++i) D.parts.push_back((Part *)parts[i]);
  D.comm = (Comm *)comm;
  return D;
}

int b200fem_dist_bicgstab(b200fem_part **parts, int32_t np, b200fem_comm *comm, double *const *b, double *const *x,
                          int32_t has_x0, double rel_tol, double abs_tol, int64_t max_iters, b200fem_solve_info *info,
                          b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (info) memset(info, 0, sizeof(*info));
  if (np < 1 || !comm || (((Comm *)comm)->kind == 1 && np != 1)) return B200FEM_E_INVALID;
  if (!(rel_tol > 0) || !(abs_tol > 0)) {
    set_err(err, B200FEM_E_INVALID, "linear solver tolerances must be positive");
    return B200FEM_E_INVALID;
  }
  Dist D = make_dist(parts, np, comm);
  const int st = dist_bicgstab(D, b, x, has_x0, rel_tol, abs_tol, max_iters, info, err);
  cudaFree(D.res_dev);
  return st;
}

int b200fem_dist_pcg(b200fem_part **parts, int32_t np, b200fem_comm *comm, double *const *b, double *const *x,
                     int32_t has_x0, double rel_tol, double abs_tol, int64_t max_iters, b200fem_solve_info *info,
                     b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (info) memset(info, 0, sizeof(*info));
  if (np < 1 || !comm || (((Comm *)comm)->kind == 1 && np != 1)) return B200FEM_E_INVALID;
  if (!(rel_tol > 0) || !(abs_tol > 0)) {
    set_err(err, B200FEM_E_INVALID, "linear solver tolerances must be positive");
    return B200FEM_E_INVALID;
  }
  Dist D = make_dist(parts, np, comm);
  const int st = dist_pcg(D, b, x, has_x0, rel_tol, abs_tol, max_iters, info, err);
  cudaFree(D.res_dev);
  return st;
}

int b200fem_dist_halo(b200fem_part **parts, int32_t np, b200fem_comm *comm, double *const *vec) {
  Dist D = make_dist(parts, np, comm);
  return D.halo(vec);
}

int b200fem_dist_dot(b200fem_part **parts, int32_t np, b200fem_comm *comm, double *const *x, double *const *y,
                     double *out_host) {
  Dist D = make_dist(parts, np, comm);
  for (int p = 0; p < np; ++p)
    if (ensure_work(D.parts[p]->m)) return B200FEM_E_CUDA;
  if (D.comm->kind == 0 && np > 1) {
    std::vector<double *> rp(np);
    for (int p = 0; p < np; ++p) rp[p] = D.parts[p]->m->kw->red.result;
    B200_CUDA(dalloc(&D.res_dev, np));
    B200_CUDA(cudaMemcpy(D.res_dev, rp.data(), np * sizeof(double *), cudaMemcpyHostToDevice));
  }
  const int st = D.dot(x, y, out_host);
  cudaFree(D.res_dev);
  return st;
}

int b200fem_comm_allreduce(b200fem_comm *comm, double *buf_dev, int64_t n, void *stream) {
  Comm *c = (Comm *)comm;
  if (c->kind != 1) return 0;
  if (ncclAllReduce(buf_dev, buf_dev, n, ncclDouble, ncclSum, c->nccl, (cudaStream_t)stream) != ncclSuccess)
    return B200FEM_E_CUDA;
  return 0;
}

}  // extern "C"
