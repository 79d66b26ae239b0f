// Jacobi-preconditioned BiCGSTAB with the reference's exact control flow
// (solvers.py:87-167), run on the device: all recurrence scalars (rho, alpha, omega,
// beta, the iteration counter and the status) live in device memory and are updated by
// the last block of each reduction, so the host never waits inside the inner loop.  The
// inner loop is one CUDA-graph WHILE node per (re)start (run_loop_graph; B200FEM_NO_GRAPH=1:
// batches of iterations with double-buffered status polling); the host C++ loop reproduces
// the outer restart loop: explicit residual check, LinearSolverError at max_iters, restart
// on breakdown, BreakdownError when a restart makes no progress.
//
// Per iteration (5 launches):
//   K_a  p = r + beta (p - omega v)                                      (solvers.py:140)
//   K_b  v = D^-1 A p  (+ r0.v -> alpha, breakdown if 0)                  (141-143, 158)
//   K_c  s = r - alpha v                                                  (159)
//   K_d  t = D^-1 A s  (+ t.t, t.s -> omega)                              (160-162)
//   K_e  x += alpha p + omega s ; r = s - omega t (+ ||D r||, r0.r, r.r)  (163-165)
//        last block: convergence test, then the next iteration's start:
//        it += 1, rho_new = r0.r, breakdown test, beta                   (131-139)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace b200 {

__global__ void k_begin_cg(KrylovScalars *S) {
  if (S->status != KS_RUNNING) return;
  if (S->it >= S->max_iters) S->status = KS_MAXED;
  else S->it += 1;
}

__global__ void k_begin(KrylovScalars *S) {
  if (S->status == KS_RUNNING) iter_start(S);
}

__global__ void __launch_bounds__(kThreads) k_update_p(int64_t n, const double *__restrict__ r,
                                                       const double *__restrict__ v, double *__restrict__ p,
                                                       const KrylovScalars *S) {
  if (S->status != KS_RUNNING) return;
  const double beta = S->beta, omega = S->omega;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = r[i] + beta * (p[i] - omega * v[i]);
}

__global__ void __launch_bounds__(kThreads) k_update_s(int64_t n, const double *__restrict__ r,
                                                       const double *__restrict__ v, double *__restrict__ s,
                                                       const KrylovScalars *S) {
  if (S->status != KS_RUNNING) return;
  const double alpha = S->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s[i] = r[i] - alpha * v[i];
}

__global__ void __launch_bounds__(kThreads) k_update_xr(int64_t n, double *__restrict__ x, double *__restrict__ r,
                                                        const double *__restrict__ p, const double *__restrict__ s,
                                                        const double *__restrict__ t, const double *__restrict__ r0,
                                                        const double *__restrict__ dg, KrylovScalars *S,
                                                        RedScratch red, int inline_stage) {
  if (S->status != KS_RUNNING) return;
  const double alpha = S->alpha, omega = S->omega;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i] + omega * s[i];
    const double ri = s[i] - omega * t[i];
    r[i] = ri;
    const double dr = dg[i] * ri;
    acc[0] = fma(dr, dr, acc[0]);
    acc[1] = fma(r0[i], ri, acc[1]);
    acc[2] = fma(ri, ri, acc[2]);
  }
  double tot[3];
  if (block_partials_and_finish<3>(acc, red, tot) && threadIdx.x == 0 && inline_stage) apply_stage(ST_XR, S, tot);
}

// ---------------------------------------------------------------- Jacobi-PCG
// For symmetric operators (Poisson, LE, NH, SIMP, J2 tangents; BASELINE config 2 "linear
// assembly + PCG").  The Dirichlet rows of the assembled K are identity rows, so starting
// from x_d = b_d keeps r_d = z_d = p_d = 0 and the row-replaced K acts on the Krylov space
// as the SPD block K_ff (the lifting K_fd x_d enters through the first residual).
__global__ void k_set_dirichlet(double *__restrict__ x, const double *__restrict__ b, const int32_t *__restrict__ d,
                                int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[d[i]] = b[d[i]];
}

__global__ void __launch_bounds__(kThreads) k_cg_update_xrz(int64_t n, double *__restrict__ x, double *__restrict__ r,
                                                            const double *__restrict__ p, const double *__restrict__ q,
                                                            const double *__restrict__ inv, double *__restrict__ z,
                                                            KrylovScalars *S, RedScratch red, int inline_stage) {
  if (S->status != KS_RUNNING) return;
  const double alpha = S->alpha;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    const double zi = inv[i] * ri;
    z[i] = zi;
    acc[0] = fma(ri, ri, acc[0]);
    acc[1] = fma(ri, zi, acc[1]);
  }
  double tot[2];
  if (block_partials_and_finish<2>(acc, red, tot) && threadIdx.x == 0 && inline_stage) apply_stage(ST_CGXR, S, tot);
}

__global__ void __launch_bounds__(kThreads) k_cg_update_p(int64_t n, const double *__restrict__ z,
                                                          double *__restrict__ p, const KrylovScalars *S) {
  if (S->status != KS_RUNNING) return;
  const double beta = S->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

int ensure_work(Matrix *m) {
  if (m->kw) return 0;
  KrylovWork *w = new KrylovWork();
  w->n = m->n;
  double **vecs[] = {&w->r, &w->r0, &w->p, &w->v, &w->s, &w->t, &w->diag, &w->inv};
  for (double **v : vecs) B200_CUDA(dalloc(v, m->n));
  B200_CUDA(dalloc(&w->sc, 1));
  B200_CUDA(cudaMallocHost((void **)&w->sc_host, 3 * sizeof(KrylovScalars)));
  if (red_alloc(&w->red)) return B200FEM_E_CUDA;
  B200_CUDA(cudaEventCreateWithFlags(&w->ev[0], cudaEventDisableTiming));
  B200_CUDA(cudaEventCreateWithFlags(&w->ev[1], cudaEventDisableTiming));
  m->kw = w;
  return 0;
}

void free_work(KrylovWork *w) {
  if (!w) return;
  double *vecs[] = {w->r, w->r0, w->p, w->v, w->s, w->t, w->diag, w->inv};
  for (double *v : vecs) cudaFree(v);
  cudaFree(w->sc);
  cudaFreeHost(w->sc_host);
  red_free(&w->red);
  cudaEventDestroy(w->ev[0]);
  cudaEventDestroy(w->ev[1]);
  delete w;
}


// ------------------------------------------------------------ device-side Krylov loop
// The iterations run as a CUDA graph WHILE node: its body is one captured iteration plus a
// one-thread kernel that keeps the loop going while the device-side status is RUNNING.
// Convergence, breakdown and max_iters are decided by the scalar stages on the device, so
// the host launches one graph per (re)start and waits once -- no polling batches, and no
// no-op launches after convergence (the batched loop enqueues up to 64 extra iterations).
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const KrylovScalars *S) {
  cudaGraphSetConditional(h, S->status == KS_RUNNING ? 1u : 0u);
}

__global__ void k_loop_status(const KrylovScalars *S) {
  if (S->status == 12345) __trap();  // same single-thread read of the status as k_loop_cond
}

static bool use_graph_loop() {
  static int v = -1;
  if (v < 0) v = getenv("B200FEM_NO_GRAPH") ? 0 : 1;
  return v == 1;
}

// The while-graph of `enqueue` is built once per solve (x and b differ between calls) and
// relaunched on the matrix's stream at every (re)start of that solve: restart-heavy solves
// (BiCGSTAB breakdowns near the round-off floor) do not pay a graph instantiation per restart.
struct LoopGraph {
  cudaGraphExec_t exec = nullptr;
  ~LoopGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

template <class F>
static int run_loop_graph(Matrix *m, LoopGraph &lg, F &&enqueue, b200fem_error *err) {
  KrylovWork *w = m->kw;
  cudaStream_t s = m->stream;
  cudaError_t e = cudaSuccess;
  const char *where = "cudaGraphLaunch";
  if (!lg.exec) {
    // capture needs a non-default stream (the caller's may be the legacy stream): the body is
    // captured on a private stream, the graph then runs on the matrix's stream
    static thread_local cudaStream_t cs = nullptr;
    if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_status(cudaGetLastError(), err, "capture stream");
    cudaGraph_t g = nullptr;
    cudaGraphConditionalHandle h;
    do {
      where = "cudaGraphCreate";
      if ((e = cudaGraphCreate(&g, 0)) != cudaSuccess) break;
      where = "cudaGraphConditionalHandleCreate";
      if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) break;
      cudaGraphNodeParams np{};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = h;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      where = "cudaGraphAddNode(while)";
      if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &np)) != cudaSuccess) break;
      cudaGraph_t body = np.conditional.phGraph_out[0];
      where = "cudaStreamBeginCaptureToGraph";
      if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) !=
          cudaSuccess)
        break;
      m->stream = cs;
      enqueue();
      k_loop_cond<<<1, 1, 0, cs>>>(h, w->sc);
      m->stream = s;
      cudaGraph_t cap = nullptr;
      where = "cudaStreamEndCapture";
      if ((e = cudaStreamEndCapture(cs, &cap)) != cudaSuccess) break;
      where = "cudaGraphInstantiate";
      if ((e = cudaGraphInstantiate(&lg.exec, g, 0)) != cudaSuccess) break;
    } while (false);
    m->stream = s;
    if (g) cudaGraphDestroy(g);
  }
  if (e == cudaSuccess) {
    where = "cudaGraphLaunch";
    e = cudaGraphLaunch(lg.exec, s);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_err(err, B200FEM_E_CUDA, "Krylov while-graph: %s failed: %s", where, cudaGetErrorString(e));
    return B200FEM_E_CUDA;
  }
  return 0;
}

static int grid_vec(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + kThreads - 1) / kThreads)); }

// Blocks of the reducing vector updates: one full wave.  k_update_xr needs 48 registers, so
// 5 of its 256-thread blocks fit an SM; kRedBlocks (8 per SM) would run as a full wave plus a
// 60 % one.  B200FEM_XR_BLOCKS=<n> overrides (<= kRedBlocks; the A/B switch).
template <class K>
static int wave_blocks(K kernel) {
  int nb = 0, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, 0) != cudaSuccess || nb <= 0) {
    cudaGetLastError();
    return kRedBlocks;
  }
  return std::min(kRedBlocks, nb * sms);
}
int xr_blocks() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("B200FEM_XR_BLOCKS");
    v = e && atoi(e) > 0 ? std::min(atoi(e), kRedBlocks) : wave_blocks(k_update_xr);
  }
  return v;
}

static void enqueue_iteration(Matrix *m, const double *b, double *x) {
  KrylovWork *w = m->kw;
  cudaStream_t s = m->stream;
  const int64_t n = m->n;
  k_update_p<<<grid_vec(n), kThreads, 0, s>>>(n, w->r, w->v, w->p, w->sc);
  SpmvArgs a1{w->p, w->v, w->inv, w->diag, w->r0, nullptr, w->sc, 1};
  launch_spmv(m, SP_JACOBI_R0, a1, &w->red);
  k_update_s<<<grid_vec(n), kThreads, 0, s>>>(n, w->r, w->v, w->s, w->sc);
  SpmvArgs a2{w->s, w->t, w->inv, w->diag, nullptr, nullptr, w->sc, 1};
  launch_spmv(m, SP_JACOBI_TT, a2, &w->red);
  k_update_xr<<<xr_blocks(), kThreads, 0, s>>>(n, x, w->r, w->p, w->s, w->t, w->r0, w->diag, w->sc, w->red, 1);
  count_launch(3);
  (void)b;
}

// Diagnostics (bench.py "krylov_profile"): one BiCGSTAB iteration of `m` as it runs inside the
// while-graph, against its kernels timed one by one (CUDA events on the matrix's stream).
// out_us[0] = graph-loop time per iteration (`iters` iterations, tolerance 0), out_us[1..6] =
// k_update_p, SpMV (v = D^-1 A p, r0.v), k_update_s, SpMV (t = D^-1 A s, t.t, t.s),
// k_update_xr, k_loop_cond, each averaged over `iters` back-to-back launches; out_us[7] = sum.
static int bicgstab_profile(Matrix *m, const double *b, double *x, int iters, double *out_us) {
  if (ensure_work(m)) return B200FEM_E_CUDA;
  KrylovWork *w = m->kw;
  cudaStream_t s = m->stream;
  const int64_t n = m->n;
  int64_t nz = 0;
  if (launch_diagonal(m, w->diag, w->inv, &w->red, &nz) || nz) return B200FEM_E_INVALID;
  B200_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  KrylovScalars H{};
  H.status = KS_RUNNING;
  H.first = 1;
  H.rho = H.alpha = H.omega = 1.0;
  H.tol = 0.0;
  H.max_iters = iters;
  B200_CUDA(cudaMemcpyAsync(w->sc, &H, sizeof(H), cudaMemcpyHostToDevice, s));
  SpmvArgs ar{x, w->r, w->inv, w->diag, b, w->r0, w->sc, 1};
  if (launch_spmv(m, SP_RESIDUAL, ar, &w->red)) return B200FEM_E_CUDA;
  B200_CUDA(cudaMemsetAsync(w->v, 0, n * sizeof(double), s));
  B200_CUDA(cudaMemsetAsync(w->p, 0, n * sizeof(double), s));
  k_begin<<<1, 1, 0, s>>>(w->sc);
  cudaEvent_t e0, e1;
  B200_CUDA(cudaEventCreate(&e0));
  B200_CUDA(cudaEventCreate(&e1));
  int rc = 0;
  {
    LoopGraph lg;
    b200fem_error err{};
    B200_CUDA(cudaEventRecord(e0, s));
    rc = run_loop_graph(m, lg, [&] { enqueue_iteration(m, b, x); }, &err);
    B200_CUDA(cudaEventRecord(e1, s));
    B200_CUDA(cudaEventSynchronize(e1));
  }
  KrylovScalars done{};
  B200_CUDA(cudaMemcpy(&done, w->sc, sizeof(done), cudaMemcpyDeviceToHost));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  out_us[0] = 1e3 * ms / std::max<long long>(done.it, 1);
  // kernels one at a time (status forced RUNNING, no iteration cap)
  H = done;
  H.status = KS_RUNNING;
  H.max_iters = 1ll << 60;
  B200_CUDA(cudaMemcpyAsync(w->sc, &H, sizeof(H), cudaMemcpyHostToDevice, s));
  SpmvArgs a1{w->p, w->v, w->inv, w->diag, w->r0, nullptr, w->sc, 1};
  SpmvArgs a2{w->s, w->t, w->inv, w->diag, nullptr, nullptr, w->sc, 1};
  for (int k = 1; k <= 6 && !rc; ++k) {
    B200_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < iters; ++i) {
      switch (k) {
        case 1: k_update_p<<<grid_vec(n), kThreads, 0, s>>>(n, w->r, w->v, w->p, w->sc); break;
        case 2: rc |= launch_spmv(m, SP_JACOBI_R0, a1, &w->red); break;
        case 3: k_update_s<<<grid_vec(n), kThreads, 0, s>>>(n, w->r, w->v, w->s, w->sc); break;
        case 4: rc |= launch_spmv(m, SP_JACOBI_TT, a2, &w->red); break;
        case 5:
          k_update_xr<<<xr_blocks(), kThreads, 0, s>>>(n, x, w->r, w->p, w->s, w->t, w->r0, w->diag, w->sc, w->red, 1);
          break;
        default: k_loop_status<<<1, 1, 0, s>>>(w->sc); break;
      }
    }
    B200_CUDA(cudaEventRecord(e1, s));
    B200_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    out_us[k] = 1e3 * ms / iters;
    // keep the recurrence alive (a breakdown would gate the kernels off)
    B200_CUDA(cudaMemcpyAsync(w->sc, &H, sizeof(H), cudaMemcpyHostToDevice, s));
  }
  out_us[7] = out_us[1] + out_us[2] + out_us[3] + out_us[4] + out_us[5] + out_us[6];
  count_launch(6 * iters + 2);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc ? B200FEM_E_CUDA : 0;
}

// B200FEM_KRYLOV_TRACE=1: host timeline of each BiCGSTAB solve on stderr (setup, every
// restart's explicit residual, every inner loop), for attributing solve time outside the loop.
static bool krylov_trace() {
  static int v = -1;
  if (v < 0) v = getenv("B200FEM_KRYLOV_TRACE") ? 1 : 0;
  return v == 1;
}
static double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int bicgstab(Matrix *m, const double *b, double *x, int has_x0, double rel_tol, double abs_tol, int64_t max_iters,
             b200fem_solve_info *info, b200fem_error *err) {
  const bool trace = krylov_trace();
  const double t_start = trace ? host_ms() : 0.0;
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (info) memset(info, 0, sizeof(*info));
  if (!(rel_tol > 0) || !(abs_tol > 0)) {
    set_err(err, B200FEM_E_INVALID, "linear solver tolerances must be positive");
    return B200FEM_E_INVALID;
  }
  int st = ensure_work(m);
  if (st) return set_err(err, st, "Krylov workspace allocation failed"), st;
  KrylovWork *w = m->kw;
  cudaStream_t s = m->stream;
  const int64_t n = m->n;
  int64_t nzero = 0;
  st = launch_diagonal(m, w->diag, w->inv, &w->red, &nzero);
  if (st) return set_err(err, st, "diagonal extraction failed"), st;
  if (nzero) {
    set_err(err, B200FEM_E_ZERO_DIAGONAL, "zero diagonal entry; Jacobi preconditioner undefined");
    return B200FEM_E_ZERO_DIAGONAL;
  }
  if (!has_x0) B200_CUDA_E(cudaMemsetAsync(x, 0, n * sizeof(double), s), err);
  if (launch_dot(b, b, n, &w->red, s)) return B200FEM_E_CUDA;
  double bb = 0.0;
  B200_CUDA_E(cudaMemcpyAsync(&bb, w->red.result, sizeof(double), cudaMemcpyDeviceToHost, s), err);
  B200_CUDA_E(cudaStreamSynchronize(s), err);
  const double tol = std::max(rel_tol * std::sqrt(bb), abs_tol);
  const int64_t max_it = max_iters > 0 ? max_iters : 10 * n;
  if (trace) fprintf(stderr, "[krylov] setup (diagonal, ||b||, sync) %.3f ms\n", host_ms() - t_start);

  KrylovScalars *H = w->sc_host;  // [0] control, [1],[2] poll buffers
  memset(H, 0, 3 * sizeof(KrylovScalars));
  H[0].tol = tol;
  H[0].max_iters = max_it;
  long long it = 0, mv = 0, restarts = 0;
  double last_bd = -1.0;
  const size_t ssz = sizeof(KrylovScalars);
  LoopGraph loop_graph;  // built at the first inner loop, relaunched at every restart
  for (;;) {
    // ---- (re)start: r = D^-1 (b - A x), r0 = r, res = ||D r||   (solvers.py:115-118)
    H[0].status = KS_RUNNING;
    H[0].first = 1;
    H[0].rho = H[0].alpha = H[0].omega = 1.0;
    H[0].it = it;
    H[0].mv = mv;
    B200_CUDA_E(cudaMemcpyAsync(w->sc, &H[0], ssz, cudaMemcpyHostToDevice, s), err);
    SpmvArgs ar{x, w->r, w->inv, w->diag, b, w->r0, w->sc, 1};
    const double t_res = trace ? host_ms() : 0.0;
    if (launch_spmv(m, SP_RESIDUAL, ar, &w->red)) return B200FEM_E_CUDA;
    ++restarts;
    B200_CUDA_E(cudaMemcpyAsync(&H[1], w->sc, ssz, cudaMemcpyDeviceToHost, s), err);
    B200_CUDA_E(cudaStreamSynchronize(s), err);
    mv = H[1].mv;
    const double res = H[1].res;
    if (trace)
      fprintf(stderr, "[krylov] restart %lld: explicit residual %.3e (tol %.3e) %.3f ms, total %.3f ms\n", restarts, res,
              tol, host_ms() - t_res, host_ms() - t_start);
    if (res <= tol) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, res, tol};
      return 0;
    }
    if (it >= max_it) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, res, tol};
      if (err) {
        err->iterations = it;
        err->value = res;
      }
      set_err(err, B200FEM_E_LINEAR_SOLVER, "BiCGSTAB did not converge in %lld iterations (residual %.3e, tol %.3e)",
              (long long)max_it, res, tol);
      return B200FEM_E_LINEAR_SOLVER;
    }
    B200_CUDA_E(cudaMemsetAsync(w->v, 0, n * sizeof(double), s), err);
    B200_CUDA_E(cudaMemsetAsync(w->p, 0, n * sizeof(double), s), err);
    k_begin<<<1, 1, 0, s>>>(w->sc);
    count_launch();
    // ---- inner loop: a device-side while-graph, or batches with double-buffered polling
    int cur = 0;
    KrylovScalars done{};
    if (use_graph_loop()) {
      const long long it0 = it;
      const double t_loop = trace ? host_ms() : 0.0;
      const bool built = loop_graph.exec != nullptr;
      if (int rc = run_loop_graph(m, loop_graph, [&] { enqueue_iteration(m, b, x); }, err)) return rc;
      const double t_launched = trace ? host_ms() : 0.0;
      B200_CUDA_E(cudaMemcpyAsync(&H[1], w->sc, ssz, cudaMemcpyDeviceToHost, s), err);
      B200_CUDA_E(cudaStreamSynchronize(s), err);
      count_launch(5 * (H[1].it - it0) + 1);
      if (trace)
        fprintf(stderr, "[krylov] loop: %lld iterations, status %d, %s+launch %.3f ms, run %.3f ms (%.1f us/it)\n",
                (long long)(H[1].it - it0), (int)H[1].status, built ? "relaunch" : "capture+instantiate",
                t_launched - t_loop, host_ms() - t_launched,
                1e3 * (host_ms() - t_launched) / std::max<long long>(1, H[1].it - it0));
      cur = 1;  // the snapshot is in H[1 + (cur ^ 1)]
    } else {
      int batch = 4;
      auto enqueue_batch = [&](int slot) -> int {
        for (int i = 0; i < batch; ++i) enqueue_iteration(m, b, x);
        B200_CUDA_E(cudaMemcpyAsync(&H[1 + slot], w->sc, ssz, cudaMemcpyDeviceToHost, s), err);
        B200_CUDA_E(cudaEventRecord(w->ev[slot], s), err);
        return 0;
      };
      if (enqueue_batch(cur)) return B200FEM_E_CUDA;
      for (;;) {
        batch = std::min(batch * 2, 32);
        if (enqueue_batch(cur ^ 1)) return B200FEM_E_CUDA;
        B200_CUDA_E(cudaEventSynchronize(w->ev[cur]), err);
        if (H[1 + cur].status != KS_RUNNING) break;
        cur ^= 1;
      }
      B200_CUDA_E(cudaStreamSynchronize(s), err);  // drain the no-op batch
    }
    done = H[1 + (cur ^ 1)];                     // latest snapshot (status is sticky)
    it = done.it;
    mv = done.mv;
    B200_CUDA_E(cudaGetLastError(), err);
    if (done.status == KS_BREAKDOWN) {
      // shadow residual went orthogonal: restart from the explicit residual unless the
      // previous restart made no progress (solvers.py:144-157)
      if (last_bd >= 0.0 && done.res >= 0.999 * last_bd) {
        if (info) *info = b200fem_solve_info{it, mv, restarts, done.res, tol};
        if (err) {
          err->iterations = it;
          err->value = done.res;
        }
        set_err(err, B200FEM_E_BREAKDOWN, "BiCGSTAB breakdown without progress at iteration %lld (residual %.3e)",
                it, done.res);
        return B200FEM_E_BREAKDOWN;
      }
      last_bd = done.res;
    }
    // KS_CONV_INNER / KS_MAXED / restart: back to the explicit residual check
  }
}

static void enqueue_cg_iteration(Matrix *m, double *x) {
  KrylovWork *w = m->kw;
  cudaStream_t s = m->stream;
  const int64_t n = m->n;
  SpmvArgs a{w->p, w->v, w->inv, w->diag, nullptr, nullptr, w->sc, 1};
  launch_spmv(m, SP_PQ, a, &w->red);
  k_cg_update_xrz<<<kRedBlocks, kThreads, 0, s>>>(n, x, w->r, w->p, w->v, w->inv, w->s, w->sc, w->red, 1);
  k_cg_update_p<<<grid_vec(n), kThreads, 0, s>>>(n, w->s, w->p, w->sc);
  count_launch(2);
}

int pcg(Matrix *m, const double *b, double *x, int has_x0, double rel_tol, double abs_tol, int64_t max_iters,
        b200fem_solve_info *info, b200fem_error *err) {
  if (err) memset(err, 0, sizeof(*err)), err->cell = -1, err->qp = -1;
  if (info) memset(info, 0, sizeof(*info));
  if (!(rel_tol > 0) || !(abs_tol > 0)) {
    set_err(err, B200FEM_E_INVALID, "linear solver tolerances must be positive");
    return B200FEM_E_INVALID;
  }
  int st = ensure_work(m);
  if (st) return set_err(err, st, "Krylov workspace allocation failed"), st;
  KrylovWork *w = m->kw;
  cudaStream_t s = m->stream;
  const int64_t n = m->n;
  int64_t nzero = 0;
  st = launch_diagonal(m, w->diag, w->inv, &w->red, &nzero);
  if (st) return set_err(err, st, "diagonal extraction failed"), st;
  if (nzero) {
    set_err(err, B200FEM_E_ZERO_DIAGONAL, "zero diagonal entry; Jacobi preconditioner undefined");
    return B200FEM_E_ZERO_DIAGONAL;
  }
  if (!has_x0) B200_CUDA_E(cudaMemsetAsync(x, 0, n * sizeof(double), s), err);
  if (m->n_dir) {
    k_set_dirichlet<<<grid_vec(m->n_dir), kThreads, 0, s>>>(x, b, m->dir_dofs, m->n_dir);
    count_launch();
  }
  if (launch_dot(b, b, n, &w->red, s)) return B200FEM_E_CUDA;
  double bb = 0.0;
  B200_CUDA_E(cudaMemcpyAsync(&bb, w->red.result, sizeof(double), cudaMemcpyDeviceToHost, s), err);
  B200_CUDA_E(cudaStreamSynchronize(s), err);
  const double tol = std::max(rel_tol * std::sqrt(bb), abs_tol);
  const int64_t max_it = max_iters > 0 ? max_iters : 10 * n;
  KrylovScalars *H = w->sc_host;
  memset(H, 0, 3 * sizeof(KrylovScalars));
  H[0].tol = tol;
  H[0].max_iters = max_it;
  long long it = 0, mv = 0, restarts = 0;
  const size_t ssz = sizeof(KrylovScalars);
  LoopGraph loop_graph;
  for (;;) {
    H[0].status = KS_RUNNING;
    H[0].it = it;
    H[0].mv = mv;
    B200_CUDA_E(cudaMemcpyAsync(w->sc, &H[0], ssz, cudaMemcpyHostToDevice, s), err);
    SpmvArgs ar{x, w->r, w->inv, w->diag, b, w->p, w->sc, 1};  // r = b - A x, p = D^-1 r
    if (launch_spmv(m, SP_CGRES, ar, &w->red)) return B200FEM_E_CUDA;
    ++restarts;
    B200_CUDA_E(cudaMemcpyAsync(&H[1], w->sc, ssz, cudaMemcpyDeviceToHost, s), err);
    B200_CUDA_E(cudaStreamSynchronize(s), err);
    mv = H[1].mv;
    const double res = H[1].res;
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
    k_begin_cg<<<1, 1, 0, s>>>(w->sc);
    count_launch();
    int cur = 0;
    if (use_graph_loop()) {
      const long long it0 = it;
      if (int rc = run_loop_graph(m, loop_graph, [&] { enqueue_cg_iteration(m, x); }, err)) return rc;
      B200_CUDA_E(cudaMemcpyAsync(&H[1], w->sc, ssz, cudaMemcpyDeviceToHost, s), err);
      B200_CUDA_E(cudaStreamSynchronize(s), err);
      count_launch(3 * (H[1].it - it0) + 1);
      cur = 1;
    } else {
      int batch = 4;
      auto enqueue_batch = [&](int slot) -> int {
        for (int i = 0; i < batch; ++i) enqueue_cg_iteration(m, x);
        B200_CUDA_E(cudaMemcpyAsync(&H[1 + slot], w->sc, ssz, cudaMemcpyDeviceToHost, s), err);
        B200_CUDA_E(cudaEventRecord(w->ev[slot], s), err);
        return 0;
      };
      if (enqueue_batch(cur)) return B200FEM_E_CUDA;
      for (;;) {
        batch = std::min(batch * 2, 32);
        if (enqueue_batch(cur ^ 1)) return B200FEM_E_CUDA;
        B200_CUDA_E(cudaEventSynchronize(w->ev[cur]), err);
        if (H[1 + cur].status != KS_RUNNING) break;
        cur ^= 1;
      }
      B200_CUDA_E(cudaStreamSynchronize(s), err);
    }
    const KrylovScalars done = H[1 + (cur ^ 1)];
    it = done.it;
    mv = done.mv;
    B200_CUDA_E(cudaGetLastError(), err);
    if (done.status == KS_BREAKDOWN) {
      if (info) *info = b200fem_solve_info{it, mv, restarts, done.res, tol};
      if (err) err->iterations = it, err->value = done.res;
      set_err(err, B200FEM_E_BREAKDOWN, "PCG breakdown at iteration %lld: p.Ap = %.3e <= 0 (operator not SPD)", it,
              done.r0v);
      return B200FEM_E_BREAKDOWN;
    }
  }
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200fem_matrix_fem(b200fem_matrix **out, b200fem_ctx *ctx, const double *data) {
  Ctx *c = (Ctx *)ctx;
  if (!out || !c) return B200FEM_E_INVALID;
  Matrix *m = new Matrix();
  m->n = c->n_dofs;
  m->nnz = c->nnz;
  m->data = data;
  m->stream = c->stream;
  m->diag_slots = c->diag;
  m->dir_dofs = c->dir_dofs;
  m->n_dir = c->n_dir;
  if (c->vec == 3) {
    m->kind = MK_FEM3;
    m->nbr_ptr = c->nbr_ptr;
    m->nbr = c->nbr;
    m->indptr = c->indptr;
    // Bulk-copy pipelined SpMV (default): 6.30 TB/s vs 5.36 TB/s for the register-streaming
    // kernel on config 3 (profiles/r01_spmv_variants.md); B200FEM_SPMV_LDG=1 selects the latter.
    if (!getenv("B200FEM_SPMV_LDG")) {
      int st = prepare_fem3_chunks(m);
      if (st) {
        delete m;
        return st;
      }
    }
  } else {
    m->kind = MK_CSR;
    m->indptr = c->indptr;
    m->indices = c->nbr;  // vec 1: node list == column list
    m->lanes = 8;
  }
  *out = (b200fem_matrix *)m;
  return 0;
}

int b200fem_matrix_fem_sym(b200fem_matrix **out, b200fem_ctx *ctx, const double *sym) {
  Ctx *c = (Ctx *)ctx;
  if (!out || !c || c->vec != 3) return B200FEM_E_INVALID;
  Matrix *m = new Matrix();
  m->kind = MK_SYM3;
  m->n = c->n_dofs;
  m->nnz = c->nnz;
  m->data = sym;
  m->stream = c->stream;
  m->nbr_ptr = c->nbr_ptr;
  m->nbr = c->nbr;
  m->indptr = c->indptr;
  m->up_ptr = c->up_ptr;
  m->lo_blk = c->lo_blk;
  m->dir_flag = c->n_dir ? c->dir_flag : nullptr;
  m->dir_dofs = c->dir_dofs;
  m->n_dir = c->n_dir;
  if (getenv("B200FEM_SYM_TMA")) {  // bulk-copy variant: 2.83 ms vs 1.64 ms LDG (L2-gather bound)
    int st = prepare_sym3_chunks(m);
    if (st) {
      delete m;
      return st;
    }
  }
  *out = (b200fem_matrix *)m;
  return 0;
}

int b200fem_matrix_fem_grid(b200fem_matrix **out, b200fem_ctx *ctx, const double *grid) {
  return b200fem_matrix_fem_grid_ex(out, ctx, grid, 0);
}

int b200fem_matrix_fem_grid_ex(b200fem_matrix **out, b200fem_ctx *ctx, const double *grid, int32_t flags) {
  Ctx *c = (Ctx *)ctx;
  if (!out || !c || !c->grid_nx || !grid) return B200FEM_E_INVALID;
  Matrix *m = new Matrix();
  m->kind = MK_GRID3;
  m->gvec = c->vec;
  m->n = c->n_dofs;
  m->nnz = c->nnz;
  m->data = grid;
  m->stream = c->stream;
  m->nbr_ptr = c->nbr_ptr;
  m->nbr = c->nbr;
  m->indptr = c->indptr;
  const bool raw = flags & B200FEM_GRID_PRE_DIRICHLET;  // K0: no identity rows
  m->dir_flag = (c->n_dir && !raw) ? c->dir_flag : nullptr;
  m->dir_dofs = raw ? nullptr : c->dir_dofs;
  m->n_dir = raw ? 0 : c->n_dir;
  m->gnx = c->grid_nx;
  m->gny = c->grid_ny;
  m->gnz = c->grid_nz;
  m->gnpad = c->grid_npad;
  int st = prepare_grid3(m);
  if (st) {
    delete m;
    return st;
  }
  *out = (b200fem_matrix *)m;
  return 0;
}

// FP64 GRID3 values -> their FP32 copy (same layout), rounded to nearest
__global__ void k_grid_to_f32(const double *__restrict__ a, float *__restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __double2float_rn(a[i]);
}

int b200fem_grid_to_f32(const double *src, float *dst, int64_t n, void *stream) {
  if (n < 0 || n % 288 || (n && (!src || !dst))) return B200FEM_E_INVALID;
  if (!n) return 0;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n + kThreads - 1) / kThreads));
  k_grid_to_f32<<<g, kThreads, 0, (cudaStream_t)stream>>>(src, dst, n);
  count_launch();
  return cudaGetLastError() == cudaSuccess ? 0 : B200FEM_E_CUDA;
}

int b200fem_matrix_set_f32(b200fem_matrix *mat, const float *data32) {
  Matrix *m = (Matrix *)mat;
  if (!m || m->kind != MK_GRID3 || m->gvec != 3) return B200FEM_E_INVALID;
  m->data32 = data32;
  return 0;
}

int b200fem_ctx_grid_size(const b200fem_ctx *ctx, int64_t *n_values, int32_t *dims) {
  const Ctx *c = (const Ctx *)ctx;
  if (!c || !n_values) return B200FEM_E_INVALID;
  *n_values = c->grid_nx ? 14 * c->vec * c->vec * c->grid_npad : 0;
  if (dims) dims[0] = c->grid_nx, dims[1] = c->grid_ny, dims[2] = c->grid_nz;
  return 0;
}

int b200fem_ctx_sym_size(const b200fem_ctx *ctx, int64_t *n_values) {
  const Ctx *c = (const Ctx *)ctx;
  if (!c || c->vec != 3) return B200FEM_E_INVALID;
  *n_values = 9 * c->n_sym_blocks;
  return 0;
}

int b200fem_matrix_csr(b200fem_matrix **out, int64_t n, int64_t nnz, const int32_t *indptr, const int32_t *indices,
                       const double *data, void *stream) {
  if (!out || n < 0 || nnz < 0) return B200FEM_E_INVALID;
  Matrix *m = new Matrix();
  m->kind = MK_CSR;
  m->n = n;
  m->nnz = nnz;
  m->indptr = indptr;
  m->indices = indices;
  m->data = data;
  m->stream = (cudaStream_t)stream;
  const double avg = n ? (double)nnz / (double)n : 0.0;
  m->lanes = avg <= 6 ? 4 : (avg <= 24 ? 8 : (avg <= 64 ? 16 : 32));
  *out = (b200fem_matrix *)m;
  return 0;
}

int b200fem_matrix_set_data(b200fem_matrix *mm, const double *data) {
  ((Matrix *)mm)->data = data;
  return 0;
}

int b200fem_matrix_destroy(b200fem_matrix *mm) {
  Matrix *m = (Matrix *)mm;
  if (!m) return 0;
  cudaStreamSynchronize(m->stream);
  free_work(m->kw);
  cudaFree(m->chunk_node);
  delete m;
  return 0;
}

int b200fem_matvec(b200fem_matrix *mm, const double *x, double *y) {
  Matrix *m = (Matrix *)mm;
  if (m->n == 0) return 0;
  SpmvArgs a{x, y, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
  return launch_spmv(m, SP_PLAIN, a, nullptr);
}

int b200fem_diagonal(b200fem_matrix *mm, double *diag) {
  Matrix *m = (Matrix *)mm;
  if (m->n == 0) return 0;
  int st = ensure_work(m);
  if (st) return st;
  st = launch_diagonal(m, diag, m->kw->inv, &m->kw->red, nullptr);
  return st;
}

int b200fem_pcg(b200fem_matrix *mm, const double *b, double *x, int32_t has_x0, double rel_tol, double abs_tol,
                int64_t max_iters, b200fem_solve_info *info, b200fem_error *err) {
  Matrix *m = (Matrix *)mm;
  if (m->n == 0) {
    if (info) memset(info, 0, sizeof(*info));
    return 0;
  }
  return pcg(m, b, x, has_x0, rel_tol, abs_tol, max_iters, info, err);
}

int b200fem_bicgstab(b200fem_matrix *mm, const double *b, double *x, int32_t has_x0, double rel_tol, double abs_tol,
                     int64_t max_iters, b200fem_solve_info *info, b200fem_error *err) {
  Matrix *m = (Matrix *)mm;
  if (m->n == 0) {
    if (info) memset(info, 0, sizeof(*info));
    return 0;
  }
  return bicgstab(m, b, x, has_x0, rel_tol, abs_tol, max_iters, info, err);
}

int b200fem_bicgstab_profile(b200fem_matrix *mm, const double *b, double *x, int32_t iters, double *out_us) {
  Matrix *m = (Matrix *)mm;
  if (!m || !b || !x || !out_us || iters < 1) return B200FEM_E_INVALID;
  return bicgstab_profile(m, b, x, iters, out_us);
}

}  // extern "C"
