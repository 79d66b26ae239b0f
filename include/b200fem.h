/*
 * b200fem.h — C ABI of libb200fem.so, the sm_100a forward-solve hot path of the
 * differentiable HEX8 FEM (arXiv 2212.00964; reference package "gradfem").
 *
 * Conventions
 *  - Every entry point returns int status (0 = OK, see B200FEM_E_*) and, when it
 *    can fail for a data reason, fills a caller-provided b200fem_error.
 *  - "host" pointers are CPU memory read during the call; "dev" pointers are
 *    device memory (e.g. torch CUDA tensors' data_ptr()) that the library never
 *    frees. Everything a context allocates is freed by b200fem_ctx_destroy.
 *  - A context (and a matrix) is bound to one CUDA stream; calls are ordered on
 *    it and are not re-entrant per handle (reference: single logical thread,
 *    SPEC.md:452; numba threads only inside csr_matvec, kernels.py:21-28).
 *  - DOFs are node-major (dof = node*vec + comp) exactly as the reference
 *    (assembly.py:94); the CSR pattern / scatter map are bit-identical to
 *    sparse.py:75-108.
 *
 * Each entry cites the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/gradfem/).
 */
#ifndef B200FEM_H
#define B200FEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference exception classes in Python) ---- */
#define B200FEM_OK 0
#define B200FEM_E_INVERTED_ELEMENT 1     /* elements.py:124-129  InvertedElementError      */
#define B200FEM_E_INVERTED_DEFORMATION 2 /* materials.py:94-100  InvertedDeformationError  */
#define B200FEM_E_NONFINITE_VALUE 3      /* assembly.py:228-233  KernelEvaluationError     */
#define B200FEM_E_NONFINITE_DERIV 4      /* assembly.py:219-227  KernelEvaluationError     */
#define B200FEM_E_LINEAR_SOLVER 5        /* solvers.py:119-125   LinearSolverError         */
#define B200FEM_E_BREAKDOWN 6            /* solvers.py:149-155   BreakdownError            */
#define B200FEM_E_ZERO_DIAGONAL 7        /* solvers.py:102-103   LinearSolverError         */
#define B200FEM_E_INVALID 8              /* bad argument                                   */
#define B200FEM_E_CUDA 9                 /* CUDA runtime error                             */
#define B200FEM_E_UNSUPPORTED 10         /* mesh/material outside the device path          */

/* ---- materials (materials.py:134-194; problems.py:166-202) ---- */
#define B200FEM_MAT_POISSON 0 /* IsotropicDiffusion: params[0] = alpha             */
#define B200FEM_MAT_LE 1      /* LinearElastic: params[1] = lam, params[2] = mu     */
#define B200FEM_MAT_NH 2      /* NeoHookean: params[2] = G (= mu), params[3] = kappa */
#define B200FEM_MAT_J2 3      /* J2Plasticity: lam, mu, params[4] = sigma_yield      */

#define B200FEM_FLAG_SIMP 1          /* flux scaled by theta_e^penalty, params[5] = penalty */
#define B200FEM_FLAG_DESIGN_SOURCE 2 /* Poisson nodal design source b = sum theta_k phi_k   */

typedef struct b200fem_error {
  int32_t code;
  int32_t qp;     /* quadrature point of the first offender, -1 if n/a   */
  int64_t cell;   /* global cell index of the first offender, -1 if n/a  */
  double value;   /* det / min det(F) / residual, depending on code      */
  int64_t iterations;
  char msg[256];
} b200fem_error;

typedef struct b200fem_solve_info {
  int64_t iterations; /* BiCGSTAB iterations (solvers.py:131-132 counter)   */
  int64_t matvecs;    /* operator applications incl. explicit residuals     */
  int64_t restarts;   /* explicit-residual (re)starts                       */
  double residual;    /* final true residual ||A x - b||                    */
  double tol;         /* max(rel_tol * ||b||, abs_tol)                      */
} b200fem_solve_info;

typedef struct b200fem_ctx b200fem_ctx;
typedef struct b200fem_matrix b200fem_matrix;

/* ---- library ---- */
int b200fem_version(void);
/* number of kernels this library has launched since load (bench evidence) */
int64_t b200fem_launch_count(void);
/* block until all work on `stream` (cudaStream_t, 0 = legacy default) is done */
int b200fem_stream_sync(void *stream);

/* ---- context: replaces assembly.workspace() (assembly.py:83-145) ----
 * coords_host (n_nodes,3) f64, cells_host (n_cells,8) int64 in VTK HEX8 order.
 * Builds on the device: the geometry check (map_elements, elements.py:117-131),
 * the node adjacency / CSR pattern / scatter positions (sparse.py:75-108),
 * diagonal slots (assembly.py:96-97) and the node -> cell lists of the ordered
 * (ascending cell id, kernels.py:30-34) per-node gathers. */
int b200fem_ctx_create(b200fem_ctx **out, int64_t n_nodes, int64_t n_cells, int32_t vec,
                       const double *coords_host, const int64_t *cells_host, int32_t material,
                       const double *params /* [8] */, int32_t flags, void *stream,
                       b200fem_error *err);
int b200fem_ctx_destroy(b200fem_ctx *ctx);
int b200fem_ctx_info(const b200fem_ctx *ctx, int64_t *n_dofs, int64_t *nnz, int32_t *max_neighbors);

/* pattern copy-outs for bit-exact parity checks (device outputs, caller-sized) */
int b200fem_copy_indptr(b200fem_ctx *ctx, int32_t *indptr_dev /* n_dofs+1 */);
int b200fem_copy_indices(b200fem_ctx *ctx, int32_t *indices_dev /* nnz */);
int b200fem_copy_dest(b200fem_ctx *ctx, int64_t cell_lo, int64_t cell_hi,
                      int32_t *dest_dev /* (cell_hi-cell_lo, 8vec, 8vec) */);
int b200fem_copy_diag_slots(b200fem_ctx *ctx, int32_t *diag_dev /* n_dofs */);

/* ---- boundary data / design / state (assembly.py:99-128, problems.py:93-163) ---- */
int b200fem_set_dirichlet(b200fem_ctx *ctx, const int64_t *dofs_host, const double *values_host,
                          int64_t n);
int b200fem_set_loads(b200fem_ctx *ctx, const double *f_neumann_host /* nullable */,
                      const double *f_body_host /* nullable */);
/* theta: per cell (SIMP) or per node (design source); device or host pointer */
int b200fem_set_theta(b200fem_ctx *ctx, const double *theta, int64_t n, int32_t is_host);
int b200fem_set_state(b200fem_ctx *ctx, const double *eps_prev, const double *sig_prev,
                      int32_t is_host); /* (n_cells,8,3,3) each */
int b200fem_get_state(b200fem_ctx *ctx, double *eps_prev_dev, double *sig_prev_dev);

/* ---- assembly (assembly.py:236-261, 273-300) ----
 * residual: R = sum_e R_e(U) (per-node gather in ascending cell id: the reference's
 *           sequential scatter order, kernels.py:30-34; no atomics)
 *           - bc_scale*f_neumann - f_body; Dirichlet rows -> U[d]-bc_scale*u_D.
 * norm_host (nullable) receives ||R||_2 (forces a stream sync).            */
int b200fem_residual(b200fem_ctx *ctx, const double *U_dev, double bc_scale,
                     int32_t apply_dirichlet, double *R_dev, double *norm_host,
                     b200fem_error *err);
/* jacobian: CSR values (pattern of this ctx) of dR/dU with Dirichlet identity rows. */
int b200fem_jacobian(b200fem_ctx *ctx, const double *U_dev, double *data_dev, b200fem_error *err);
/* flux at every quadrature point (N_e,8,vec,3)  (solvers.py:237-250) */
int b200fem_qp_flux(b200fem_ctx *ctx, const double *U_dev, double *out_dev, b200fem_error *err);
/* volume average of the flux (vec*3 values, host)   (solvers.py:253-258) */
int b200fem_volume_average_flux(b200fem_ctx *ctx, const double *U_dev, double *out_host,
                                b200fem_error *err);
/* J2 state commit eps <- sym grad u, sig <- return map (problems.py:155-163) */
int b200fem_commit_state(b200fem_ctx *ctx, const double *U_dev);
/* geometry of every cell (map_elements, elements.py:80-131; Workspace.phys_grads / JxW,
 * assembly.py:64-80): phys_grads (N_e,8q,8i,3), JxW (N_e,8q); either output nullable */
int b200fem_geometry(b200fem_ctx *ctx, double *phys_grads_dev, double *jxw_dev);

/* ---- constitutive laws over a batch of points (materials.py:74-194) ----
 * No context needed: material_id B200FEM_MAT_*, params[8] as for ctx_create (host).
 * grad_u (n, vec, 3) dev.  J2: eps_prev, sig_prev (n,3,3) dev (the committed state).
 * Outputs (dev, nullable): flux (n, vec, 3) = linear_elastic_flux / neo_hookean_flux /
 * j2_return_map / alpha grad u; tangent (n, 3vec, 3vec) = d flux / d grad u (the hand
 * tangent the element kernels use); eps_out, sig_out (J2, both or
 * neither) = commit_state (materials.py:125-131); det_f (n) = det F (NH; 1 otherwise).
 * NH points with det F <= 0 get zero flux / tangent and the call returns
 * B200FEM_E_INVERTED_DEFORMATION (err->cell = first such point, err->value = min det F;
 * materials.py:94-100).  Synchronises `stream`. */
int b200fem_law_batch(int32_t material_id, const double *params, int64_t n, const double *grad_u_dev,
                      const double *eps_prev_dev, const double *sig_prev_dev, double *flux_dev,
                      double *tangent_dev, double *eps_out_dev, double *sig_out_dev, double *det_f_dev,
                      void *stream, b200fem_error *err);
/* neo_hookean_energy(F) (materials.py:80-85) for F (n,3,3) dev -> W (n) dev; params[2] = G,
 * params[3] = kappa.  Asynchronous on `stream`. */
int b200fem_nh_energy_batch(const double *params, int64_t n, const double *F_dev, double *W_dev, void *stream);

/* ---- adjoint half ---- */
/* param_vjp: out = w_eff^T dR/dtheta at U (assembly.py:303-341); w_eff zeroes the Dirichlet
 * rows.  SIMP ctx: out has n_cells entries (theta: n_cells); design-source ctx: n_nodes
 * (theta: n_nodes, U unused).  theta is the design vector to differentiate at (not the one
 * bound by set_theta). */
int b200fem_param_vjp(b200fem_ctx *ctx, const double *U_dev, const double *theta_dev, const double *w_dev,
                      double *out_dev, b200fem_error *err);
/* transpose_fem: values of A^T on this ctx's (structurally symmetric) pattern; a pure
 * permutation of data_dev, bit-identical to CsrMatrix.transpose (sparse.py:53-62). */
int b200fem_transpose_fem(b200fem_ctx *ctx, const double *data_dev, double *data_t_dev);
/* csr_transpose: generic CSR transpose (stable by column, sparse.py:53-62); synchronous. */
int b200fem_csr_transpose(int64_t n, int64_t nnz, const int32_t *indptr_dev, const int32_t *indices_dev,
                          const double *data_dev, int32_t *indptr_t_dev, int32_t *indices_t_dev,
                          double *data_t_dev, void *stream);

/* ---- sparse operators (sparse.py:15-51, kernels.py:37-47) ---- */
/* FEM matrix on this ctx's pattern (uses the node-blocked index, no indices array) */
int b200fem_matrix_fem(b200fem_matrix **out, b200fem_ctx *ctx, const double *data_dev);
/* Symmetric node-block operator (vec 3): the upper 3x3 node blocks of the tangent before
 * the Dirichlet row replacement (b200fem_jacobian_sym), applied with identity Dirichlet rows.
 * Same operator as the CSR Jacobian of this ctx with half of the value traffic. */
int b200fem_ctx_sym_size(const b200fem_ctx *ctx, int64_t *n_values);
int b200fem_jacobian_sym(b200fem_ctx *ctx, const double *U_dev, double *data_dev /* nullable */,
                         double *sym_dev, b200fem_error *err);
int b200fem_matrix_fem_sym(b200fem_matrix **out, b200fem_ctx *ctx, const double *sym_dev);
/* GRID3: the same operator for contexts whose connectivity is a z-major box lattice
 * (generate_box_mesh, mesh.py:134-168): self + 13 upper-offset node blocks stored as 14
 * offset-major arrays (pre-Dirichlet), lower blocks read back as their transposes, identity
 * Dirichlet rows.  grid_size gives 0 values when the mesh is not a lattice (dims = nodes per
 * axis, nullable).  Replaces the K passed to bicgstab_jacobi by newton_solve
 * (solvers.py:177-184, 218) -- assemble_jacobian still returns the reference CSR. */
int b200fem_ctx_grid_size(const b200fem_ctx *ctx, int64_t *n_values, int32_t *dims /* [3], nullable */);
int b200fem_jacobian_grid(b200fem_ctx *ctx, const double *U_dev, double *data_dev /* nullable */,
                          double *grid_dev, b200fem_error *err);
int b200fem_matrix_fem_grid(b200fem_matrix **out, b200fem_ctx *ctx, const double *grid_dev);
/* flags: B200FEM_GRID_PRE_DIRICHLET = the pre-Dirichlet tangent K0 (no identity rows): the
 * adjoint's lambda_d = b_d - (K^T x)_d with x_d = 0 (adjoint.py:25-31, PCG split) */
#define B200FEM_GRID_PRE_DIRICHLET 1
int b200fem_matrix_fem_grid_ex(b200fem_matrix **out, b200fem_ctx *ctx, const double *grid_dev, int32_t flags);
/* Opt-in mixed-precision Newton operator (LinearSolveConfig(operator="grid32")): the GRID3
 * matvec streams a single-precision copy of the values (half the bytes), with FP64 operands,
 * products, sums and Krylov vectors; the diagonal (Jacobi) stays FP64.  An inexact-Newton
 * variant of the K handed to bicgstab_jacobi by newton_solve (solvers.py:218): the residual
 * and the Newton stopping test are unchanged FP64.  grid_to_f32 rounds the n values to nearest
 * (same layout);
 * set_f32(m, NULL) restores the FP64 values (GRID3, vec 3 only). */
int b200fem_grid_to_f32(const double *grid_dev, float *grid32_dev, int64_t n_values, void *stream);
int b200fem_matrix_set_f32(b200fem_matrix *m, const float *data32_dev);
/* generic CSR on the device (any square matrix with sorted unique columns) */
int b200fem_matrix_csr(b200fem_matrix **out, int64_t n, int64_t nnz, const int32_t *indptr_dev,
                       const int32_t *indices_dev, const double *data_dev, void *stream);
int b200fem_matrix_set_data(b200fem_matrix *m, const double *data_dev);
int b200fem_matrix_destroy(b200fem_matrix *m);
int b200fem_matvec(b200fem_matrix *m, const double *x_dev, double *y_dev);
int b200fem_diagonal(b200fem_matrix *m, double *diag_dev);

/* ---- Krylov (solvers.py:87-167) ----
 * x_dev holds x0 on entry when has_x0 != 0 (else it is zeroed) and the solution on exit.
 * max_iters <= 0 means 10*n. Same termination, restart and breakdown rules as the reference. */
int b200fem_bicgstab(b200fem_matrix *m, const double *b_dev, double *x_dev, int32_t has_x0,
                     double rel_tol, double abs_tol, int64_t max_iters, b200fem_solve_info *info,
                     b200fem_error *err);

/* Jacobi-preconditioned CG for symmetric operators (north_star "CG/BiCGSTAB"; BASELINE
 * config 2).  FEM matrices: starts from x_d = b_d on Dirichlet rows so the row-replaced K
 * acts as its SPD free block.  Same termination rule as bicgstab (true residual); restarts
 * from the explicit residual; BreakdownError if p.Ap <= 0. */
/* diagnostics: one BiCGSTAB iteration as run inside the while-graph (out_us[0], over `iters`
 * iterations from x = 0 with tolerance 0) against its kernels timed one by one (out_us[1..6]:
 * update_p, SpMV r0.v, update_s, SpMV t.t/t.s, update_xr, loop condition; out_us[7] = sum).
 * Overwrites x; b is the right-hand side. */
int b200fem_bicgstab_profile(b200fem_matrix *m, const double *b_dev, double *x_dev, int32_t iters, double *out_us);
int b200fem_pcg(b200fem_matrix *m, const double *b_dev, double *x_dev, int32_t has_x0, double rel_tol,
                double abs_tol, int64_t max_iters, b200fem_solve_info *info, b200fem_error *err);

/* ---- partitioned solve (new — the reference is single-process) ----
 * A part = the local FEM matrix of one contiguous node range plus its ghost layer.  Halo
 * lists are local node ids: send_nodes[k] (owned, needed by peer i) and recv_nodes[k]
 * (ghost, owned by peer i), grouped per peer.  Communicator: NCCL (one part per process)
 * or local (several parts in one process on one device, for verification). */
typedef struct b200fem_comm b200fem_comm;
typedef struct b200fem_part b200fem_part;
int b200fem_comm_unique_id(uint8_t *out /* 128 bytes */);
int b200fem_comm_create_nccl(b200fem_comm **out, const uint8_t *id /* 128 bytes */, int32_t nranks, int32_t rank);
int b200fem_comm_create_local(b200fem_comm **out);
int b200fem_comm_destroy(b200fem_comm *comm);
int b200fem_comm_allreduce(b200fem_comm *comm, double *buf_dev, int64_t n, void *stream);
int b200fem_part_create(b200fem_part **out, b200fem_matrix *local, int64_t own_node_lo, int64_t own_node_hi,
                        int32_t n_peers, const int32_t *peers_host, const int64_t *send_counts_host,
                        const int32_t *send_nodes_host, const int64_t *recv_counts_host,
                        const int32_t *recv_nodes_host);
int b200fem_part_destroy(b200fem_part *part);
/* BiCGSTAB over all parts (solvers.py:87-167 semantics, global tolerances and counters);
 * b[p], x[p] are the parts' local device vectors (owned entries are the unknowns).  Batches of
 * iterations run as one captured CUDA graph (kernels + NCCL halo / allreduce) when the parts
 * share a stream; B200FEM_NO_GRAPH=1 enqueues them eagerly.  Three allreduces per iteration,
 * two (one fused dot group) on NCCL communicators of >= 4 ranks or with
 * B200FEM_DIST_FUSED_DOTS=1 (=0 forces three); the explicit residual decides convergence. */
int b200fem_dist_bicgstab(b200fem_part **parts, int32_t nparts, b200fem_comm *comm, double *const *b,
                          double *const *x, int32_t has_x0, double rel_tol, double abs_tol, int64_t max_iters,
                          b200fem_solve_info *info, b200fem_error *err);
/* Jacobi-PCG over all parts (b200fem_pcg semantics: x_d = b_d on Dirichlet rows, symmetric
 * operator; one halo and two allreduces per iteration). */
int b200fem_dist_pcg(b200fem_part **parts, int32_t nparts, b200fem_comm *comm, double *const *b,
                     double *const *x, int32_t has_x0, double rel_tol, double abs_tol, int64_t max_iters,
                     b200fem_solve_info *info, b200fem_error *err);
/* ghost entries of vec[p] <- owners' values */
int b200fem_dist_halo(b200fem_part **parts, int32_t nparts, b200fem_comm *comm, double *const *vec);
/* sum over parts of the owned-range dot products */
int b200fem_dist_dot(b200fem_part **parts, int32_t nparts, b200fem_comm *comm, double *const *x,
                     double *const *y, double *out_host);

/* ---- design loop (inverse.py:186-346) ---- */
typedef struct b200fem_filter b200fem_filter;
/* density filter: hat weights max(0, r - |c_j - c_i|) over element centroids, row-normalised
 * (inverse.py:204-228, the reference builds it with a k-d tree).  cells: (n_cells, 8) int32. */
int b200fem_filter_create(b200fem_filter **out, int64_t n_cells, const double *coords_dev,
                          const int32_t *cells_dev, double radius, void *stream);
int b200fem_filter_info(const b200fem_filter *f, int64_t *n, int64_t *nnz);
/* copy the filter CSR into caller buffers (n+1, nnz, nnz) */
int b200fem_filter_copy(const b200fem_filter *f, int32_t *indptr_dev, int32_t *indices_dev, double *data_dev);
/* y = H (v [* mul]) [/ max(div, floor)]: filt(field) and filter_sensitivities (inverse.py:186-234) */
int b200fem_filter_apply(const b200fem_filter *f, const double *v_dev, const double *mul_dev /* nullable */,
                         const double *div_dev /* nullable */, double floor_value, double *y_dev);
int b200fem_filter_destroy(b200fem_filter *f);
/* one MMA step for a single linear constraint (inverse.py:260-346).  lower/upper: previous
 * asymptotes in (when use_history), new asymptotes out.  Synchronous. */
int b200fem_mma_update(int64_t n, const double *x_dev, const double *dj_dev, double g_value,
                       const double *g_grad_dev, const double *lb_dev, const double *ub_dev, double *lower_dev,
                       double *upper_dev, const double *x_prev_dev, const double *x_prev2_dev,
                       int32_t use_history, double asym_init, double asym_expand, double asym_shrink,
                       double move_limit, double *x_new_dev, void *stream);
/* relative L2 field error terms by quadrature (inverse.py:45-56): out_host = {sum (u_p-u_t)^2 JxW,
 * sum u_t^2 JxW} for nodal scalar fields on (n_cells, 8) int32 cells. */
int b200fem_l2_field_error(int64_t n_cells, const double *coords_dev, const int32_t *cells_dev,
                           const double *u_pred_dev, const double *u_true_dev, double *out_host, void *stream);

/* ---- small vector helpers (deterministic) ---- */
int b200fem_norm2(const double *x_dev, int64_t n, double *out_host, void *stream);
int b200fem_dot(const double *x_dev, const double *y_dev, int64_t n, double *out_host, void *stream);
int b200fem_gather_sum(const double *x_dev, const int64_t *idx_dev, int64_t n, double *out_host,
                       void *stream);
int b200fem_axpy(int64_t n, double a, const double *x_dev, double *y_dev, void *stream);
int b200fem_scale(int64_t n, double a, const double *x_dev, double *y_dev, void *stream);

/* ---- the reference's low seam (gradfem.kernels, kernels.py:1-55; SURVEY 8(b) seam 1),
 * bit-identical to its numba kernels (same accumulation order, no FMA contraction).
 * csr_matvec: replaces kernels.csr_matvec (kernels.py:37-47, numba body 21-28): y = A x,
 * per row sequential in storage order.  int32 indptr/indices as the reference's CsrMatrix.
 * scatter_add: replaces kernels.scatter_add (kernels.py:50-55, numba body 30-34):
 * values[dest[k]] += contribs[k] in ascending k, in place; B200FEM_E_INVALID if a dest is
 * outside [0, n_values). */
int b200fem_csr_matvec_seq(int64_t n_rows, const int32_t *indptr_dev, const int32_t *indices_dev,
                           const double *data_dev, const double *x_dev, double *y_dev, void *stream);
int b200fem_scatter_add(double *values_dev, int64_t n_values, const int64_t *dest_dev, const double *contribs_dev,
                        int64_t n, void *stream, b200fem_error *err);

/* ---- host output formatting.  Rows of a (rows, cols) array as text lines,
 * values space-separated, "%.17g" for doubles (= Python f"{x:.17g}", the reference's
 * io_vtk._fmt, io_vtk.py:18-19), "%lld" for integers with an optional leading `prefix`
 * column (the VTK CELLS count; < 0 = none).  Multi-threaded on the host.  Returns the bytes
 * written, or -(bytes needed) when `out` is null or `cap` is too small. */
int64_t b200fem_format_f64_rows(const double *v_host, int64_t rows, int32_t cols, char *out, int64_t cap);
int64_t b200fem_format_i64_rows(const int64_t *v_host, int64_t rows, int32_t cols, int64_t prefix, char *out,
                                int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* B200FEM_H */
