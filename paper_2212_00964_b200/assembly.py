"""Residual and CSR-Jacobian assembly on the GPU (reference gradfem/assembly.py:36-300).

``workspace(problem)`` replaces the reference's host cache (assembly.py:83-145) with a
device context (csrc/context.cu): geometry check, CSR pattern, scatter positions, diagonal
slots and the node -> cell lists of the ordered gathers are built on the B200; the Dirichlet
table and the fixed Neumann / body load vectors are computed here on the host once
(north_star: host code keeps the Dirichlet handling) and uploaded.

``assemble_residual`` / ``assemble_jacobian`` keep the reference signatures and return
host arrays for host inputs (drop-in); pass a CUDA tensor U to stay on the device.
"""

from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _device as D
from . import _lib
from .elements import cell_jxw, face_quadrature, quad_point_coords, shape_values_at_gauss
from .errors import ConflictingConstraintError, KernelEvaluationError, UnsupportedKernelError, raise_for
from .materials import BUILTIN_LAWS, QuadPointState, _DeviceLaw
from .mesh import BoundaryLocator, FacetSet, Mesh, locate_nodes
from .sparse import CsrMatrix

__all__ = ["DirichletSpec", "NeumannSpec", "ConflictingConstraintError", "KernelEvaluationError",
           "UnsupportedKernelError", "workspace", "assemble_residual", "assemble_jacobian",
           "impose_dirichlet_residual", "assemble_param_vjp"]


@dataclass(frozen=True)
class DirichletSpec:
    """Component-wise prescribed value on geometrically located nodes."""

    locator: BoundaryLocator
    component: int
    value_fn: Callable


@dataclass(frozen=True)
class NeumannSpec:
    """Prescribed traction integrated over a boundary facet set."""

    facet_set: FacetSet
    traction_fn: Callable


def _eval_pointwise(fn, pts, shape):
    try:
        out = np.asarray(fn(pts), dtype=np.float64)
        if out.shape == shape:
            return out
    except Exception:
        pass
    return np.array([fn(p) for p in pts], dtype=np.float64).reshape(shape)


def _dirichlet_table(mesh: Mesh, vec: int, specs):
    """Sorted unique constrained DOFs and values; conflicting duplicates raise (assembly.py:148-173)."""
    dofs, vals = [], []
    for spec in specs:
        if not 0 <= spec.component < vec:
            raise ValueError(f"Dirichlet component {spec.component} out of range for vec={vec}")
        nodes = locate_nodes(mesh, spec.locator)
        if nodes.size:
            vals.append(_eval_pointwise(spec.value_fn, mesh.nodes[nodes], (nodes.size,)))
            dofs.append(nodes * vec + spec.component)
    if not dofs:
        return np.empty(0, dtype=np.int64), np.empty(0)
    d = np.concatenate(dofs)
    v = np.concatenate(vals)
    o = np.argsort(d, kind="stable")
    d, v = d[o], v[o]
    same = d[1:] == d[:-1]
    clash = same & (v[1:] != v[:-1])
    if clash.any():
        k = int(d[1:][clash][0])
        raise ConflictingConstraintError(
            f"DOF {k} (node {k // vec}, component {k % vec}) receives two different prescribed values")
    keep = np.ones(d.size, dtype=bool)
    keep[1:] = ~same
    return d[keep], v[keep]


def _neumann_load(mesh: Mesh, vec: int, specs) -> np.ndarray:
    f = np.zeros(mesh.n_nodes * vec)
    for spec in specs:
        facets = spec.facet_set.facets
        if facets.size == 0:
            continue
        fq = face_quadrature(mesh, facets)
        t = _eval_pointwise(spec.traction_fn, fq.points.reshape(-1, 3), (facets.shape[0] * 4, vec))
        fe = np.einsum("fqv,qa,fq->fav", t.reshape(-1, 4, vec), fq.shape_values, fq.JxW)
        dofs = mesh.cells[facets[:, 0][:, None], fq.local_nodes][:, :, None] * vec + np.arange(vec)
        f += _ordered_scatter(dofs.ravel(), fe.ravel(), f.size)
    return f


def _ordered_scatter(idx, vals, n):
    """sum_k vals[k] into out[idx[k]] in ascending k (same order as the reference's
    sequential scatter_add, kernels.py:30-34); np.bincount accumulates in input order."""
    return np.bincount(idx, weights=vals, minlength=n)


def _body_load(mesh: Mesh, vec: int, body) -> np.ndarray:
    f = np.zeros(mesh.n_nodes * vec)
    if body is None:
        return f
    xq = quad_point_coords(mesh)
    b = _eval_pointwise(body, xq.reshape(-1, 3), (mesh.n_cells * 8, vec)).reshape(-1, 8, vec)
    fe = np.einsum("nqv,qi,nq->niv", b, shape_values_at_gauss(), cell_jxw(mesh))
    edofs = mesh.cells[:, :, None] * vec + np.arange(vec)
    return f + _ordered_scatter(edofs.ravel(), fe.ravel(), f.size)


def check_supported(problem):
    """Raise UnsupportedKernelError unless the sm_100a kernels implement this problem."""
    from .problems import PoissonProblem, SimpElasticityProblem, WeakFormProblem

    mat = problem.material
    cls = type(problem)
    if not isinstance(mat, BUILTIN_LAWS) or type(mat).flux is not _DeviceLaw.flux:
        raise UnsupportedKernelError(
            f"material {type(mat).__name__} has no device kernel; supported: "
            "LinearElastic, NeoHookean, J2Plasticity, IsotropicDiffusion")
    allowed_flux = {WeakFormProblem.flux_kernel, SimpElasticityProblem.flux_kernel}
    if cls.flux_kernel not in allowed_flux or (
            cls.flux_kernel is SimpElasticityProblem.flux_kernel and not isinstance(problem, SimpElasticityProblem)):
        raise UnsupportedKernelError(f"{cls.__name__}.flux_kernel is a user map; the device path "
                                     "evaluates only the built-in constitutive laws")
    if cls.source_kernel not in (WeakFormProblem.source_kernel, PoissonProblem.source_kernel):
        raise UnsupportedKernelError(f"{cls.__name__}.source_kernel is a user map")
    if isinstance(problem, SimpElasticityProblem) and mat.material_id not in (_lib.MAT_LE, _lib.MAT_NH):
        raise UnsupportedKernelError("SIMP base material must be LinearElastic or NeoHookean")
    if problem.design_layout == "node" and not isinstance(problem, PoissonProblem):
        raise UnsupportedKernelError("nodal design layout is only implemented for the Poisson source")


class DeviceWorkspace:
    """Per-problem device context (replaces the reference Workspace, assembly.py:64-80)."""

    def __init__(self, problem):
        from .problems import J2PlasticityProblem, SimpElasticityProblem

        check_supported(problem)
        lib = _lib.lib()
        mesh, vec = problem.mesh, problem.vec
        self.vec = vec
        self.n_cells = mesh.n_cells
        self.n_nodes = mesh.n_nodes
        self.dir_dofs, self.dir_values = _dirichlet_table(mesh, vec, problem.dirichlet)
        self.f_neumann = _neumann_load(mesh, vec, problem.neumann)
        self.f_body = _body_load(mesh, vec, problem.body_force)
        params = (C.c_double * 8)(*problem.material.device_params())
        flags = 0
        if isinstance(problem, SimpElasticityProblem):
            flags |= _lib.FLAG_SIMP
            params[5] = problem.penalty
        if problem.design_layout == "node":
            flags |= _lib.FLAG_DESIGN_SOURCE
        self.flags = flags
        coords = np.ascontiguousarray(mesh.nodes, dtype=np.float64)
        cells = np.ascontiguousarray(mesh.cells, dtype=np.int64)
        err = _lib.Error()
        ctx = C.c_void_p()
        self._stream = D.stream()
        st = lib.b200fem_ctx_create(C.byref(ctx), mesh.n_nodes, mesh.n_cells, vec, D.hptr(coords), D.hptr(cells),
                                    problem.material.material_id, C.cast(params, C.c_void_p), flags,
                                    self._stream, C.byref(err))
        raise_for(st, err, "ctx_create")
        self.ctx = ctx
        n_dofs, nnz, mx = C.c_int64(), C.c_int64(), C.c_int32()
        lib.b200fem_ctx_info(ctx, C.byref(n_dofs), C.byref(nnz), C.byref(mx))
        self.n_dofs, self.nnz, self.max_neighbors = n_dofs.value, nnz.value, mx.value
        dd = np.ascontiguousarray(self.dir_dofs, dtype=np.int64)
        dv = np.ascontiguousarray(self.dir_values, dtype=np.float64)
        raise_for(lib.b200fem_set_dirichlet(ctx, D.hptr(dd), D.hptr(dv), dd.size), None, "set_dirichlet")
        fn = self.f_neumann if np.any(self.f_neumann) else None
        fb = self.f_body if np.any(self.f_body) else None
        raise_for(lib.b200fem_set_loads(ctx, D.hptr(fn) if fn is not None else None,
                                        D.hptr(fb) if fb is not None else None), None, "set_loads")
        self._theta_host = None  # copy of the theta last uploaded (content-keyed sync)
        if isinstance(problem, J2PlasticityProblem):
            self.upload_state(problem._host_state)
        self._cache = {}

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and _lib._lib is not None:
            try:
                _lib._lib.b200fem_ctx_destroy(ctx)
            except Exception:
                pass

    @contextlib.contextmanager
    def on_stream(self):
        """Make the context's stream torch's current stream for the block: every launch, torch
        allocation and copy of a multi-call sequence (the Newton loop) then shares one stream
        with the library's kernels.  When the caller's stream differs it is joined both ways
        (the context waits for the caller's pending work, the caller for the block's); yields
        the caller's stream in that case, else None."""
        t = D.torch()
        cur = t.cuda.current_stream()
        if cur.cuda_stream == (self._stream.value or 0):
            yield None
            return
        ext = t.cuda.ExternalStream(self._stream.value or 0)
        ext.wait_stream(cur)
        try:
            with t.cuda.stream(ext):
                yield cur
        finally:
            cur.wait_stream(ext)

    # ------------------------------------------------------------ syncing
    def sync(self, problem):
        """Mirror the host-side mutable inputs the reference re-reads at every assembly
        (problems.py:76-93 theta, 150-157 J2 state): theta is compared by CONTENT with the copy
        last uploaded (in-place edits and attribute reassignment both count; O(n_design) host
        compare), and a live host view of the J2 state is re-uploaded."""
        sv = getattr(problem, "_state_view", None)
        if sv is not None:
            self.upload_state(sv)
        if problem.design_layout is None:
            return
        if problem.theta is None:
            raise ValueError("problem has a design layout but no theta bound")
        th = np.asarray(problem.theta, dtype=np.float64)
        if th.shape != (problem.n_design,):
            raise ValueError(f"theta must have shape ({problem.n_design},), got {th.shape}")
        if self._theta_host is None or not np.array_equal(th, self._theta_host):
            th = np.array(th, dtype=np.float64, order="C", copy=True)
            raise_for(_lib.lib().b200fem_set_theta(self.ctx, D.hptr(th), th.size, 1), None, "set_theta")
            self._theta_host = th

    def upload_state(self, st: QuadPointState):
        eps = np.ascontiguousarray(st.eps_prev, dtype=np.float64)
        sig = np.ascontiguousarray(st.sig_prev, dtype=np.float64)
        if eps.size != self.n_cells * 72 or sig.size != self.n_cells * 72:
            raise ValueError("state must have shape (n_cells, 8, 3, 3)")
        raise_for(_lib.lib().b200fem_set_state(self.ctx, D.hptr(eps), D.hptr(sig), 1), None, "set_state")

    def download_state(self) -> QuadPointState:
        e = D.empty(self.n_cells * 72)
        s = D.empty(self.n_cells * 72)
        raise_for(_lib.lib().b200fem_get_state(self.ctx, D.ptr(e), D.ptr(s)), None, "get_state")
        return QuadPointState(D.to_host(e).reshape(-1, 8, 3, 3), D.to_host(s).reshape(-1, 8, 3, 3))

    # ------------------------------------------------------------ kernels
    def residual(self, problem, U, R, apply_dirichlet=True) -> float:
        """R <- residual(U) on the device; returns ||R||_2 (one stream sync)."""
        self.sync(problem)
        err = _lib.Error()
        nrm = C.c_double()
        st = _lib.lib().b200fem_residual(self.ctx, D.ptr(U), float(problem.bc_scale), int(bool(apply_dirichlet)),
                                        D.ptr(R), C.byref(nrm), C.byref(err))
        raise_for(st, err, "residual")
        return nrm.value

    def jacobian(self, problem, U, data):
        self.sync(problem)
        err = _lib.Error()
        st = _lib.lib().b200fem_jacobian(self.ctx, D.ptr(U), D.ptr(data), C.byref(err))
        raise_for(st, err, "jacobian")

    @property
    def has_sym(self) -> bool:
        return self.vec == 3

    def sym_size(self) -> int:
        n = C.c_int64()
        raise_for(_lib.lib().b200fem_ctx_sym_size(self.ctx, C.byref(n)), None, "sym_size")
        return n.value

    def jacobian_sym(self, problem, U, sym, data=None):
        """Upper symmetric node blocks of the tangent (and optionally the full CSR values)."""
        self.sync(problem)
        err = _lib.Error()
        st = _lib.lib().b200fem_jacobian_sym(self.ctx, D.ptr(U), D.ptr(data) if data is not None else None,
                                             D.ptr(sym), C.byref(err))
        raise_for(st, err, "jacobian_sym")

    @property
    def has_grid(self) -> bool:
        """True when the connectivity is a z-major box lattice (GRID3 operator available)."""
        return self.grid_size() > 0

    def grid_size(self) -> int:
        if not hasattr(self, "_grid_size"):
            n = C.c_int64()
            raise_for(_lib.lib().b200fem_ctx_grid_size(self.ctx, C.byref(n), None), None, "grid_size")
            self._grid_size = n.value
        return self._grid_size

    def jacobian_grid(self, problem, U, grid, data=None):
        """Self + upper-offset node blocks of the tangent in GRID3 layout (optionally also CSR)."""
        self.sync(problem)
        err = _lib.Error()
        st = _lib.lib().b200fem_jacobian_grid(self.ctx, D.ptr(U), D.ptr(data) if data is not None else None,
                                              D.ptr(grid), C.byref(err))
        raise_for(st, err, "jacobian_grid")

    def param_vjp(self, problem, U, theta, w, out):
        """out <- w_eff^T dR/dtheta at (U, theta) on the device (assembly.py:303-341)."""
        err = _lib.Error()
        st = _lib.lib().b200fem_param_vjp(self.ctx, D.ptr(U) if U is not None else None, D.ptr(theta), D.ptr(w),
                                          D.ptr(out), C.byref(err))
        raise_for(st, err, "param_vjp")

    def qp_flux(self, problem, U):
        self.sync(problem)
        out = D.empty(self.n_cells * 8 * self.vec * 3)
        err = _lib.Error()
        raise_for(_lib.lib().b200fem_qp_flux(self.ctx, D.ptr(U), D.ptr(out), C.byref(err)), err, "qp_flux")
        return out.view(self.n_cells, 8, self.vec, 3)

    def volume_average(self, problem, U) -> np.ndarray:
        self.sync(problem)
        out = np.zeros(self.vec * 3)
        err = _lib.Error()
        raise_for(_lib.lib().b200fem_volume_average_flux(self.ctx, D.ptr(U), D.hptr(out), C.byref(err)), err,
                  "volume_average")
        return out.reshape(self.vec, 3)

    def commit(self, U):
        Ud = D.to_device(U)
        raise_for(_lib.lib().b200fem_commit_state(self.ctx, D.ptr(Ud)), None, "commit")

    # ------------------------------------------------ host views (parity)
    def _cached(self, name, fn):
        if name not in self._cache:
            self._cache[name] = fn()
        return self._cache[name]

    @property
    def indptr(self) -> np.ndarray:
        def f():
            t = D.empty(self.n_dofs + 1, D.torch().int32)
            raise_for(_lib.lib().b200fem_copy_indptr(self.ctx, D.ptr(t)), None, "indptr")
            return D.to_host(t)
        return self._cached("indptr", f)

    @property
    def indices(self) -> np.ndarray:
        def f():
            t = D.empty(self.nnz, D.torch().int32)
            raise_for(_lib.lib().b200fem_copy_indices(self.ctx, D.ptr(t)), None, "indices")
            return D.to_host(t)
        return self._cached("indices", f)

    @property
    def diag_slots(self) -> np.ndarray:
        def f():
            t = D.empty(self.n_dofs, D.torch().int32)
            raise_for(_lib.lib().b200fem_copy_diag_slots(self.ctx, D.ptr(t)), None, "diag_slots")
            return D.to_host(t).astype(np.int64)
        return self._cached("diag", f)

    def dest_slice(self, lo, hi) -> np.ndarray:
        nd = 8 * self.vec
        t = D.empty((hi - lo) * nd * nd, D.torch().int32)
        raise_for(_lib.lib().b200fem_copy_dest(self.ctx, lo, hi, D.ptr(t)), None, "dest")
        return D.to_host(t).reshape(hi - lo, nd, nd)

    @property
    def dest(self) -> np.ndarray:
        return self._cached("dest", lambda: self.dest_slice(0, self.n_cells).astype(np.int64))

    def _geometry(self):
        pg = D.empty(self.n_cells * 8 * 8 * 3)
        jxw = D.empty(self.n_cells * 8)
        raise_for(_lib.lib().b200fem_geometry(self.ctx, D.ptr(pg), D.ptr(jxw)), None, "geometry")
        return D.to_host(pg).reshape(self.n_cells, 8, 8, 3), D.to_host(jxw).reshape(self.n_cells, 8)

    @property
    def phys_grads(self) -> np.ndarray:
        """(N_e, 8q, 8i, 3) physical shape-function gradients (Workspace.phys_grads, assembly.py:64-80;
        map_elements, elements.py:117-131), computed on the device on first access (the kernels
        recompute them per cell instead of streaming 1.5 KB/cell)."""
        if "geometry" not in self._cache:
            self._cache["geometry"] = self._geometry()
        return self._cache["geometry"][0]

    @property
    def JxW(self) -> np.ndarray:
        """(N_e, 8q) det J times the Gauss weights (all 1) (Workspace.JxW)."""
        if "geometry" not in self._cache:
            self._cache["geometry"] = self._geometry()
        return self._cache["geometry"][1]

    @property
    def shape_values(self) -> np.ndarray:
        """(8q, 8i) shape functions at the Gauss points (Workspace.shape_values)."""
        return shape_values_at_gauss()

    @property
    def edofs(self) -> np.ndarray:
        """(N_e, 8*vec) global DOF of each element-local DOF, node-major (assembly.py:94)."""
        return self._cache["edofs"]

    @property
    def dir_row_slots(self) -> np.ndarray:
        def f():
            ip = self.indptr
            if not self.dir_dofs.size:
                return np.empty(0, dtype=np.int64)
            return np.concatenate([np.arange(ip[d], ip[d + 1]) for d in self.dir_dofs])
        return self._cached("dir_rows", f)


def _edofs(mesh, vec):
    return (mesh.cells[:, :, None] * vec + np.arange(vec)).reshape(mesh.n_cells, 8 * vec)


def workspace(problem) -> DeviceWorkspace:
    """Build (once) and return the device assembly context of a problem."""
    ws = getattr(problem, "_ws", None)
    if ws is None:
        ws = DeviceWorkspace(problem)
        ws._cache["edofs"] = _edofs(problem.mesh, problem.vec)
        problem._ws = ws
    return ws


def assemble_residual(problem, U, apply_dirichlet: bool = True):
    """Weak-form residual at U minus loads; Dirichlet rows -> U[d] - scale*u_D (assembly.py:236-261)."""
    ws = workspace(problem)
    n = problem.n_dofs
    as_host = not D.is_device_tensor(U)
    Ud = D.to_device(U)
    if tuple(Ud.shape) != (n,):
        raise ValueError(f"U must have shape ({n},), got {tuple(Ud.shape)}")
    R = D.empty(n)
    ws.residual(problem, Ud, R, apply_dirichlet)
    return D.to_host(R) if as_host else R


def impose_dirichlet_residual(R, U, mesh, vec, specs, scale: float = 1.0) -> np.ndarray:
    """Overwrite constrained rows of R with U[d] - scale*u_D(x_d) (host helper, assembly.py:264-270)."""
    dofs, values = _dirichlet_table(mesh, vec, specs)
    out = np.array(R, dtype=np.float64, copy=True)
    if dofs.size:
        out[dofs] = np.asarray(U)[dofs] - scale * values
    return out


def assemble_jacobian(problem, U) -> CsrMatrix:
    """dR/dU in the fixed CSR pattern, Dirichlet rows -> identity (assembly.py:273-300)."""
    ws = workspace(problem)
    Ud = D.to_device(U)
    if tuple(Ud.shape) != (problem.n_dofs,):
        raise ValueError(f"U must have shape ({problem.n_dofs},), got {tuple(Ud.shape)}")
    data = D.empty(ws.nnz)
    ws.jacobian(problem, Ud, data)
    return CsrMatrix._from_workspace(ws, data)


def assemble_param_vjp(problem, U, theta, w):
    """w^T (dR/dtheta) accumulated into design space (assembly.py:303-341).

    Constrained residual rows are design-independent: their w entries are zeroed.  SIMP
    problems return one entry per cell, a Poisson design source one per node.  Host inputs
    give a host array (drop-in); CUDA tensors stay on the device."""
    ws = workspace(problem)
    if problem.design_layout is None:
        raise ValueError("problem has no design parameters bound")
    as_host = not D.is_device_tensor(w)
    Ud = D.to_device(U)
    if tuple(Ud.shape) != (problem.n_dofs,):
        raise ValueError(f"U must have shape ({problem.n_dofs},), got {tuple(Ud.shape)}")
    th = D.to_device(theta)
    if tuple(th.shape) != (problem.n_design,):
        raise ValueError(f"theta must have shape ({problem.n_design},), got {tuple(th.shape)}")
    wd = D.to_device(w)
    if tuple(wd.shape) != (problem.n_dofs,):
        raise ValueError(f"w must have shape ({problem.n_dofs},), got {tuple(wd.shape)}")
    out = D.empty(problem.n_design)
    ws.sync(problem)
    ws.param_vjp(problem, Ud, th, wd, out)
    return D.to_host(out) if as_host else out
