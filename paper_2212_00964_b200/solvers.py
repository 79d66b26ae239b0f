"""Linear, Newton and incremental-load solvers (reference gradfem/solvers.py:40-349).

The Newton and load-step loops stay Python (north_star); every vector stays on the
device between iterations and each linear solve is one C-ABI call that runs the whole
BiCGSTAB recurrence on the GPU (csrc/krylov.cu).  Host arrays in -> host arrays out, CUDA
tensors in -> CUDA tensors out.
"""

from __future__ import annotations

import csv
import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _device as D
from . import _lib
from .assembly import assemble_jacobian, workspace
from .errors import BreakdownError, LinearSolverError, NonConvergenceError, raise_for
from .mesh import BoundaryLocator, locate_nodes
from .sparse import CsrMatrix, GridOperator, SymOperator

__all__ = ["LinearSolveConfig", "NewtonConfig", "LoadSchedule", "LinearSolverError", "BreakdownError",
           "NonConvergenceError", "bicgstab_jacobi", "pcg_jacobi", "newton_solve", "incremental_solve", "reaction_force",
           "quad_point_stress", "volume_averaged_stress", "NewtonReport", "StepRecord", "LoadHistory"]


@dataclass(frozen=True)
class LinearSolveConfig:
    rel_tol: float = 1e-10
    abs_tol: float = 1e-12
    max_iters: int = 0  # 0 -> 10 * N
    # "bicgstab" = the reference solver (solvers.py:87-167, default); "pcg" = Jacobi-CG for
    # symmetric tangents (north_star "CG/BiCGSTAB", BASELINE config 2), same stopping rule
    method: str = "bicgstab"
    # operator of the Newton-loop solves (all the same linear operator as the assembled CSR):
    #  "auto" (default) = "grid" when the mesh is a box lattice and vec = 3, else "csr";
    #  "csr"  = the assembled reference CSR values;
    #  "grid" = GRID3: self + 13 upper-offset node blocks, offset-major (half the DRAM bytes,
    #           lower blocks re-read from L2 as contiguous slices; csrc/spmv.cu);
    #  "sym"  = symmetric node-block storage for any vec-3 mesh (L2-gather bound: 1.64 ms vs
    #           0.85 ms per config-3 matvec, profiles/)
    #  "grid32" = opt-in inexact Newton: GRID3 with the values rounded to FP32 (half the
    #           bytes; FP64 vectors, products and sums; FP64 residual and Newton test), for
    #           vec-3 box lattices only.  NOT the reference's FP64 operator.
    operator: str = "auto"

    def __post_init__(self):
        if self.rel_tol <= 0 or self.abs_tol <= 0:
            raise ValueError("linear solver tolerances must be positive")
        if self.method not in ("bicgstab", "pcg"):
            raise ValueError(f"unknown linear solver {self.method!r}")
        if self.operator not in ("auto", "grid", "sym", "csr", "grid32"):
            raise ValueError(f"unknown operator {self.operator!r}")


@dataclass(frozen=True)
class NewtonConfig:
    rel_tol: float = 1e-8
    abs_tol: float = 1e-10
    max_iters: int = 20

    def __post_init__(self):
        if self.rel_tol <= 0 or self.abs_tol <= 0:
            raise ValueError("Newton tolerances must be positive")


@dataclass(frozen=True)
class LoadSchedule:
    """Ordered boundary-value scale factors (solvers.py:62-84)."""

    factors: tuple

    def __post_init__(self):
        f = tuple(float(v) for v in self.factors)
        if not f:
            raise ValueError("load schedule must contain at least one step")
        if not all(np.isfinite(f)):
            raise ValueError("load schedule factors must be finite")
        object.__setattr__(self, "factors", f)

    @staticmethod
    def ramp(n_steps: int, amplitude: float = 1.0) -> "LoadSchedule":
        return LoadSchedule(tuple(amplitude * (k + 1) / n_steps for k in range(n_steps)))

    @staticmethod
    def ramp_and_back(n_steps: int, amplitude: float = 1.0) -> "LoadSchedule":
        up = [amplitude * (k + 1) / n_steps for k in range(n_steps)]
        return LoadSchedule(tuple(up + [amplitude * (n_steps - 1 - k) / n_steps for k in range(n_steps)]))


@dataclass
class SolveStats:
    iterations: int = 0
    matvecs: int = 0
    restarts: int = 0
    residual: float = 0.0
    tol: float = 0.0


def _bicgstab_device(A: CsrMatrix, b, x, has_x0: bool, cfg: LinearSolveConfig, method=None) -> SolveStats:
    info = _lib.SolveInfo()
    err = _lib.Error()
    method = method or cfg.method
    fn = _lib.lib().b200fem_pcg if method == "pcg" else _lib.lib().b200fem_bicgstab
    st = fn(A._device_handle(), D.ptr(b), D.ptr(x), int(has_x0), float(cfg.rel_tol), float(cfg.abs_tol),
            int(cfg.max_iters), C.byref(info), C.byref(err))
    raise_for(st, err, method)
    return SolveStats(info.iterations, info.matvecs, info.restarts, info.residual, info.tol)


def bicgstab_jacobi(A: CsrMatrix, b, x0=None, cfg: LinearSolveConfig = LinearSolveConfig(), stats=None):
    """Solve A x = b by left-Jacobi BiCGSTAB on the GPU (solvers.py:87-167 semantics).

    Terminates on the true residual ||A x - b|| <= max(rel_tol ||b||, abs_tol); raises
    LinearSolverError at max_iters and BreakdownError when a restart makes no progress."""
    as_host = not D.is_device_tensor(b)
    bd = D.to_device(b)
    n = A.shape[0]
    if tuple(bd.shape) != (n,):
        raise ValueError(f"b must have shape ({n},), got {tuple(bd.shape)}")
    x = D.zeros(n) if x0 is None else D.to_device(x0, copy=True)
    s = _bicgstab_device(A, bd, x, x0 is not None, cfg, method="bicgstab")
    if stats is not None:
        stats.append(s)
    return D.to_host(x) if as_host else x


def pcg_jacobi(A: CsrMatrix, b, x0=None, cfg: LinearSolveConfig = LinearSolveConfig(), stats=None):
    """Solve A x = b by Jacobi-preconditioned CG on the GPU (symmetric A; FEM matrices with
    Dirichlet identity rows are handled by starting from x_d = b_d).  Same termination rule
    and exceptions as bicgstab_jacobi; BreakdownError if A is found not positive definite."""
    as_host = not D.is_device_tensor(b)
    bd = D.to_device(b)
    n = A.shape[0]
    if tuple(bd.shape) != (n,):
        raise ValueError(f"b must have shape ({n},), got {tuple(bd.shape)}")
    x = D.zeros(n) if x0 is None else D.to_device(x0, copy=True)
    s = _bicgstab_device(A, bd, x, x0 is not None, cfg, method="pcg")
    if stats is not None:
        stats.append(s)
    return D.to_host(x) if as_host else x


@dataclass
class NewtonReport:
    residual_norms: list
    n_iterations: int
    converged: bool
    linear_stats: list = field(default_factory=list)
    # device time per phase (CUDA events on the solve's stream): residual, jacobian, linear
    timings: dict = field(default_factory=dict)


def _tangent_matrix(problem, U, operator="csr"):
    """K at U; cached for jacobian_constant problems (solvers.py:177-184)."""
    ws = workspace(problem)
    if operator == "grid32":
        if not (ws.has_grid and problem.vec == 3):
            raise ValueError('operator "grid32" needs a vec-3 box-lattice problem')
        K = ws._cache.get("newton_grid32")
        if K is None:  # one FP64 GRID3 value buffer for both Newton operators (2.6 GB at config 3)
            base = ws._cache.get("newton_grid")
            K = GridOperator(ws, data=base.device_data if base is not None else None)
            ws._cache["newton_grid32"] = K
        ws.jacobian_grid(problem, U, K.device_data)
        K.refresh_f32()
        return K
    if operator in ("auto", "grid") and ws.has_grid:
        if problem.jacobian_constant:
            K = getattr(problem, "_jac_cache", None)
            if isinstance(K, GridOperator):
                return K
        K = ws._cache.get("newton_grid")
        if K is None:
            other = ws._cache.get("newton_grid32")
            K = GridOperator(ws, data=other.device_data if other is not None else None)
            ws._cache["newton_grid"] = K
        ws.jacobian_grid(problem, U, K.device_data)
        if problem.jacobian_constant:
            problem._jac_cache = K
        return K
    if operator == "sym" and ws.has_sym:
        key = "newton_sym"
        if problem.jacobian_constant:
            K = getattr(problem, "_jac_cache", None)
            if isinstance(K, SymOperator):
                return K
        K = ws._cache.get(key)
        if K is None:
            K = SymOperator(ws)
            ws._cache[key] = K
        ws.jacobian_sym(problem, U, K.device_data)
        if problem.jacobian_constant:
            problem._jac_cache = K
        return K
    if problem.jacobian_constant:
        K = getattr(problem, "_jac_cache", None)
        if not isinstance(K, CsrMatrix):
            data = D.empty(ws.nnz)
            ws.jacobian(problem, U, data)
            K = CsrMatrix._from_workspace(ws, data)
            problem._jac_cache = K
        return K
    K = ws._cache.get("newton_K")
    if K is None:
        K = CsrMatrix._from_workspace(ws, D.empty(ws.nnz))
        ws._cache["newton_K"] = K
    ws.jacobian(problem, U, K.device_data)
    return K


class _PhaseTimer:
    """CUDA-event phase accounting (no host synchronisation added)."""

    def __init__(self):
        self.events = []

    def mark(self, phase):
        ev = D.torch().cuda.Event(enable_timing=True)
        ev.record()
        self.events.append((phase, ev))

    def totals(self):
        out = {}
        if self.events:
            self.events[-1][1].synchronize()  # the closing mark may still be in flight
        for (ph, a), (_, b) in zip(self.events, self.events[1:]):
            out[ph] = out.get(ph, 0.0) + a.elapsed_time(b) / 1e3
        return out


def _newton_device(problem, U, cfg: NewtonConfig, lin_cfg: LinearSolveConfig):
    """Newton on device vectors; U (CUDA tensor) is updated in place."""
    ws = workspace(problem)
    n = problem.n_dofs
    R = D.empty(n)
    rhs = D.empty(n)
    dU = D.empty(n)
    lib = _lib.lib()
    stream = D.stream()
    tm = _PhaseTimer()
    tm.mark("residual_s")
    norms = [ws.residual(problem, U, R)]
    r0 = norms[0]
    lin = []

    def report(its, ok):
        tm.mark("end")
        return NewtonReport(norms, its, ok, lin, tm.totals())

    for it in range(cfg.max_iters):
        if norms[-1] <= max(cfg.rel_tol * r0, cfg.abs_tol):
            return U, report(it, True)
        tm.mark("jacobian_s")
        K = _tangent_matrix(problem, U, lin_cfg.operator)
        tm.mark("linear_s")
        lib.b200fem_scale(n, -1.0, D.ptr(R), D.ptr(rhs), stream)
        lin.append(_bicgstab_device(K, rhs, dU, False, lin_cfg))
        lib.b200fem_axpy(n, 1.0, D.ptr(dU), D.ptr(U), stream)
        tm.mark("residual_s")
        norms.append(ws.residual(problem, U, R))
    if norms[-1] <= max(cfg.rel_tol * r0, cfg.abs_tol):
        return U, report(cfg.max_iters, True)
    raise NonConvergenceError(
        f"Newton did not converge in {cfg.max_iters} iterations "
        f"(residual history {['%.3e' % v for v in norms]})", residual_norms=norms)


def tangent_transpose(problem, U) -> CsrMatrix:
    """Transpose of the (Dirichlet-modified) tangent at U (solvers.py:187-195), on the device;
    cached for jacobian_constant problems."""
    if problem.jacobian_constant:
        cached = getattr(problem, "_jac_t_cache", None)
        if cached is None:
            K = _tangent_matrix(problem, D.to_device(U), "csr")
            if not isinstance(K, CsrMatrix):  # a symmetric-storage cache: assemble the CSR
                K = assemble_jacobian(problem, U)
            cached = K.transpose()
            problem._jac_t_cache = cached
        return cached
    return assemble_jacobian(problem, U).transpose()


def newton_solve(problem, U0=None, cfg: NewtonConfig = NewtonConfig(),
                 lin_cfg: LinearSolveConfig = LinearSolveConfig()):
    """Newton iteration on the assembled residual (solvers.py:198-227); returns (U, NewtonReport).

    Runs on the workspace's stream (the one every assembly and Krylov kernel of this problem
    is bound to), ordered after the caller's current stream and before its later work."""
    as_host = U0 is None or not D.is_device_tensor(U0)
    ws = workspace(problem)
    with ws.on_stream() as caller:
        U = D.zeros(problem.n_dofs) if U0 is None else D.to_device(U0, copy=True)
        if tuple(U.shape) != (problem.n_dofs,):
            raise ValueError(f"U0 must have shape ({problem.n_dofs},)")
        U, rep = _newton_device(problem, U, cfg, lin_cfg)
        if caller is not None and not as_host:
            U.record_stream(caller)
    return (D.to_host(U) if as_host else U), rep


def reaction_force(problem, U, locator: BoundaryLocator, component: int) -> float:
    """Unconstrained residual summed over the located DOFs (solvers.py:230-234)."""
    ws = workspace(problem)
    Ud = D.to_device(U)
    R = D.empty(problem.n_dofs)
    ws.residual(problem, Ud, R, apply_dirichlet=False)
    idx = locate_nodes(problem.mesh, locator).astype(np.int64) * problem.vec + component
    if idx.size == 0:
        return 0.0
    di = D.to_device(idx, D.torch().int64)
    out = C.c_double()
    raise_for(_lib.lib().b200fem_gather_sum(D.ptr(R), D.ptr(di), idx.size, C.byref(out), D.stream()), None,
              "gather_sum")
    return float(out.value)


def quad_point_stress(problem, U):
    """Flux at every quadrature point, (N_e, 8, vec, 3) (solvers.py:237-250)."""
    as_host = not D.is_device_tensor(U)
    out = workspace(problem).qp_flux(problem, D.to_device(U))
    return D.to_host(out) if as_host else out


def volume_averaged_stress(problem, U) -> np.ndarray:
    """Volume average of the flux, (vec, 3) (solvers.py:253-258)."""
    return workspace(problem).volume_average(problem, D.to_device(U))


@dataclass
class StepRecord:
    step: int
    scale: float
    U: np.ndarray
    newton_iterations: int
    residual_norm: float
    residual_history: list = field(default_factory=list)
    reaction: Optional[float] = None
    avg_stress: Optional[np.ndarray] = None


@dataclass
class LoadHistory:
    steps: list = field(default_factory=list)

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "scale", "newton_iterations", "residual_norm", "reaction", "avg_stress_zz"])
            for r in self.steps:
                w.writerow([r.step, repr(r.scale), r.newton_iterations, repr(r.residual_norm),
                            "" if r.reaction is None else repr(r.reaction),
                            "" if r.avg_stress is None else repr(float(r.avg_stress[-1, -1]))])

    def write_newton_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["step", "iteration", "residual_norm"])
            for r in self.steps:
                for i, v in enumerate(r.residual_history):
                    w.writerow([r.step, i, repr(v)])


def incremental_solve(problem, schedule: LoadSchedule, cfg: NewtonConfig = NewtonConfig(),
                      lin_cfg: LinearSolveConfig = LinearSolveConfig(),
                      reaction_locator: Optional[BoundaryLocator] = None, reaction_component: int = 2,
                      record_stress: bool = True, on_step=None) -> LoadHistory:
    """Quasi-static driver: scale boundary data, warm-started Newton, record, commit (solvers.py:305-349)."""
    ws = workspace(problem)
    hist = LoadHistory()
    U = D.zeros(problem.n_dofs)
    for k, factor in enumerate(schedule.factors):
        problem.bc_scale = factor
        try:
            U, rep = _newton_device(problem, U, cfg, lin_cfg)
        except (NonConvergenceError, LinearSolverError) as err:
            raise NonConvergenceError(f"load step {k} (scale {factor}) failed: {err}", step=k) from err
        rec = StepRecord(step=k, scale=factor, U=D.to_host(U), newton_iterations=rep.n_iterations,
                         residual_norm=rep.residual_norms[-1], residual_history=list(rep.residual_norms))
        if record_stress:
            rec.avg_stress = ws.volume_average(problem, U)
        if reaction_locator is not None:
            rec.reaction = reaction_force(problem, U, reaction_locator, reaction_component)
        if on_step is not None:
            on_step(rec)
        if problem.material.path_dependent:
            problem.commit(U)
        hist.steps.append(rec)
    return hist
