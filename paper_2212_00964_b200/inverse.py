"""The two shipped design applications (reference inverse.py): Poisson source inference and
SIMP compliance topology optimisation, with their per-iteration vector work on the device
(SURVEY 8(f) f2): density filter (csrc/design.cu), filtered sensitivities, the MMA update
and the L2 field error.  The drivers (run_inference, run_topopt) are host loops, as in the
reference.

The compliance is the work of the boundary tractions.  The reference integrates u . t over
the loaded facets (inverse.py:157-176); that is exactly U . F_N with F_N the assembled
traction load vector (same quadrature, same shape functions), so it is evaluated here as one
device dot product with the workspace's load vector (agreement to round-off)."""

from __future__ import annotations

import csv
import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _device as D
from . import _lib
from .assembly import workspace
from .errors import raise_for

__all__ = ["THETA_MIN", "poisson_objective", "poisson_objective_gradient", "l2_field_error", "InferenceResult",
           "run_inference", "compliance", "compliance_load_vector", "FilterOperator", "element_centroids",
           "density_filter", "filter_sensitivities", "MmaState", "mma_update", "TopOptResult", "run_topopt"]

THETA_MIN = 1e-3


def _mesh_device(mesh):
    """(coords, int32 cells) of a mesh on the device, uploaded once per mesh."""
    geo = getattr(mesh, "_dev_geom", None)
    if geo is None:
        geo = (D.to_device(np.ascontiguousarray(mesh.nodes, dtype=np.float64)),
               D.to_device(np.ascontiguousarray(mesh.cells, dtype=np.int32), D.torch().int32))
        object.__setattr__(mesh, "_dev_geom", geo)
    return geo


def _dev(a, n=None):
    """float64 device vector (scalars / host arrays broadcast to n)."""
    if D.is_device_tensor(a):
        t = a.to(D.torch().float64)
        return t.expand(n).contiguous() if (n is not None and t.dim() == 0) else t.contiguous()
    arr = np.asarray(a, dtype=np.float64)
    if n is not None:
        arr = np.broadcast_to(arr, (n,))
    return D.to_device(np.ascontiguousarray(arr))


def poisson_objective(U, obs_indices, obs_values) -> float:
    """Sum of squared misfits at the observed DOFs (inverse.py:31-35)."""
    u = D.to_host(U) if D.is_device_tensor(U) else np.asarray(U)
    r = u[np.asarray(obs_indices)] - np.asarray(obs_values)
    return float(np.dot(r, r))


def poisson_objective_gradient(U, obs_indices, obs_values) -> np.ndarray:
    """d/dU of poisson_objective (inverse.py:38-42)."""
    u = D.to_host(U) if D.is_device_tensor(U) else np.asarray(U)
    idx = np.asarray(obs_indices)
    g = np.zeros(u.shape[0])
    g[idx] = 2.0 * (u[idx] - np.asarray(obs_values))
    return g


def compliance_load_vector(problem) -> np.ndarray:
    """dJ/dU of the compliance: the assembled traction load vector (inverse.py:179-182)."""
    return problem.bc_scale * workspace(problem).f_neumann


def compliance(problem, U) -> float:
    """Work of the boundary tractions, U . (bc_scale F_N), on the device."""
    f = D.to_device(compliance_load_vector(problem))
    u = D.to_device(U)
    if tuple(u.shape) != tuple(f.shape):
        raise ValueError(f"U must have shape ({f.shape[0]},), got {tuple(u.shape)}")
    out = C.c_double()
    raise_for(_lib.lib().b200fem_dot(D.ptr(u), D.ptr(f), f.shape[0], C.byref(out), D.stream()), None, "dot")
    return float(out.value)


# -------------------------------------------------------------- inference
def l2_field_error(mesh, u_pred, u_true) -> float:
    """Relative L2 error ||u_pred - u_true|| / ||u_true|| by quadrature (inverse.py:45-56)."""
    X, cells = _mesh_device(mesh)
    up, ut = _dev(u_pred), _dev(u_true)
    out = (C.c_double * 2)()
    raise_for(_lib.lib().b200fem_l2_field_error(mesh.n_cells, D.ptr(X), D.ptr(cells), D.ptr(up), D.ptr(ut), out,
                                                D.stream()), None, "l2_field_error")
    with np.errstate(divide="ignore", invalid="ignore"):
        return float(np.sqrt(out[0]) / np.sqrt(out[1]))


@dataclass
class InferenceResult:
    theta: np.ndarray
    u_pred: np.ndarray
    u_true: np.ndarray
    obs_indices: np.ndarray
    objective_history: list
    error_history: list
    relative_l2_error: float

    def write_csv(self, path) -> None:
        _write_rows(path, ["step", "objective", "relative_l2_error"],
                    [[k, repr(o), repr(e)] for k, (o, e) in enumerate(zip(self.objective_history, self.error_history))])


def _write_rows(path, header, rows):
    with open(path, "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(header)
        wr.writerows(rows)


def run_inference(problem, true_source: Callable, n_obs: int, seed: int = 0, max_iters: int = 100,
                  lin_cfg=None, observe_all: bool = False) -> InferenceResult:
    """Recover the nodal Poisson source from sparse observations (inverse.py:68-150): ground
    truth from a forward solve with ``true_source`` at the nodes, observations drawn (seeded)
    from the unconstrained nodes, L-BFGS on the adjoint-gradient reduced objective."""
    from scipy.optimize import minimize

    from .adjoint import OptimizeHistory, ReducedObjective
    from .solvers import LinearSolveConfig, NewtonConfig, newton_solve

    if problem.design_layout != "node":
        raise ValueError("inference requires a PoissonProblem with design_source=True")
    lin_cfg = lin_cfg or LinearSolveConfig()
    mesh = problem.mesh
    ncfg = NewtonConfig(rel_tol=1e-10, abs_tol=1e-10)
    theta_true = np.array([true_source(x) for x in mesh.nodes], dtype=np.float64)
    problem.set_theta(theta_true)
    u_true, _ = newton_solve(problem, cfg=ncfg, lin_cfg=lin_cfg)
    free = np.setdiff1d(np.arange(mesh.n_nodes), workspace(problem).dir_dofs)
    if observe_all:
        obs = np.arange(mesh.n_nodes)
    else:
        if not 0 < n_obs <= free.size:
            raise ValueError(f"n_obs must lie in [1, {free.size}], got {n_obs}")
        obs = np.sort(np.random.default_rng(seed).choice(free, size=n_obs, replace=False))
    obs_values = u_true[obs]
    obj = ReducedObjective(problem, objective=lambda U, t: poisson_objective(U, obs, obs_values),
                           dj_du=lambda U, t: poisson_objective_gradient(U, obs, obs_values),
                           newton_cfg=ncfg, lin_cfg=lin_cfg)
    hist, errs = OptimizeHistory(), []

    def fun(t):
        v, g = obj.value_and_gradient(t)
        hist.record(v, g)
        errs.append(l2_field_error(mesh, obj._U_warm, u_true))
        return v, g

    res = minimize(fun, np.zeros(mesh.n_nodes), jac=True, method="L-BFGS-B",
                   options={"maxiter": max_iters, "gtol": 1e-12, "ftol": 1e-16})
    u_pred = obj.forward(res.x)
    return InferenceResult(theta=res.x, u_pred=u_pred, u_true=u_true, obs_indices=obs,
                           objective_history=hist.objective, error_history=errs,
                           relative_l2_error=l2_field_error(mesh, u_pred, u_true))


# -------------------------------------------------------------- filter
def element_centroids(mesh) -> np.ndarray:
    """Mean of the 8 vertex coordinates per cell (inverse.py:200-201)."""
    return mesh.cell_coords().mean(axis=1)


class FilterOperator:
    """Normalised hat-weight average over element centroids (inverse.py:186-197), built and
    applied on the device.  ``matrix`` is the same operator as a CsrMatrix."""

    def __init__(self, mesh, radius):
        X, cells = _mesh_device(mesh)
        h = C.c_void_p()
        raise_for(_lib.lib().b200fem_filter_create(C.byref(h), mesh.n_cells, D.ptr(X), D.ptr(cells), float(radius),
                                                   D.stream()), None, "filter_create")
        self._h = h
        self.n = mesh.n_cells
        self.radius = float(radius)
        self._matrix = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.b200fem_filter_destroy(h)
            except Exception:
                pass

    @property
    def nnz(self) -> int:
        nnz = C.c_int64()
        _lib.lib().b200fem_filter_info(self._h, None, C.byref(nnz))
        return nnz.value

    @property
    def matrix(self):
        if self._matrix is None:
            from .sparse import CsrMatrix

            t = D.torch()
            nnz = self.nnz
            indptr = D.empty(self.n + 1, t.int32)
            indices = D.empty(max(nnz, 1), t.int32)
            data = D.empty(max(nnz, 1))
            raise_for(_lib.lib().b200fem_filter_copy(self._h, D.ptr(indptr), D.ptr(indices), D.ptr(data)), None,
                      "filter_copy")
            self._matrix = CsrMatrix(D.to_host(indptr), D.to_host(indices)[:nnz], data[:nnz])
        return self._matrix

    def apply(self, field, mul=None, div=None, floor=0.0):
        as_host = not D.is_device_tensor(field)
        v = _dev(field)
        if tuple(v.shape) != (self.n,):
            raise ValueError(f"field must have shape ({self.n},), got {tuple(v.shape)}")
        m = _dev(mul) if mul is not None else None
        dv = _dev(div) if div is not None else None
        y = D.empty(self.n)
        raise_for(_lib.lib().b200fem_filter_apply(self._h, D.ptr(v), D.ptr(m) if m is not None else None,
                                                  D.ptr(dv) if dv is not None else None, float(floor), D.ptr(y)),
                  None, "filter_apply")
        return D.to_host(y) if as_host else y

    def __call__(self, field):
        return self.apply(field)


def density_filter(mesh, radius: float) -> FilterOperator:
    """Hat-weight averaging operator for the given radius (inverse.py:204-228)."""
    if not radius > 0:
        raise ValueError(f"filter radius must be positive, got {radius}")
    return FilterOperator(mesh, radius)


def filter_sensitivities(filt: FilterOperator, theta, sens, theta_floor=THETA_MIN):
    """Classic sensitivity blur H(theta * sens) / max(theta, floor) (inverse.py:231-234), one
    fused device pass."""
    return filt.apply(sens, mul=theta, div=theta, floor=theta_floor) if D.is_device_tensor(sens) else \
        filt.apply(np.asarray(sens, dtype=np.float64), mul=theta, div=theta, floor=theta_floor)


# -------------------------------------------------------------- MMA
@dataclass
class MmaState:
    """Asymptotes and the two previous iterates (inverse.py:240-257); device vectors."""

    lower: Optional[object] = None
    upper: Optional[object] = None
    x_prev: Optional[object] = None
    x_prev2: Optional[object] = None
    iteration: int = 0
    move_limit: float = 0.2
    asym_init: float = 0.5
    asym_expand: float = 1.2
    asym_shrink: float = 0.7

    @staticmethod
    def fresh(n: int, move_limit: float = 0.2) -> "MmaState":
        return MmaState(move_limit=move_limit)


def mma_update(state: MmaState, x, dj, g_value, g_grad, lb, ub):
    """One MMA step for a single linear inequality constraint g(x) <= 0 (inverse.py:260-346):
    convex separable moving-asymptote model of the objective, the linear constraint exact,
    the dual solved by bisection on its multiplier with per-variable bisection for the
    stationarity roots -- all on the device (csrc/design.cu)."""
    as_host = not D.is_device_tensor(x)
    xd = _dev(x)
    n = xd.shape[0]
    djd, cd, lbd, ubd = _dev(dj, n), _dev(g_grad, n), _dev(lb, n), _dev(ub, n)
    hist = state.iteration >= 2 and state.x_prev is not None and state.x_prev2 is not None
    low = _dev(state.lower, n).clone() if hist else D.empty(n)
    upp = _dev(state.upper, n).clone() if hist else D.empty(n)
    xp = _dev(state.x_prev, n) if hist else None
    xpp = _dev(state.x_prev2, n) if hist else None
    xn = D.empty(n)
    st = _lib.lib().b200fem_mma_update(n, D.ptr(xd), D.ptr(djd), float(g_value), D.ptr(cd), D.ptr(lbd), D.ptr(ubd),
                                       D.ptr(low), D.ptr(upp), D.ptr(xp) if hist else None,
                                       D.ptr(xpp) if hist else None, int(hist), float(state.asym_init),
                                       float(state.asym_expand), float(state.asym_shrink), float(state.move_limit),
                                       D.ptr(xn), D.stream())
    raise_for(st, None, "mma_update")
    state.lower, state.upper = low, upp
    state.x_prev2 = state.x_prev
    state.x_prev = xd.clone()
    state.iteration += 1
    return D.to_host(xn) if as_host else xn


# -------------------------------------------------------------- topology optimisation
@dataclass
class TopOptResult:
    theta: np.ndarray
    compliance_history: list
    volume_history: list
    final_compliance: float
    final_volume: float

    def write_csv(self, path) -> None:
        _write_rows(path, ["step", "compliance", "volume_fraction"],
                    [[k, repr(c), repr(v)] for k, (c, v) in enumerate(zip(self.compliance_history,
                                                                          self.volume_history))])


def run_topopt(problem, volume_fraction: float, n_steps: int, filter_radius: Optional[float] = None,
               design_mask=None, move_limit: float = 0.2, newton_cfg=None, lin_cfg=None,
               callback: Optional[Callable] = None) -> TopOptResult:
    """Compliance minimisation with volume-constrained MMA (inverse.py:367-432), starting from
    the uniform design theta = volume_fraction; each step: forward solve, adjoint compliance
    gradient, sensitivity filter, MMA update.  Cells outside ``design_mask`` stay solid."""
    from .adjoint import adjoint_solve, total_derivative
    from .solvers import LinearSolveConfig, NewtonConfig, newton_solve

    newton_cfg = newton_cfg or NewtonConfig()
    lin_cfg = lin_cfg or LinearSolveConfig()
    mesh = problem.mesh
    n_e = mesh.n_cells
    mask = np.ones(n_e, dtype=bool) if design_mask is None else np.asarray(design_mask, dtype=bool)
    if filter_radius is None:
        cc = mesh.cell_coords(0)
        filter_radius = 1.5 * float(np.linalg.norm(cc[1] - cc[0]))
    filt = density_filter(mesh, filter_radius)
    theta = np.full(n_e, float(volume_fraction))
    theta[~mask] = 1.0
    n_design = int(mask.sum())
    state = MmaState.fresh(n_design, move_limit=move_limit)
    g_grad = np.full(n_design, 1.0 / n_design)
    comp, vol = [], []
    U_warm = None
    for step in range(n_steps):
        problem.set_theta(theta)
        U, _ = newton_solve(problem, U_warm, cfg=newton_cfg, lin_cfg=lin_cfg)
        U_warm = U.copy()
        c = compliance(problem, U)
        comp.append(c)
        vol.append(float(theta[mask].mean()))
        lam = adjoint_solve(problem, U, compliance_load_vector(problem), lin_cfg=lin_cfg)
        sens = total_derivative(problem, U, lam, problem.theta)
        sens = filter_sensitivities(filt, problem.theta, sens, problem.theta_min)
        g_value = float(theta[mask].mean()) - volume_fraction
        new = theta.copy()
        new[mask] = mma_update(state, theta[mask], sens[mask], g_value, g_grad, problem.theta_min, 1.0)
        theta = new
        if callback is not None:
            callback(step, theta, c)
    problem.set_theta(theta)
    U, _ = newton_solve(problem, U_warm, cfg=newton_cfg, lin_cfg=lin_cfg)
    return TopOptResult(theta=theta, compliance_history=comp, volume_history=vol,
                        final_compliance=compliance(problem, U), final_volume=float(theta[mask].mean()))
