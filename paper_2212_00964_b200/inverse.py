"""Objectives of the two shipped design applications (reference inverse.py), as far as the
adjoint row needs them: the Poisson observation misfit and the SIMP compliance.

The compliance is the work of the boundary tractions.  The reference integrates u . t over
the loaded facets (inverse.py:157-176); that is exactly U . F_N with F_N the assembled
traction load vector (same quadrature, same shape functions), so it is evaluated here as one
device dot product with the workspace's load vector (agreement to round-off)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as D
from . import _lib
from .assembly import workspace
from .errors import raise_for

__all__ = ["poisson_objective", "poisson_objective_gradient", "compliance", "compliance_load_vector"]


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
