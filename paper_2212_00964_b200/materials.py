"""Constitutive laws (reference gradfem/materials.py:27-194).

The classes carry the constants and the identity of the law.  Every evaluation runs on the
GPU: inside the element kernels (csrc/element.cu) during assembly, and through
``b200fem_law_batch`` (csrc/material.cu, the same device functions of csrc/laws.cuh) when
host code calls a law directly -- ``Material.flux``, ``J2Plasticity.commit`` and the module
functions ``linear_elastic_flux``, ``neo_hookean_energy``, ``neo_hookean_flux``,
``j2_return_map``, ``commit_state`` keep the reference signatures (numpy in -> numpy out,
CUDA tensor in -> CUDA tensor out).  There is no host restatement of the laws.  Only the four
built-in laws are supported on the device path; a user class that overrides ``flux`` is
rejected with UnsupportedKernelError before any device work.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib


class InvertedDeformationError(ValueError):
    """det(F) <= 0: deformation state outside the model's domain (materials.py:19-24)."""

    def __init__(self, message, bad_mask=None):
        super().__init__(message)
        self.bad_mask = bad_mask


@dataclass(frozen=True)
class ElasticConstants:
    """E, nu (and sigma_yield) with derived lam, mu = G, kappa (materials.py:27-53)."""

    E: float
    nu: float
    sigma_yield: float = np.inf
    lam: float = field(init=False)
    mu: float = field(init=False)
    G: float = field(init=False)
    kappa: float = field(init=False)

    def __post_init__(self):
        if not self.E > 0:
            raise ValueError(f"Young's modulus must be positive, got {self.E}")
        if not (-1.0 < self.nu < 0.5):
            raise ValueError(f"Poisson's ratio must lie in (-1, 0.5), got {self.nu}")
        if not self.sigma_yield > 0:
            raise ValueError(f"yield strength must be positive, got {self.sigma_yield}")
        E, nu = self.E, self.nu
        object.__setattr__(self, "lam", E * nu / ((1 + nu) * (1 - 2 * nu)))
        object.__setattr__(self, "mu", E / (2 * (1 + nu)))
        object.__setattr__(self, "G", E / (2 * (1 + nu)))
        object.__setattr__(self, "kappa", E / (3 * (1 - 2 * nu)))


@dataclass
class QuadPointState:
    """Committed strain / stress per quadrature point, (..., 3, 3) each."""

    eps_prev: np.ndarray
    sig_prev: np.ndarray

    @staticmethod
    def fresh(shape=()) -> "QuadPointState":
        return QuadPointState(np.zeros(tuple(shape) + (3, 3)), np.zeros(tuple(shape) + (3, 3)))


class _DeviceLaw:
    vec = 3
    path_dependent = False
    linear = False
    material_id = -1

    def device_params(self):
        """[alpha, lam, mu, kappa, sigma_yield, penalty, 0, 0] for b200fem_ctx_create."""
        raise NotImplementedError

    def flux(self, grad_u, state=None):
        """Flux at a batch of points, evaluated on the device (materials.py:139-194)."""
        return law_batch(self, grad_u, state)["flux"]

    def tangent(self, grad_u, state=None):
        """d flux / d grad_u, (..., vec, 3, vec, 3): the hand tangent the element kernels use
        (the reference obtains it by forward-mode AD of ``flux``, autodiff.py:294-310)."""
        return law_batch(self, grad_u, state, flux=False, tangent=True)["tangent"]


class LinearElastic(_DeviceLaw):
    """sigma = lam tr(eps) I + 2 mu eps, eps = sym grad u (materials.py:74-77)."""

    linear = True
    material_id = _lib.MAT_LE

    def __init__(self, constants: ElasticConstants):
        self.constants = constants

    def device_params(self):
        c = self.constants
        return [0.0, c.lam, c.mu, c.kappa, 0.0, 0.0, 0.0, 0.0]


class NeoHookean(_DeviceLaw):
    """P = dW/dF, W = G/2 (J^-2/3 I1 - 3) + kappa/2 (J-1)^2 (materials.py:80-101)."""

    material_id = _lib.MAT_NH

    def __init__(self, constants: ElasticConstants):
        self.constants = constants

    def device_params(self):
        c = self.constants
        return [0.0, c.lam, c.G, c.kappa, 0.0, 0.0, 0.0, 0.0]


class J2Plasticity(_DeviceLaw):
    """Perfect J2 plasticity, radial return from committed state (materials.py:104-131)."""

    path_dependent = True
    material_id = _lib.MAT_J2

    def __init__(self, constants: ElasticConstants):
        if not np.isfinite(constants.sigma_yield):
            raise ValueError("J2 plasticity requires a finite sigma_yield")
        self.constants = constants

    def device_params(self):
        c = self.constants
        return [0.0, c.lam, c.mu, c.kappa, c.sigma_yield, 0.0, 0.0, 0.0]

    def commit(self, grad_u, state: "QuadPointState") -> "QuadPointState":
        """State for the next load step (materials.py:125-131, 168-169)."""
        out = law_batch(self, grad_u, state, flux=False, commit=True)
        return QuadPointState(out["eps"], out["sig"])


class IsotropicDiffusion(_DeviceLaw):
    """Scalar flux alpha grad u (materials.py:181-194)."""

    vec = 1
    linear = True
    material_id = _lib.MAT_POISSON

    def __init__(self, alpha: float = 1.0):
        if not alpha > 0:
            raise ValueError(f"diffusivity must be positive, got {alpha}")
        self.alpha = alpha

    def device_params(self):
        return [float(self.alpha), 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0]


BUILTIN_LAWS = (LinearElastic, NeoHookean, J2Plasticity, IsotropicDiffusion)


# ---------------------------------------------------------------- device batch evaluation
def law_batch(material, grad_u, state=None, flux=True, tangent=False, commit=False):
    """Evaluate a built-in law at every point of ``grad_u`` (..., vec, 3) on the device.

    Returns a dict with "flux" (..., vec, 3), "tangent" (..., vec, 3, vec, 3), "eps"/"sig"
    (J2 commit, (..., 3, 3)) as requested -- numpy for numpy input, CUDA tensors for CUDA
    input.  NH points with det F <= 0 raise InvertedDeformationError with ``bad_mask``
    (materials.py:94-100)."""
    import ctypes as C

    from . import _device as D
    from .errors import raise_for

    if not isinstance(material, BUILTIN_LAWS):
        raise TypeError(f"{type(material).__name__} is not a built-in law")
    vec = material.vec
    host = not D.is_device_tensor(grad_u)
    g = D.to_device(grad_u)
    shape = tuple(g.shape)
    if vec == 3 and shape[-2:] != (3, 3):
        raise ValueError(f"grad_u must have shape (..., 3, 3), got {shape}")
    if vec == 1 and (len(shape) < 1 or shape[-1] != 3):
        raise ValueError(f"grad_u must have shape (..., 3) or (..., 1, 3), got {shape}")
    lead = shape[:-2] if (vec == 3 or (len(shape) >= 2 and shape[-2] == 1)) else shape[:-1]
    n = int(np.prod(lead)) if lead else 1
    g = g.reshape(n, vec * 3).contiguous()
    ep = sp = None
    if isinstance(material, J2Plasticity):
        if state is None:
            raise ValueError("J2Plasticity needs the committed QuadPointState")
        ep, sp = _state_rows(state.eps_prev, lead), _state_rows(state.sig_prev, lead)
    out = {}
    fl = D.empty(n * vec * 3) if flux else None
    tg = D.empty(n * 9 * vec * vec) if tangent else None
    eo = D.empty(n * 9) if commit else None
    so = D.empty(n * 9) if commit else None
    det = D.empty(n) if isinstance(material, NeoHookean) else None
    params = (C.c_double * 8)(*material.device_params())
    err = _lib.Error()
    st = _lib.lib().b200fem_law_batch(material.material_id, C.cast(params, C.c_void_p), n, D.ptr(g),
                                      D.ptr(ep) if ep is not None else None, D.ptr(sp) if sp is not None else None,
                                      D.ptr(fl) if fl is not None else None, D.ptr(tg) if tg is not None else None,
                                      D.ptr(eo) if eo is not None else None, D.ptr(so) if so is not None else None,
                                      D.ptr(det) if det is not None else None, D.stream(), C.byref(err))
    if st == _lib.E_INVERTED_DEFORMATION:
        bad = (det <= 0.0).reshape(lead)
        raise InvertedDeformationError(err.message, bad_mask=D.to_host(bad) if host else bad)
    raise_for(st, err, "law_batch")
    conv = D.to_host if host else (lambda x: x)
    if fl is not None:
        out["flux"] = conv(fl.reshape(shape))
    if tg is not None:
        out["tangent"] = conv(tg.reshape(shape + shape[len(lead):]))
    if eo is not None:
        out["eps"] = conv(eo.reshape(lead + (3, 3)))
        out["sig"] = conv(so.reshape(lead + (3, 3)))
    return out


def _state_rows(x, lead):
    """Committed-state array broadcast to the batch, as (n, 9) device rows."""
    from . import _device as D

    if D.is_device_tensor(x):
        return x.to(D.torch().float64).expand(lead + (3, 3)).reshape(-1, 9).contiguous()
    return D.to_device(np.ascontiguousarray(np.broadcast_to(np.asarray(x, dtype=np.float64), lead + (3, 3)))).reshape(-1, 9)


def linear_elastic_flux(grad_u, constants: ElasticConstants):
    """Cauchy stress lam tr(eps) I + 2 mu eps, eps = sym(grad u) (materials.py:74-77), on the device."""
    return law_batch(LinearElastic(constants), grad_u)["flux"]


def neo_hookean_flux(grad_u, constants: ElasticConstants):
    """First Piola-Kirchhoff stress P = dW/dF at F = I + grad u (materials.py:88-101), on the device."""
    return law_batch(NeoHookean(constants), grad_u)["flux"]


def neo_hookean_energy(F, constants: ElasticConstants):
    """W(F) = G/2 (J^{-2/3} I1 - 3) + kappa/2 (J - 1)^2 (materials.py:80-85), on the device."""
    import ctypes as C

    from . import _device as D
    from .errors import raise_for

    host = not D.is_device_tensor(F)
    f = D.to_device(F)
    if tuple(f.shape[-2:]) != (3, 3):
        raise ValueError(f"F must have shape (..., 3, 3), got {tuple(f.shape)}")
    lead = tuple(f.shape[:-2])
    n = int(np.prod(lead)) if lead else 1
    f = f.reshape(n, 9).contiguous()
    W = D.empty(n)
    params = (C.c_double * 8)(*NeoHookean(constants).device_params())
    raise_for(_lib.lib().b200fem_nh_energy_batch(C.cast(params, C.c_void_p), n, D.ptr(f), D.ptr(W), D.stream()),
              None, "nh_energy")
    W = W.reshape(lead)
    if host:
        out = D.to_host(W)
        return out[()] if out.ndim == 0 else out
    return W


def j2_return_map(grad_u_k, state: QuadPointState, constants: ElasticConstants):
    """Radially returned stress of perfect J2 plasticity (materials.py:104-122), on the device."""
    return law_batch(J2Plasticity(constants), grad_u_k, state)["flux"]


def commit_state(grad_u_k, state: QuadPointState, constants: ElasticConstants) -> QuadPointState:
    """State for the next load step: eps <- sym grad u, sig <- return map (materials.py:125-131)."""
    out = law_batch(J2Plasticity(constants), grad_u_k, state, flux=False, commit=True)
    return QuadPointState(out["eps"], out["sig"])
