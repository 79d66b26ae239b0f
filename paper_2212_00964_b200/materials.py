"""Constitutive-law descriptors (reference gradfem/materials.py:27-194).

These classes carry the constants and the identity of the law; the flux and its
consistent tangent are evaluated on the GPU (csrc/element.cu).  Only the four built-in
laws are supported on the device path; a user class that overrides ``flux`` is rejected
with UnsupportedKernelError before any device work.
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

    def flux(self, grad_u, state=None):  # host evaluation is not part of the product path
        raise NotImplementedError(f"{type(self).__name__}.flux is evaluated on the GPU (csrc/element.cu)")


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
