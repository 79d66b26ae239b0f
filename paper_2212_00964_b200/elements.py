"""HEX8 reference element on the host: only what one-time setup needs (face and body
quadrature for the fixed load vectors, assembly.py:106-128).  Per-cell geometry for the
hot path is recomputed inside the device kernels (csrc/element.cu) instead of being
cached as the reference's (N_e, 8, 8, 3) phys_grads array (elements.py:117-131).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .mesh import HEX_FACES, Mesh

VERTEX_SIGNS = np.array(
    [[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]],
    dtype=np.float64)


class InvertedElementError(ValueError):
    """Non-positive Jacobian determinant at a quadrature point."""


def _gauss_1d():
    return 1.0 / np.sqrt(3.0)


@lru_cache(maxsize=1)
def _tables():
    g = _gauss_1d()
    qp = np.array([[x, y, z] for z in (-g, g) for y in (-g, g) for x in (-g, g)])  # x fastest
    t = 1.0 + qp[:, None, :] * VERTEX_SIGNS
    phi = t[..., 0] * t[..., 1] * t[..., 2] / 8.0
    return qp, phi


def shape_values_at_gauss() -> np.ndarray:
    """phi_k at the 8 Gauss points, (8 q, 8 k)."""
    return _tables()[1]


def quad_point_coords(mesh: Mesh) -> np.ndarray:
    """Physical quadrature-point positions, (N_e, 8, 3)."""
    return np.einsum("qk,nkd->nqd", shape_values_at_gauss(), mesh.cell_coords())


def cell_jxw(mesh: Mesh) -> np.ndarray:
    """det J at each Gauss point, (N_e, 8) — host setup only (body-force load)."""
    g = _gauss_1d()
    qp = _tables()[0]
    t = 1.0 + qp[:, None, :] * VERTEX_SIGNS  # (8q, 8k, 3)
    dN = np.stack([VERTEX_SIGNS[:, 0] * t[..., 1] * t[..., 2], VERTEX_SIGNS[:, 1] * t[..., 0] * t[..., 2],
                   VERTEX_SIGNS[:, 2] * t[..., 0] * t[..., 1]], axis=-1) / 8.0
    del g
    J = np.einsum("nka,qkb->nqab", mesh.cell_coords(), dN)
    return np.linalg.det(J)


@dataclass(frozen=True)
class FaceQuadrature:
    points: np.ndarray      # (F, 4q, 3)
    JxW: np.ndarray         # (F, 4q)
    shape_values: np.ndarray  # (4q, 4a)
    local_nodes: np.ndarray   # (F, 4a)


def face_quadrature(mesh: Mesh, facets: np.ndarray) -> FaceQuadrature:
    """2x2 Gauss rule on boundary faces; weight |t1 x t2| (elements.py:157-203)."""
    facets = np.asarray(facets, dtype=np.int64).reshape(-1, 2)
    g = _gauss_1d()
    q2 = np.array([[x, y] for y in (-g, g) for x in (-g, g)])
    s2 = np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], dtype=np.float64)
    t = 1.0 + q2[:, None, :] * s2
    vals = t[..., 0] * t[..., 1] / 4.0
    dv = np.stack([s2[:, 0] * t[..., 1] / 4.0, s2[:, 1] * t[..., 0] / 4.0], axis=-1)
    local = HEX_FACES[facets[:, 1]]
    corners = mesh.nodes[mesh.cells[facets[:, 0][:, None], local]]
    pts = np.einsum("qa,fad->fqd", vals, corners)
    tan = np.einsum("qag,fad->fqdg", dv, corners)
    area = np.linalg.norm(np.cross(tan[..., 0], tan[..., 1]), axis=-1)
    return FaceQuadrature(points=pts, JxW=area, shape_values=vals, local_nodes=local)


def check_positive_jacobians(mesh: Mesh) -> None:
    """Raise InvertedElementError if any cell is inverted (elements.py:115-131, 152-154):
    det J by the cofactor expansion at the 8 Gauss points, first offender in (cell, qp)
    order, the reference's message."""
    qp = _tables()[0]
    t = 1.0 + qp[:, None, :] * VERTEX_SIGNS
    dN = np.stack([VERTEX_SIGNS[:, 0] * t[..., 1] * t[..., 2], VERTEX_SIGNS[:, 1] * t[..., 0] * t[..., 2],
                   VERTEX_SIGNS[:, 2] * t[..., 0] * t[..., 1]], axis=-1) / 8.0
    J = np.einsum("nka,qkb->nqab", mesh.cell_coords(), dN)
    c0 = J[..., 1, 1] * J[..., 2, 2] - J[..., 1, 2] * J[..., 2, 1]
    c1 = J[..., 1, 2] * J[..., 2, 0] - J[..., 1, 0] * J[..., 2, 2]
    c2 = J[..., 1, 0] * J[..., 2, 1] - J[..., 1, 1] * J[..., 2, 0]
    det = J[..., 0, 0] * c0 + J[..., 0, 1] * c1 + J[..., 0, 2] * c2
    if np.any(det <= 0.0):
        n, q = np.argwhere(det <= 0.0)[0]
        raise InvertedElementError(f"non-positive Jacobian determinant {det[n, q]:.3e} "
                                   f"(cell {n} of batch, quad point {q})")
