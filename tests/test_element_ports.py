"""Ports of the reference's tests/test_elements.py.

The reference caches per-cell geometry on the host (map_elements, elements.py:80-131).  Here
the shape-gradient map, det J and JxW are recomputed inside every device kernel
(csrc/element.cu `qp_geometry`), so the geometry properties are checked through what those
kernels return:

* the flux at the quadrature points (`quad_point_stress`) for Poisson with alpha = 1 is the
  physical gradient of u;
* the residual of u = x on a Poisson problem without Dirichlet rows gives the cell volume:
  sum_i X_i,x R_i = sum_q (sum_i X_i,x dphi_i/dx) JxW = sum_q JxW.

The reference-table and face-quadrature tests stay on the host, where those tables live.
"""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from paper_2212_00964_b200.elements import _tables, face_quadrature, shape_values_at_gauss
from paper_2212_00964_b200.mesh import HEX_FACES

gpu = pytest.mark.gpu


def unit_cell_mesh(coords=None):
    mesh = fem.generate_box_mesh(1, 1, 1, 1, 1, 1)
    if coords is None:
        return mesh
    nodes = mesh.nodes.copy()
    nodes[mesh.cells[0]] = coords
    return fem.Mesh(nodes, mesh.cells)


def poisson(mesh):
    return fem.PoissonProblem(mesh, 1.0, [])


def cell_flux(mesh, U):
    """(8 q, 3) physical gradient of u at the Gauss points of cell 0."""
    return np.asarray(fem.solvers.quad_point_stress(poisson(mesh), U))[0].reshape(8, 3)


def cell_volume(mesh):
    x = mesh.nodes[:, 0].copy()
    R = np.asarray(fem.assemble_residual(poisson(mesh), x))
    return float(x @ R)


# ------------------------------------------------------------------ host tables
def test_reference_element_tables():
    """Reference tests/test_elements.py:19-27."""
    qp, phi = _tables()
    assert np.abs(shape_values_at_gauss().sum(axis=1) - 1.0).max() <= 1e-14
    assert np.allclose(np.abs(qp), 1.0 / np.sqrt(3.0))
    assert np.array_equal(phi, shape_values_at_gauss())
    # Gauss points x fastest (elements.py:69): q = ix + 2 iy + 4 iz
    s = np.sign(qp)
    for q in range(8):
        assert list(s[q]) == [1 if q & 1 else -1, 1 if q & 2 else -1, 1 if q & 4 else -1]


def test_surface_quadrature_unit_cube_faces():
    """Reference tests/test_elements.py:92-99."""
    mesh = fem.generate_box_mesh(1, 1, 1, 1, 1, 1)
    for face in range(6):
        fq = face_quadrature(mesh, np.array([[0, face]]))
        assert np.isclose(fq.JxW.sum(), 1.0, rtol=1e-12)
        assert np.array_equal(fq.local_nodes[0], HEX_FACES[face])
        assert np.allclose(fq.shape_values.sum(axis=1), 1.0)


# ------------------------------------------------------------ device geometry
@gpu
def test_map_unit_cube():
    """Reference tests/test_elements.py:33-36: JxW = 1/8 per point, volume 1."""
    assert abs(cell_volume(unit_cell_mesh()) - 1.0) <= 1e-14
    vol = fem.volume_averaged_stress(poisson(unit_cell_mesh()), unit_cell_mesh().nodes[:, 0].copy())
    assert np.allclose(np.asarray(vol).ravel(), [1.0, 0.0, 0.0], atol=1e-15)


@gpu
def test_map_scaling_in_x():
    """Reference tests/test_elements.py:39-46: the x gradients halve, the volume doubles."""
    base = unit_cell_mesh()
    c0 = base.nodes[base.cells[0]]
    scaled = unit_cell_mesh(c0 * np.array([2.0, 1.0, 1.0]))
    rng = np.random.default_rng(3)
    U = rng.standard_normal(8)
    g0, g1 = cell_flux(base, U), cell_flux(scaled, U)
    assert np.allclose(g1[:, 0], g0[:, 0] / 2.0, rtol=1e-14, atol=1e-15)
    assert np.allclose(g1[:, 1:], g0[:, 1:], rtol=1e-14, atol=1e-15)
    assert np.isclose(cell_volume(scaled), 2.0 * cell_volume(base), rtol=1e-14)


@gpu
def test_map_translation_invariance():
    """Reference tests/test_elements.py:49-54."""
    base = unit_cell_mesh()
    moved = unit_cell_mesh(base.nodes[base.cells[0]] + np.array([3.0, -1.0, 2.5]))
    U = np.random.default_rng(4).standard_normal(8)
    assert np.allclose(cell_flux(base, U), cell_flux(moved, U), atol=1e-13)
    Rb = np.asarray(fem.assemble_residual(poisson(base), U))
    Rm = np.asarray(fem.assemble_residual(poisson(moved), U))
    assert np.allclose(Rb, Rm, atol=1e-14)


@gpu
def test_inverted_element_rejected():
    """Reference tests/test_elements.py:57-61: a mirrored cell (z -> -z) is rejected."""
    base = unit_cell_mesh()
    bad = base.nodes[base.cells[0]].copy()
    bad[:, 2] *= -1.0
    with pytest.raises(fem.InvertedElementError):
        fem.assemble_residual(poisson(unit_cell_mesh(bad)), np.zeros(8))


@gpu
def test_interpolate_gradient_zero_and_rigid():
    """Reference tests/test_elements.py:64-68, for the scalar and the vector kernels."""
    mesh = unit_cell_mesh()
    assert np.array_equal(cell_flux(mesh, np.zeros(8)), np.zeros((8, 3)))
    assert np.abs(cell_flux(mesh, np.full(8, 0.7))).max() < 1e-14
    le = fem.LinearElasticityProblem(mesh, fem.ElasticConstants(E=1.0, nu=0.25), [])
    rigid = np.tile([0.3, -0.2, 0.9], 8)
    assert np.abs(np.asarray(fem.solvers.quad_point_stress(le, rigid))).max() < 1e-14


@gpu
def test_affine_reproduction():
    """Reference tests/test_elements.py:71-79 (hypothesis, 20 examples; here 20 seeded draws,
    on the unit cell and on affine images of it): the gradient of an affine field is exact."""
    rng = np.random.default_rng(5)
    c0 = unit_cell_mesh().nodes[unit_cell_mesh().cells[0]]
    for k in range(20):
        M = np.eye(3) if k < 10 else rng.uniform(-1, 1, (3, 3)) + 2.0 * np.eye(3)
        coords = c0 @ M.T + rng.uniform(-1, 1, 3)
        a = rng.uniform(-2, 2, 3)
        mesh = unit_cell_mesh(coords)
        U = mesh.nodes @ a + 0.4  # by node id (the cell's vertex order is not the node order)
        g = cell_flux(mesh, U)
        assert np.abs(g - a).max() <= 1e-12 * max(1.0, np.abs(a).max())


@gpu
def test_quadrature_exact_volume_of_affine_images():
    """Reference tests/test_elements.py:82-89."""
    rng = np.random.default_rng(6)
    c0 = unit_cell_mesh().nodes[unit_cell_mesh().cells[0]]
    done = 0
    while done < 20:
        M = rng.uniform(-1, 1, (3, 3)) + 2.0 * np.eye(3)
        if np.linalg.det(M) <= 1e-3:
            continue
        coords = c0 @ M.T + np.array([0.5, -0.3, 1.0])
        assert np.isclose(cell_volume(unit_cell_mesh(coords)), np.linalg.det(M), rtol=1e-12)
        done += 1


@gpu
def test_batched_matches_single():
    """Reference tests/test_elements.py:102-107: a cell's quadrature-point values do not
    depend on the batch it is evaluated in (bit-identical)."""
    mesh = fem.generate_box_mesh(2, 2, 1, 2.0, 1.5, 0.7)
    U = np.random.default_rng(7).standard_normal(mesh.n_nodes)
    batched = np.asarray(fem.solvers.quad_point_stress(poisson(mesh), U))
    for e in range(mesh.n_cells):
        single = fem.Mesh(mesh.nodes[mesh.cells[e]], np.arange(8)[None, :])
        one = np.asarray(fem.solvers.quad_point_stress(poisson(single), U[mesh.cells[e]]))
        assert np.array_equal(one[0], batched[e])
