"""Ports of the reference's tests/test_mesh.py (the Gmsh import tests are in test_mesh_io.py).

Mesh generation, locators and facets stay host Python, as in the reference (mesh.py); the
volume check runs through the device geometry (see test_element_ports.py for the identity
sum_i X_i,x R_i = sum_q JxW used here).
"""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from paper_2212_00964_b200.mesh import locate_nodes


def test_single_unit_cell():
    """Reference tests/test_mesh.py:19-24."""
    m = fem.generate_box_mesh(1, 1, 1, 1, 1, 1)
    assert m.n_nodes == 8 and m.n_cells == 1
    assert {tuple(p) for p in m.nodes} == {(float(i), float(j), float(k)) for i in (0, 1) for j in (0, 1)
                                           for k in (0, 1)}


def test_inference_demo_mesh_counts():
    """Reference tests/test_mesh.py:27-30."""
    m = fem.generate_box_mesh(50, 50, 10, 1.0, 1.0, 0.2)
    assert m.n_nodes == 51 * 51 * 11 == 28611
    assert m.n_cells == 25000


@pytest.mark.parametrize("args", [(0, 1, 1, 1, 1, 1), (1, -2, 1, 1, 1, 1), (1, 1, 1, 0.0, 1, 1),
                                  (1, 1, 1, 1, 1, -3.0)])
def test_generator_rejects_bad_arguments(args):
    """Reference tests/test_mesh.py:39-50."""
    with pytest.raises(fem.MeshError):
        fem.generate_box_mesh(*args)


def test_locate_nodes_bottom_face():
    """Reference tests/test_mesh.py:71-75."""
    assert len(locate_nodes(fem.generate_box_mesh(1, 1, 1, 1, 1, 1), fem.BoundaryLocator.plane(2, 0.0))) == 4
    assert len(locate_nodes(fem.generate_box_mesh(2, 2, 2, 1, 1, 1), fem.BoundaryLocator.plane(2, 0.0))) == 9


def test_locate_nodes_empty_and_partition():
    """Reference tests/test_mesh.py:78-86."""
    m = fem.generate_box_mesh(2, 2, 2, 1, 1, 1)
    never = fem.BoundaryLocator(lambda p: np.zeros(np.asarray(p).shape[:-1], dtype=bool))
    assert locate_nodes(m, never).size == 0
    sel = locate_nodes(m, fem.BoundaryLocator.plane(0, 0.5))
    other = locate_nodes(m, fem.BoundaryLocator(lambda p: ~(np.abs(np.asarray(p)[..., 0] - 0.5) <= 1e-5)))
    assert np.array_equal(np.sort(np.concatenate([sel, other])), np.arange(m.n_nodes))
    assert np.intersect1d(sel, other).size == 0


def test_boundary_facets_interior_plane():
    """Reference tests/test_mesh.py:89-97."""
    assert len(fem.boundary_facets(fem.generate_box_mesh(1, 1, 1, 1, 1, 1), fem.BoundaryLocator.plane(2, 1.0))) == 1
    assert len(fem.boundary_facets(fem.generate_box_mesh(2, 2, 1, 1, 1, 1), fem.BoundaryLocator.plane(2, 0.0))) == 4
    assert len(fem.boundary_facets(fem.generate_box_mesh(1, 1, 2, 1, 1, 1), fem.BoundaryLocator.plane(2, 0.5))) == 0


def test_boundary_nodes_counts():
    """Reference tests/test_mesh.py:100-102."""
    assert fem.boundary_nodes(fem.generate_box_mesh(3, 3, 3, 1, 1, 1)).size == 4 ** 3 - 2 ** 3


def test_mesh_validation():
    """Reference tests/test_mesh.py:105-112."""
    with pytest.raises(fem.MeshError):
        fem.Mesh(nodes=np.zeros((4, 3)), cells=np.array([[0, 1, 2, 3, 4, 5, 6, 7]]))
    m = fem.generate_box_mesh(1, 1, 1, 1, 1, 1)
    with pytest.raises(fem.MeshError, match="not referenced"):
        fem.Mesh(nodes=np.vstack([m.nodes, [[5.0, 5.0, 5.0]]]), cells=m.cells)


@pytest.mark.gpu
def test_unit_cells_jacobian_and_structured_volume():
    """Reference tests/test_mesh.py:33-36 and 53-68 (hypothesis, 25 examples; here 25 seeded
    draws): det J of axis-aligned unit cells is 1/8 per point and the quadrature volume of a
    box is lx*ly*lz -- through the device geometry."""
    m = fem.generate_box_mesh(2, 1, 1, 2.0, 1.0, 1.0)
    g = np.asarray(fem.solvers.quad_point_stress(fem.PoissonProblem(m, 1.0, []), m.nodes[:, 0].copy()))
    assert np.abs(g.reshape(-1, 3) - [1.0, 0.0, 0.0]).max() <= 1e-15
    rng = np.random.default_rng(8)
    for _ in range(25):
        nx, ny, nz = (int(v) for v in rng.integers(1, 5, 3))
        lx, ly, lz = (float(v) for v in rng.uniform(0.1, 10, 3))
        m = fem.generate_box_mesh(nx, ny, nz, lx, ly, lz)
        assert m.n_nodes == (nx + 1) * (ny + 1) * (nz + 1) and m.n_cells == nx * ny * nz
        x = m.nodes[:, 0].copy()
        vol = float(x @ np.asarray(fem.assemble_residual(fem.PoissonProblem(m, 1.0, []), x)))
        assert np.isclose(vol, lx * ly * lz, rtol=1e-12)
