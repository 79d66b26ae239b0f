"""Gmsh MSH v2.2 import (reference mesh.py:216-285) on the host: the
reference's own import tests (tests/test_mesh.py:115-171), bit-exact nodes/cells against
the reference importer on the unstructured O-grid meshes, and the oracle pinned to the
reference's R, K and integer maps on those meshes."""

import numpy as np
import pytest

import oracle as orc
import paper_2212_00964_b200 as fem
from conftest import load_golden
from gmsh_cases import GMSH_CASES, write_case_mesh
from paper_2212_00964_b200.elements import InvertedElementError, cell_jxw

GMSH_UNIT_CUBE = """$MeshFormat
2.2 0 8
$EndMeshFormat
$Nodes
9
1 0 0 0
2 1 0 0
3 1 1 0
4 0 1 0
5 0 0 1
6 1 0 1
7 1 1 1
8 0 1 1
9 4 4 4
$EndNodes
$Elements
3
1 15 2 0 1 9
2 3 2 0 1 1 2 3 4
3 5 2 0 1 1 2 3 4 5 6 7 8
$EndElements
"""


def test_import_gmsh_v22(tmp_path):
    path = tmp_path / "cube.msh"
    path.write_text(GMSH_UNIT_CUBE)
    m = fem.import_mesh(path)
    assert m.n_cells == 1 and m.n_nodes == 8  # point entity, surface quad, orphan node dropped
    assert np.isclose(cell_jxw(m).sum(), 1.0, rtol=1e-12)


def test_import_rejects_unsupported_volume_cells(tmp_path):
    path = tmp_path / "tet.msh"
    path.write_text(GMSH_UNIT_CUBE.replace("3 5 2 0 1 1 2 3 4 5 6 7 8", "3 4 2 0 1 1 2 3 5"))
    with pytest.raises(fem.MeshError, match="type 4"):
        fem.import_mesh(path)


def test_import_rejects_inverted_cells(tmp_path):
    path = tmp_path / "inv.msh"
    path.write_text(GMSH_UNIT_CUBE.replace("3 5 2 0 1 1 2 3 4 5 6 7 8", "3 5 2 0 1 5 6 7 8 1 2 3 4"))
    with pytest.raises(InvertedElementError, match="Jacobian"):
        fem.import_mesh(path)


def test_import_rejects_wrong_version(tmp_path):
    path = tmp_path / "v4.msh"
    path.write_text(GMSH_UNIT_CUBE.replace("2.2 0 8", "4.1 0 8"))
    with pytest.raises(fem.MeshError, match="version"):
        fem.import_mesh(path)


def test_import_rejects_missing_section_and_bad_counts(tmp_path):
    path = tmp_path / "x.msh"
    path.write_text(GMSH_UNIT_CUBE.replace("$Elements", "$Elementz"))
    with pytest.raises(fem.MeshError, match="missing"):
        fem.import_mesh(path)
    path.write_text(GMSH_UNIT_CUBE.replace("$Nodes\n9", "$Nodes\n10"))
    with pytest.raises(fem.MeshError, match="count mismatch"):
        fem.import_mesh(path)
    path.write_text(GMSH_UNIT_CUBE.replace("3 5 2 0 1 1 2 3 4 5 6 7 8", "3 5 2 0 1 1 2 3 4 5 6 7"))
    with pytest.raises(fem.MeshError, match="malformed"):
        fem.import_mesh(path)


@pytest.mark.parametrize("name", list(GMSH_CASES))
def test_import_matches_reference_importer(name, tmp_path):
    g = load_golden(name)
    m = fem.import_mesh(write_case_mesh(name, tmp_path))
    assert np.array_equal(m.nodes, g["nodes"]) and np.array_equal(m.cells, g["cells"])
    assert np.bincount(m.cells.ravel()).min() < 8 < np.bincount(m.cells.ravel()).max() + 1  # irregular valence


@pytest.mark.parametrize("name", list(GMSH_CASES))
def test_oracle_on_unstructured_mesh(name):
    """The CPU oracle against the reference's maps, R and K on the imported mesh."""
    g = load_golden(name)
    law = orc.Law("poisson", alpha=1.0) if name.endswith("poisson") else orc.Law(
        name.split("_")[1], E=70e3, nu=0.3, sigma_yield=250.0)
    src = None
    if name.endswith("poisson"):
        src = lambda p: np.full(np.asarray(p).shape[:-1] + (1,), 1.0)  # noqa: E731
    fb = orc.body_load(g["nodes"], g["cells"], law.vec, src)
    p = orc.OracleProblem(g["nodes"], g["cells"], law, g["dir_dofs"], g["dir_values"], g["f_neumann"], fb)
    assert np.array_equal(p.indptr, g["indptr"]) and np.array_equal(p.indices, g["indices"])
    assert np.array_equal(p.dest.reshape(g["dest"].shape), g["dest"])
    R = orc.residual(p, g["U_test"])
    assert np.linalg.norm(R - g["R_test"]) <= 1e-12 * np.linalg.norm(g["R_test"])
    K = orc.jacobian(p, g["U_test"])
    assert np.linalg.norm(K - g["K_test"]) <= 1e-12 * np.linalg.norm(g["K_test"])
