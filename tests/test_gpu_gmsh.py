"""Unstructured HEX8 meshes through the device path: Gmsh-imported O-grid
cylinders whose core-corner nodes are shared by 6 cells instead of 8.  Integer maps
bit-exact, R and K to 1e-12, Newton solutions to 1e-8 against the reference goldens
(tests/golden/make_golden_gmsh.py); the partitioned solve on node-range parts."""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from conftest import load_golden
from gmsh_cases import GMSH_CASES, build_gmsh, ogrid_cylinder, write_case_mesh
from paper_2212_00964_b200.distributed import newton_solve_partitioned

pytestmark = pytest.mark.gpu
NAMES = list(GMSH_CASES)
TIGHT = dict(cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-12), lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11,
                                                                                             abs_tol=1e-14))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", NAMES)
def test_gmsh_maps_residual_jacobian(name, tmp_path):
    g = load_golden(name)
    mesh, prob, U = build_gmsh(fem, name, write_case_mesh(name, tmp_path))
    ws = fem.workspace(prob)
    assert not ws.has_grid  # not a lattice: the CSR operator
    assert np.array_equal(ws.indptr, g["indptr"]) and np.array_equal(ws.indices, g["indices"])
    assert np.array_equal(ws.dest, g["dest"]) and np.array_equal(ws.diag_slots, g["diag_slots"])
    assert np.array_equal(ws.dir_dofs, g["dir_dofs"]) and np.array_equal(ws.dir_values, g["dir_values"])
    assert np.allclose(ws.f_neumann, g["f_neumann"], rtol=1e-13, atol=1e-15)
    assert rel(fem.assemble_residual(prob, g["U_test"]), g["R_test"]) < 1e-12
    assert rel(fem.assemble_jacobian(prob, g["U_test"]).data, g["K_test"]) < 1e-12


@pytest.mark.parametrize("method", ["bicgstab", "pcg"])
@pytest.mark.parametrize("name", NAMES)
def test_gmsh_newton_matches_reference(name, method, tmp_path):
    g = load_golden(name)
    _, prob, _ = build_gmsh(fem, name, write_case_mesh(name, tmp_path))
    kw = dict(TIGHT, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method))
    U, rep = fem.newton_solve(prob, **kw)
    assert rep.converged and rel(U, g["U_tight"]) < 1e-8


@pytest.mark.parametrize("nparts", [2, 3])
def test_gmsh_partitioned_matches_single(nparts, tmp_path):
    """Node-range parts of an unstructured mesh (no plane cuts, arbitrary halos)."""
    text, _ = ogrid_cylinder(6, 4, 10)
    path = tmp_path / "big.msh"
    path.write_text(text)
    GMSH_CASES["_big"] = dict(GMSH_CASES["gmsh_nh"], grid=(6, 4, 10))
    try:
        _, p1, _ = build_gmsh(fem, "_big", str(path))
        U1, r1 = fem.newton_solve(p1, **TIGHT)
        _, p2, _ = build_gmsh(fem, "_big", str(path))
        U2, r2 = newton_solve_partitioned(p2, nparts=nparts, mode="local", **TIGHT)
    finally:
        del GMSH_CASES["_big"]
    assert r2.n_iterations == r1.n_iterations and rel(U2, U1) < 1e-9
