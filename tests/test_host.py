"""CPU tests of the host-side mirror (mesh, locators, Dirichlet tables, loads, support checks)
and of the C-ABI library surface (loads, exports every declared symbol) — no GPU needed."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from paper_2212_00964_b200 import _lib
from paper_2212_00964_b200.assembly import _body_load, _dirichlet_table, _neumann_load, check_supported
from cases import CASES, node_mask, traction_fn
from conftest import ROOT, load_golden
from pkg_cases import build, locator


@pytest.mark.parametrize("name", list(CASES))
def test_mesh_generation_bit_exact(name):
    g = load_golden(name)
    c = CASES[name]
    mesh = fem.generate_box_mesh(*c["dims"], *c["L"])
    assert np.array_equal(mesh.nodes, g["nodes"])
    assert np.array_equal(mesh.cells, g["cells"])


@pytest.mark.parametrize("name", list(CASES))
def test_dirichlet_tables_and_loads(name):
    g = load_golden(name)
    mesh, prob, _ = build(name)
    d, v = _dirichlet_table(mesh, prob.vec, prob.dirichlet)
    assert np.array_equal(d, g["dir_dofs"]) and np.array_equal(v, g["dir_values"])
    assert np.allclose(_neumann_load(mesh, prob.vec, prob.neumann), g["f_neumann"], rtol=1e-13, atol=1e-15)
    assert np.allclose(_body_load(mesh, prob.vec, prob.body_force), g["f_body"], rtol=1e-13, atol=1e-15)


def test_box_mesh_counts_and_validation():
    m = fem.generate_box_mesh(3, 2, 4, 1.5, 1.0, 2.0)
    assert m.n_nodes == 4 * 3 * 5 and m.n_cells == 24
    with pytest.raises(fem.MeshError):
        fem.generate_box_mesh(0, 1, 1, 1, 1, 1)
    with pytest.raises(fem.MeshError):
        fem.Mesh(np.zeros((9, 3)), np.arange(8)[None])  # orphan node 8


def test_boundary_facets_and_nodes():
    m = fem.generate_box_mesh(2, 3, 2, 2.0, 1.5, 1.0)
    top = fem.boundary_facets(m, fem.BoundaryLocator.plane(2, 1.0))
    assert len(top) == 6 and np.all(top.facets[:, 1] == 1)
    assert fem.boundary_nodes(m).size == m.n_nodes - 1 * 2 * 1  # interior: (nx-1)(ny-1)(nz-1)
    area = 0.0
    from paper_2212_00964_b200.elements import face_quadrature
    fq = face_quadrature(m, top.facets)
    area = fq.JxW.sum()
    assert abs(area - 3.0) < 1e-12


def test_neumann_total_load():
    """Reference tests/test_assembly.py:192-200 on the host load builder."""
    m = fem.generate_box_mesh(2, 3, 2, 2.0, 1.5, 1.0)
    t = np.array([0.3, -0.8, 2.0])
    spec = fem.NeumannSpec(fem.boundary_facets(m, fem.BoundaryLocator.plane(2, 1.0)), traction_fn(t))
    f = _neumann_load(m, 3, [spec])
    assert np.allclose(f.reshape(-1, 3).sum(axis=0), t * 3.0, rtol=1e-12)


def test_conflicting_constraints_rejected():
    m = fem.generate_box_mesh(1, 1, 1, 1, 1, 1)
    top = fem.BoundaryLocator.plane(2, 1.0)
    specs = [fem.DirichletSpec(top, 2, lambda p: 0.1), fem.DirichletSpec(top, 2, lambda p: 0.2)]
    with pytest.raises(fem.ConflictingConstraintError):
        _dirichlet_table(m, 3, specs)
    _dirichlet_table(m, 3, [specs[0], specs[0]])


def test_unsupported_user_maps_rejected_before_device_work():
    m = fem.generate_box_mesh(1, 1, 1, 1, 1, 1)
    alu = fem.ElasticConstants(E=70e3, nu=0.3)

    class MyProblem(fem.LinearElasticityProblem):
        def flux_kernel(self, grad_u, theta_e, state):
            return grad_u

    class MyLaw(fem.LinearElastic):
        def flux(self, grad_u, state=None):
            return grad_u

    with pytest.raises(fem.UnsupportedKernelError):
        check_supported(MyProblem(m, alu, []))
    p = fem.LinearElasticityProblem(m, alu, [])
    p.material = MyLaw(alu)
    with pytest.raises(fem.UnsupportedKernelError):
        check_supported(p)
    with pytest.raises(fem.UnsupportedKernelError):
        fem.assemble_residual(MyProblem(m, alu, []), np.zeros(24))
    check_supported(fem.SimpElasticityProblem(m, fem.NeoHookean(alu), []))
    with pytest.raises(fem.UnsupportedKernelError):
        check_supported(fem.SimpElasticityProblem(m, fem.J2Plasticity(fem.ElasticConstants(70e3, 0.3, 250.0)), []))


def test_no_cpu_fallback():
    """Without a GPU the product path must fail loudly, never compute on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    _, prob, U = build("poisson")
    with pytest.raises(fem.DeviceUnavailableError):
        fem.assemble_residual(prob, U)


def test_schedules_and_configs():
    assert fem.LoadSchedule.ramp(4).factors == (0.25, 0.5, 0.75, 1.0)
    assert fem.LoadSchedule.ramp_and_back(2).factors == (0.5, 1.0, 0.5, 0.0)
    with pytest.raises(ValueError):
        fem.LinearSolveConfig(rel_tol=0.0)
    with pytest.raises(ValueError):
        fem.NewtonConfig(abs_tol=-1.0)
    with pytest.raises(ValueError):
        fem.LoadSchedule(())


# ------------------------------------------------------------------- C ABI
HEADER = os.path.join(ROOT, "include", "b200fem.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(b200fem_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2212_00964_b200._build import LIB, build as build_lib
    if not os.path.exists(LIB):
        build_lib()
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    L = _lib.load_library(LIB)
    assert L.b200fem_version() == 1
