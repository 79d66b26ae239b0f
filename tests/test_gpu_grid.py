"""GRID3 operator (csrc/spmv.cu k_spmv_grid3): the symmetric offset-major storage used by the
Newton loop on box lattices must be the same linear operator as the reference CSR Jacobian
(assembly.py:273-300 with identity Dirichlet rows), and solves through it must agree with
the CSR-operator solves and the reference goldens."""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from cases import CASES
from conftest import load_golden
from pkg_cases import build

pytestmark = pytest.mark.gpu

VEC3 = ["c1", "nh_block", "j2_block", "simp", "simp_nh", "le_body", "nh_crit6"]
VEC1 = ["poisson", "poisson_design"]
# shapes that exercise the staged (bulk-copy) chunks, chunk tails, NX = 2 (offset aliasing
# in linear ids) and long/flat lattices
SHAPES = [(12, 7, 9), (1, 4, 30), (5, 1, 40), (31, 2, 6), (40, 3, 3), (6, 6, 6)]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def D_(U):
    import torch
    return torch.tensor(U, device="cuda")


def grid_of(prob, U):
    from paper_2212_00964_b200.sparse import GridOperator
    ws = fem.workspace(prob)
    assert ws.has_grid
    G = GridOperator(ws)
    ws.jacobian_grid(prob, D_(U), G.device_data)
    return G


@pytest.mark.parametrize("name", VEC3 + VEC1)
def test_grid_operator_equals_csr_jacobian(name, rng):
    g = load_golden(name)
    _, prob, U = build(name)
    if "state_eps" in g:
        prob.state = fem.QuadPointState(g["state_eps"], g["state_sig"])
        U = g["U_test"]
    K = fem.assemble_jacobian(prob, U)
    assert rel(K.data, g["K_test"]) < 1e-12
    G = grid_of(prob, U)
    for _ in range(3):
        x = rng.standard_normal(prob.n_dofs)
        assert rel(G @ x, K @ x) < 1e-14


@pytest.mark.parametrize("dims", SHAPES)
def test_grid_operator_shapes(dims, rng):
    _, prob, U = build("nh_block", dict(CASES["nh_block"], dims=dims))
    U = U if U is not None else np.zeros(prob.n_dofs)
    U = U + 1e-3 * rng.standard_normal(prob.n_dofs)
    K = fem.assemble_jacobian(prob, U)
    G = grid_of(prob, U)
    x = rng.standard_normal(prob.n_dofs)
    y = G @ x
    assert rel(y, K @ x) < 1e-14
    dd = fem.workspace(prob).dir_dofs
    assert np.array_equal(y[dd], x[dd])  # identity Dirichlet rows, exactly


def test_grid_not_used_for_non_lattice_meshes():
    mesh = fem.generate_box_mesh(4, 3, 3, 1.0, 1.0, 1.0)
    perm = np.random.default_rng(3).permutation(mesh.n_nodes)
    inv = np.argsort(perm)
    m2 = fem.Mesh(nodes=mesh.nodes[perm], cells=inv[mesh.cells])
    spec = [fem.DirichletSpec(fem.BoundaryLocator.plane(2, 0.0), c, lambda p: 0.0) for c in range(3)]
    prob = fem.NeoHookeanProblem(m2, fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0), spec)
    assert not fem.workspace(prob).has_grid
    box = fem.NeoHookeanProblem(mesh, fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0), spec)
    assert fem.workspace(box).has_grid


@pytest.mark.parametrize("method", ["bicgstab", "pcg"])
@pytest.mark.parametrize("dims", [(6, 5, 4), (9, 8, 12)])
def test_newton_grid_operator_matches_csr_operator(method, dims):
    _, p1, _ = build("nh_block", dict(CASES["nh_block"], dims=dims))
    _, p2, _ = build("nh_block", dict(CASES["nh_block"], dims=dims))
    kw = dict(cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-11))
    U1, r1 = fem.newton_solve(p1, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method,
                                                               operator="csr"), **kw)
    U2, r2 = fem.newton_solve(p2, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method,
                                                               operator="grid"), **kw)
    assert r1.n_iterations == r2.n_iterations
    assert rel(U2, U1) < 1e-9
    for a, b in zip(r1.residual_norms, r2.residual_norms):
        assert abs(a - b) <= 1e-6 * max(abs(b), 1e-9) or b < 1e-8


def test_newton_grid_default_matches_reference_golden():
    g = load_golden("c1")
    _, prob, _ = build("c1")
    U, rep = fem.newton_solve(prob, cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-11),
                              lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14))
    from paper_2212_00964_b200.sparse import GridOperator
    assert isinstance(prob._jac_cache, GridOperator)  # LE: jacobian_constant, cached GRID3 tangent
    assert rep.converged and rel(U, g["U_tight"]) < 1e-8


def test_grid_solve_deterministic():
    outs = []
    for _ in range(2):
        _, p, _ = build("nh_block", dict(CASES["nh_block"], dims=(10, 9, 11)))
        U, _ = fem.newton_solve(p, lin_cfg=fem.LinearSolveConfig(operator="grid"))
        outs.append(U)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("dims", SHAPES)
def test_grid_scalar_operator_shapes(dims, rng):
    """vec 1 (Poisson) GRID: one value per lattice offset."""
    _, prob, U = build("poisson", dict(CASES["poisson"], dims=dims))
    K = fem.assemble_jacobian(prob, U)
    G = grid_of(prob, U)
    x = rng.standard_normal(prob.n_dofs)
    y = G @ x
    assert rel(y, K @ x) < 1e-14
    dd = fem.workspace(prob).dir_dofs
    assert np.array_equal(y[dd], x[dd])


@pytest.mark.parametrize("method", ["bicgstab", "pcg"])
def test_newton_grid_scalar_matches_csr(method):
    case = dict(CASES["poisson"], dims=(11, 9, 13))
    _, p1, _ = build("poisson", case)
    _, p2, _ = build("poisson", case)
    kw = dict(cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-11))
    U1, r1 = fem.newton_solve(p1, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method,
                                                               operator="csr"), **kw)
    U2, r2 = fem.newton_solve(p2, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method), **kw)
    from paper_2212_00964_b200.sparse import GridOperator
    assert isinstance(p2._jac_cache, GridOperator)
    assert r1.n_iterations == r2.n_iterations and rel(U2, U1) < 1e-9


# ------------------------------------------- opt-in inexact Newton: FP32-stored GRID3 values
def test_grid32_matvec_rounds_only_the_values(rng):
    """operator "grid32": the matvec of the FP32 copy equals the FP64 operator to the FP32
    rounding of the values (FP64 products and sums), and the identity rows stay exact."""
    _, prob, U = build("nh_block", dict(CASES["nh_block"], dims=(12, 7, 9)))
    U = (U if U is not None else np.zeros(prob.n_dofs)) + 1e-3 * rng.standard_normal(prob.n_dofs)
    G = grid_of(prob, U)
    x = rng.standard_normal(prob.n_dofs)
    y64 = G @ x
    vals = G.device_data.cpu().numpy()
    G.refresh_f32()
    assert np.array_equal(G.device_data32.cpu().numpy(), vals.astype(np.float32))
    y32 = G @ x
    assert 0.0 < rel(y32, y64) < 1e-6
    dd = fem.workspace(prob).dir_dofs
    assert np.array_equal(y32[dd], x[dd])


@pytest.mark.parametrize("method", ["bicgstab", "pcg"])
def test_newton_grid32_reaches_the_fp64_solution(method):
    """Inexact Newton with the FP32-stored tangent converges to the FP64 Newton solution
    (FP64 residual and stopping test): U within the north_star bar of 1e-8."""
    dims = (9, 8, 12)
    _, p1, _ = build("nh_block", dict(CASES["nh_block"], dims=dims))
    _, p2, _ = build("nh_block", dict(CASES["nh_block"], dims=dims))
    kw = dict(cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-11))
    U1, r1 = fem.newton_solve(p1, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method,
                                                               operator="grid"), **kw)
    U2, r2 = fem.newton_solve(p2, lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method=method,
                                                               operator="grid32"), **kw)
    assert r2.converged and r2.n_iterations <= r1.n_iterations + 1
    assert rel(U2, U1) < 1e-8


def test_grid32_rejects_scalar_and_non_lattice_problems():
    _, prob, _ = build("poisson")
    with pytest.raises(ValueError, match="grid32"):
        fem.newton_solve(prob, lin_cfg=fem.LinearSolveConfig(operator="grid32"))
