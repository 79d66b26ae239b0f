"""GPU parity of the adjoint row: K^T, adjoint solve, design VJP, total
derivative and the reduced objective, against the reference goldens (*_adjoint.npz), the
oracle, and the reference's own adjoint tests (reference tests/test_adjoint.py)."""

import numpy as np
import pytest

import oracle as orc
import paper_2212_00964_b200 as fem
from conftest import load_golden
from oracle_cases import build_oracle
from paper_2212_00964_b200 import _device as D
from paper_2212_00964_b200.adjoint import (ReducedObjective, adjoint_solve, optimize, taylor_test,
                                           total_derivative)
from paper_2212_00964_b200.inverse import (compliance, compliance_load_vector, poisson_objective,
                                           poisson_objective_gradient)
from pkg_cases import build

pytestmark = pytest.mark.gpu
DESIGN = ["poisson_design", "simp", "simp_nh"]
TIGHT_N = fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-12)
TIGHT_L = fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14)
REF_TIGHT_N = fem.NewtonConfig(rel_tol=1e-12, abs_tol=1e-12)  # reference tests/test_adjoint.py:23-24
REF_TIGHT_L = fem.LinearSolveConfig(rel_tol=1e-12, abs_tol=1e-14)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- goldens
@pytest.mark.parametrize("name", DESIGN)
def test_param_vjp_matches_reference(name):
    g = load_golden(f"{name}_adjoint")
    _, prob, U = build(name)
    v = fem.assemble_param_vjp(prob, U, g["theta_vjp"], g["w_test"])
    assert v.shape == g["vjp"].shape
    assert rel(v, g["vjp"]) < 1e-12


@pytest.mark.parametrize("name", DESIGN)
def test_transpose_is_the_reference_permutation(name):
    g = load_golden(f"{name}_adjoint")
    _, prob, U = build(name)
    K = fem.assemble_jacobian(prob, U)
    KT = K.transpose()
    assert np.array_equal(KT.indptr, g["KT_indptr"]) and np.array_equal(KT.indices, g["KT_indices"])
    _, _, perm = orc.csr_transpose(K.indptr, K.indices, K.data)
    assert np.array_equal(KT.data, perm)  # bit-exact permutation of our K
    assert rel(KT.data, g["KT_data"]) < 1e-12
    assert np.array_equal(KT.transpose().data, K.data)


def test_generic_csr_transpose_bit_exact():
    g = load_golden("generic_transpose")
    A = fem.CsrMatrix(g["indptr"], g["indices"], g["data"])
    T = A.transpose()
    assert np.array_equal(T.indptr, g["t_indptr"]) and np.array_equal(T.indices, g["t_indices"])
    assert np.array_equal(T.data, g["t_data"])
    x = np.random.default_rng(3).standard_normal(A.shape[0])
    assert np.allclose(T.matvec(x), A.todense().T @ x, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("name", DESIGN)
def test_adjoint_solution_and_gradient_match_reference(name):
    g = load_golden(f"{name}_adjoint")
    _, prob, _ = build(name)
    lam = adjoint_solve(prob, g["U_tight"], g["dj_du"], lin_cfg=TIGHT_L)
    assert rel(lam, g["lam_tight"]) < 1e-8
    grad = total_derivative(prob, g["U_tight"], lam, prob.theta)
    assert rel(grad, g["grad_tight"]) < 1e-8


@pytest.mark.parametrize("name", DESIGN)
def test_reduced_objective_matches_reference(name):
    g = load_golden(f"{name}_adjoint")
    _, prob, _ = build(name)
    if "obs" in g:
        obs, vals = g["obs"], g["obs_values"]
        ro = ReducedObjective(prob, lambda U, t: poisson_objective(U, obs, vals),
                              lambda U, t: poisson_objective_gradient(U, obs, vals), newton_cfg=TIGHT_N, lin_cfg=TIGHT_L)
    else:
        ro = ReducedObjective(prob, lambda U, t: compliance(prob, U), lambda U, t: compliance_load_vector(prob),
                              newton_cfg=TIGHT_N, lin_cfg=TIGHT_L)
    v, grad = ro.value_and_gradient(g["theta"])
    assert abs(v - float(g["ro_value"])) <= 1e-8 * abs(float(g["ro_value"]))
    assert rel(grad, g["ro_grad"]) < 1e-8


# ------------------------------------------------------------ oracle, larger
@pytest.mark.parametrize("dims", [(12, 6, 4), (9, 7, 5)])
def test_vjp_and_transpose_vs_oracle_larger(dims):
    from cases import CASES

    case = dict(CASES["simp"], dims=dims, L=(float(dims[0]) / 2, float(dims[1]) / 2, float(dims[2]) / 2),
                neumann=[(("plane", 0, float(dims[0]) / 2), (0.0, 0.0, -1.0))])
    _, prob, U = build("simp", case)
    oprob, _ = build_oracle("simp", case)
    rng = np.random.default_rng(5)
    w = rng.standard_normal(prob.n_dofs)
    th = rng.uniform(0.2, 1.0, prob.mesh.n_cells)
    assert rel(fem.assemble_param_vjp(prob, U, th, w), orc.param_vjp(oprob, U, th, w)) < 1e-12
    K = fem.assemble_jacobian(prob, U)
    x, y = rng.standard_normal(prob.n_dofs), rng.standard_normal(prob.n_dofs)
    lhs = float(np.dot(K.matvec(x), y))
    rhs = float(np.dot(x, K.transpose().matvec(y)))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


# ------------------------------------------- reference tests/test_adjoint.py
def poisson_setup(dims=(3, 3, 2), box=(1.0, 1.0, 0.4)):
    mesh = fem.generate_box_mesh(*dims, *box)
    onb = fem.BoundaryLocator(lambda p: (np.abs(np.asarray(p)) < 1e-9).any(axis=-1)
                              | (np.abs(np.asarray(p) - np.asarray(box)) < 1e-9).any(axis=-1))
    prob = fem.PoissonProblem(mesh, 1.0, [fem.DirichletSpec(onb, 0, lambda p: 0.0)], design_source=True)
    return mesh, prob


def simp_cantilever(dims=(4, 4, 1), box=(4.0, 4.0, 1.0)):
    mesh = fem.generate_box_mesh(*dims, *box)
    left = fem.BoundaryLocator.plane(0, 0.0)
    right = fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, box[0]))
    t = np.array([0.0, 0.0, -1.0])
    neu = [fem.NeumannSpec(right, lambda p: np.broadcast_to(t, np.asarray(p).shape[:-1] + (3,)))]
    specs = [fem.DirichletSpec(left, c, lambda p: 0.0) for c in range(3)]
    prob = fem.SimpElasticityProblem(mesh, fem.LinearElastic(fem.ElasticConstants(E=70e3, nu=0.3)), specs, neu)
    return mesh, prob


def test_adjoint_zero_objective_gradient():
    mesh, prob = poisson_setup()
    prob.set_theta(np.ones(mesh.n_nodes))
    U, _ = fem.newton_solve(prob, cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)
    lam = adjoint_solve(prob, U, np.zeros(prob.n_dofs), lin_cfg=REF_TIGHT_L)
    assert np.array_equal(lam, np.zeros(prob.n_dofs))


def test_adjoint_selfadjoint_equals_unit_load_forward(rng):
    mesh, prob = poisson_setup()
    prob.set_theta(rng.standard_normal(mesh.n_nodes))
    U, _ = fem.newton_solve(prob, cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)
    ws = fem.workspace(prob)
    free = np.setdiff1d(np.arange(prob.n_dofs), ws.dir_dofs)
    ind = np.zeros(prob.n_dofs)
    ind[rng.choice(free, 4, replace=False)] = 1.0
    lam = adjoint_solve(prob, U, ind, lin_cfg=REF_TIGHT_L)
    u_unit = fem.bicgstab_jacobi(fem.assemble_jacobian(prob, U), ind, cfg=REF_TIGHT_L)
    assert np.abs(lam[free] - u_unit[free]).max() < 1e-9 * max(1.0, np.abs(u_unit).max())


def test_adjoint_compliance_selfadjoint_on_free_dofs(rng):
    mesh, prob = simp_cantilever()
    prob.set_theta(rng.uniform(0.4, 1.0, mesh.n_cells))
    U, _ = fem.newton_solve(prob, cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)
    lam = adjoint_solve(prob, U, compliance_load_vector(prob), lin_cfg=REF_TIGHT_L)
    free = np.setdiff1d(np.arange(prob.n_dofs), fem.workspace(prob).dir_dofs)
    assert np.abs(lam[free] - U[free]).max() < 1e-8 * np.abs(U).max()


def test_total_derivative_zero_cases(rng):
    mesh, prob = poisson_setup()
    theta = rng.standard_normal(mesh.n_nodes)
    prob.set_theta(theta)
    U, _ = fem.newton_solve(prob, cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)
    assert np.array_equal(total_derivative(prob, U, np.zeros(prob.n_dofs), theta), np.zeros(mesh.n_nodes))


def _poisson_obj(prob, obs, vals, scale=1.0):
    return ReducedObjective(prob, lambda U, t: scale * poisson_objective(U, obs, vals),
                            lambda U, t: scale * poisson_objective_gradient(U, obs, vals),
                            newton_cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)


def test_gradient_scales_linearly_with_objective(rng):
    mesh, prob = poisson_setup()
    obs = np.sort(rng.choice(mesh.n_nodes, 10, replace=False))
    vals = rng.standard_normal(10) * 0.01
    theta = rng.standard_normal(mesh.n_nodes)
    _, g1 = _poisson_obj(prob, obs, vals).value_and_gradient(theta)
    _, g3 = _poisson_obj(prob, obs, vals, 3.0).value_and_gradient(theta)
    assert np.allclose(g3, 3.0 * g1, rtol=1e-9)


@pytest.mark.parametrize("setup", ["poisson", "simp"])
def test_adjoint_gradient_matches_fd(setup, rng):
    if setup == "poisson":
        mesh, prob = poisson_setup((4, 4, 2), (1.0, 1.0, 0.5))
        obs = np.sort(rng.choice(mesh.n_nodes, 15, replace=False))
        obj = _poisson_obj(prob, obs, rng.standard_normal(15) * 0.01)
        theta = rng.standard_normal(prob.n_design)
    else:
        mesh, prob = simp_cantilever()
        obj = ReducedObjective(prob, lambda U, t: compliance(prob, U), lambda U, t: compliance_load_vector(prob),
                               newton_cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)
        theta = rng.uniform(0.3, 0.9, prob.n_design)
    _, g = obj.value_and_gradient(theta)
    h = 1e-6
    for _ in range(10):
        d = rng.standard_normal(theta.shape[0])
        fd = (obj.value(theta + h * d) - obj.value(theta - h * d)) / (2 * h)
        assert abs(fd - g @ d) / max(abs(fd), 1e-14) < 1e-5


def test_gradient_consistent_across_fresh_resolves(rng):
    mesh, _ = poisson_setup()
    obs = np.sort(rng.choice(mesh.n_nodes, 10, replace=False))
    vals = rng.standard_normal(10) * 0.01
    theta = rng.standard_normal(mesh.n_nodes)
    g1 = _poisson_obj(poisson_setup()[1], obs, vals).value_and_gradient(theta)[1]
    g2 = _poisson_obj(poisson_setup()[1], obs, vals).value_and_gradient(theta)[1]
    assert np.abs(g1 - g2).max() <= 1e-10 * max(1.0, np.abs(g1).max())


def test_taylor_poisson_orders_and_negative_control(rng):
    mesh, prob = poisson_setup()
    free = np.setdiff1d(np.arange(prob.n_dofs), fem.workspace(prob).dir_dofs)
    obs = np.sort(rng.choice(free, min(6, free.size), replace=False))
    obj = _poisson_obj(prob, obs, rng.standard_normal(obs.size) * 0.01)
    theta = rng.standard_normal(mesh.n_nodes)
    dtheta = np.zeros(mesh.n_nodes)
    dtheta[rng.choice(mesh.n_nodes, 5, replace=False)] = rng.standard_normal(5)
    rep = taylor_test(obj.value, obj.gradient, theta, dtheta, [1e-1, 1e-2, 1e-3, 1e-4])
    assert 0.9 <= rep.fitted_zeroth <= 1.1
    assert 1.9 <= rep.fitted_first <= 2.1
    bad = taylor_test(obj.value, lambda t: 1.1 * obj.gradient(t), theta, dtheta, [1e-1, 1e-2, 1e-3, 1e-4])
    assert bad.fitted_first < 1.5


def test_device_tensors_stay_on_device(rng):
    mesh, prob = simp_cantilever()
    prob.set_theta(rng.uniform(0.4, 1.0, mesh.n_cells))
    U, _ = fem.newton_solve(prob, D.zeros(prob.n_dofs), cfg=REF_TIGHT_N, lin_cfg=REF_TIGHT_L)
    lam = adjoint_solve(prob, U, D.to_device(compliance_load_vector(prob)), lin_cfg=REF_TIGHT_L)
    assert D.is_device_tensor(lam)
    g = total_derivative(prob, U, lam, D.to_device(prob.theta))
    assert D.is_device_tensor(g)
    gh = total_derivative(prob, D.to_host(U), D.to_host(lam), prob.theta)
    assert np.array_equal(D.to_host(g), gh)


def test_vjp_without_design_raises():
    _, prob, U = build("c1")
    with pytest.raises(ValueError):
        fem.assemble_param_vjp(prob, U, np.zeros(3), np.zeros(prob.n_dofs))


def test_optimize_lbfgs_on_poisson_inference(rng):
    mesh, prob = poisson_setup()
    free = np.setdiff1d(np.arange(prob.n_dofs), fem.workspace(prob).dir_dofs)
    obs = np.sort(rng.choice(free, min(6, free.size), replace=False))
    obj = _poisson_obj(prob, obs, rng.standard_normal(obs.size) * 0.01)
    theta, hist = optimize(obj.value_and_gradient, np.zeros(mesh.n_nodes), max_iters=30, gtol=1e-12)
    assert hist.objective[-1] < 1e-3 * hist.objective[0]


@pytest.mark.parametrize("name", DESIGN)
def test_adjoint_pcg_split_matches_reference(name):
    g = load_golden(f"{name}_adjoint")
    _, prob, _ = build(name)
    cfg = fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, method="pcg")
    lam = adjoint_solve(prob, g["U_tight"], g["dj_du"], lin_cfg=cfg)
    assert rel(lam, g["lam_tight"]) < 1e-8
