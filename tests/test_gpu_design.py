"""GPU parity of the design-loop row: density filter, filtered sensitivities,
MMA, L2 field error, run_topopt / run_inference -- against the reference goldens
(tests/golden/design.npz), the oracle, and the reference's tests/test_inverse.py."""

import numpy as np
import pytest

import oracle as orc
import paper_2212_00964_b200 as fem
from conftest import load_golden
from paper_2212_00964_b200 import _device as D
from paper_2212_00964_b200.inverse import (MmaState, compliance, density_filter, element_centroids,
                                           filter_sensitivities, l2_field_error, mma_update, poisson_objective,
                                           poisson_objective_gradient, run_inference, run_topopt)

pytestmark = pytest.mark.gpu
FILTERS = [((4, 3, 2), (4.0, 3.0, 2.0), 1.6), ((3, 3, 2), (3.0, 3.0, 2.0), 1.7), ((6, 4, 3), (3.0, 2.0, 1.5), 0.8),
           ((5, 5, 1), (1.0, 1.0, 0.2), 0.45)]
TIGHT_N = fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-12)
TIGHT_L = fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14)
ALU = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)


@pytest.fixture(scope="module")
def g():
    return load_golden("design")


# ---------------------------------------------------------------- goldens
@pytest.mark.parametrize("k", range(len(FILTERS)))
def test_density_filter_matches_reference_bit_exact(g, k):
    dims, box, r = FILTERS[k]
    mesh = fem.generate_box_mesh(*dims, *box)
    f = density_filter(mesh, r)
    M = f.matrix
    assert np.array_equal(M.indptr, g[f"f{k}_indptr"]) and np.array_equal(M.indices, g[f"f{k}_indices"])
    assert np.array_equal(M.data, g[f"f{k}_data"])
    assert np.array_equal(f(g[f"f{k}_x"]), g[f"f{k}_Hx"])
    th = g[f"f{k}_theta"]
    assert np.array_equal(filter_sensitivities(f, th, g[f"f{k}_sens"]), g[f"f{k}_fs"])


def test_mma_sequence_matches_reference(g):
    n = g["mma_x0"].size
    st = MmaState.fresh(n, move_limit=0.2)
    x = g["mma_x0"]
    for k in range(5):
        xn = mma_update(st, x, g[f"mma{k}_dj"], float(g[f"mma{k}_g"]), np.full(n, 1.0 / n), 1e-3, 1.0)
        assert np.array_equal(D.to_host(st.lower), g[f"mma{k}_low"])
        assert np.array_equal(D.to_host(st.upper), g[f"mma{k}_upp"])
        assert np.abs(xn - g[f"mma{k}_x"]).max() <= 1e-12
        x = g[f"mma{k}_x"]


def test_l2_field_error_matches_reference(g):
    mesh = fem.generate_box_mesh(3, 3, 2, 1.0, 1.0, 0.4)
    e = l2_field_error(mesh, g["l2_up"], g["l2_ut"])
    assert abs(e - float(g["l2"])) <= 1e-12 * float(g["l2"])


def simp_cantilever(dims=(8, 4, 1), box=(8.0, 4.0, 1.0), material=None, neumann=True):
    mesh = fem.generate_box_mesh(*dims, *box)
    mat = material or fem.LinearElastic(fem.ElasticConstants(E=70e3, nu=0.3))
    right = fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, box[0]))
    t = np.array([0.0, 0.0, -1.0])
    left = fem.BoundaryLocator.plane(0, 0.0)
    neu = [fem.NeumannSpec(right, lambda p: np.broadcast_to(t, np.asarray(p).shape[:-1] + (3,)))] if neumann else []
    prob = fem.SimpElasticityProblem(mesh, mat, [fem.DirichletSpec(left, c, lambda p: 0.0) for c in range(3)], neu)
    return mesh, prob


def test_run_topopt_matches_reference(g):
    _, prob = simp_cantilever()
    res = run_topopt(prob, volume_fraction=0.5, n_steps=5, newton_cfg=TIGHT_N, lin_cfg=TIGHT_L)
    c_ref = g["topo_comp"]
    assert np.max(np.abs(np.array(res.compliance_history) - c_ref) / c_ref) < 1e-8
    assert np.allclose(res.volume_history, g["topo_vol"], rtol=0, atol=1e-10)
    assert np.abs(res.theta - g["topo_theta"]).max() < 1e-7
    assert abs(res.final_compliance - float(g["topo_final"])) <= 1e-8 * float(g["topo_final"])


def bimodal(x):
    x = np.asarray(x)
    return 10 * np.exp(-10 * np.sum((x - [0.25, 0.25, 0.1]) ** 2, axis=-1)) + 10 * np.exp(
        -10 * np.sum((x - [0.75, 0.75, 0.1]) ** 2, axis=-1))


def inference_problem(dims, box):
    mesh = fem.generate_box_mesh(*dims, *box)
    b = np.asarray(box, dtype=np.float64)
    onb = fem.BoundaryLocator(lambda p: (np.abs(np.asarray(p)) < 1e-9).any(axis=-1)
                              | (np.abs(np.asarray(p) - b) < 1e-9).any(axis=-1))
    return mesh, fem.PoissonProblem(mesh, 1.0, [fem.DirichletSpec(onb, 0, lambda p: 0.0)], design_source=True)


def test_run_inference_matches_reference(g):
    _, prob = inference_problem((6, 6, 2), (1.0, 1.0, 0.2))
    res = run_inference(prob, bimodal, n_obs=12, seed=0, max_iters=15, lin_cfg=TIGHT_L)
    assert np.array_equal(res.obs_indices, g["inf_obs"])
    assert np.abs(res.u_true - g["inf_u_true"]).max() <= 1e-9 * np.abs(g["inf_u_true"]).max()
    ref = g["inf_obj"]
    m = min(len(ref), len(res.objective_history), 6)  # early L-BFGS iterates (later ones amplify round-off)
    assert np.allclose(res.objective_history[:m], ref[:m], rtol=1e-6, atol=1e-14)


# ------------------------------------------------------------ oracle, larger
def test_filter_and_mma_vs_oracle_larger():
    mesh = fem.generate_box_mesh(24, 12, 8, 6.0, 3.0, 2.0)
    f = density_filter(mesh, 0.55)
    H = orc.density_filter(mesh.nodes, mesh.cells, 0.55)
    M = f.matrix
    assert np.array_equal(M.indptr, H[0]) and np.array_equal(M.indices, H[1]) and np.array_equal(M.data, H[2])
    rng = np.random.default_rng(9)
    n = 20000
    x = rng.uniform(0.1, 0.9, n)
    dj = rng.standard_normal(n)
    st = MmaState.fresh(n)
    ost = dict(lower=None, upper=None, x_prev=None, x_prev2=None, iteration=0, move_limit=0.2, asym_init=0.5,
               asym_expand=1.2, asym_shrink=0.7)
    for k in range(3):
        gv = float(x.mean() - 0.45)
        xd = mma_update(st, x, dj, gv, np.full(n, 1.0 / n), 1e-3, 1.0)
        xo = orc.mma_update(ost, x, dj, gv, np.full(n, 1.0 / n), 1e-3, 1.0)
        assert np.abs(xd - xo).max() <= 1e-12
        x, dj = xo, rng.standard_normal(n)


# ------------------------------------------- reference tests/test_inverse.py
def test_poisson_objective_values():
    U = np.array([1.0, 2.0, 3.0, 4.0])
    assert poisson_objective(U, [1, 3], [2.0, 4.0]) == 0.0
    assert poisson_objective(U, [0], [3.0]) == 4.0
    gr = poisson_objective_gradient(U, [0, 2], [0.0, 0.0])
    assert np.count_nonzero(gr) == 2 and gr[0] == 2.0 and gr[2] == 6.0


def test_l2_error_zero_for_identical_fields(rng):
    mesh = fem.generate_box_mesh(2, 2, 2, 1, 1, 1)
    u = rng.standard_normal(mesh.n_nodes)
    assert l2_field_error(mesh, u, u) == 0.0


def test_fully_observed_inference_is_consistent():
    _, prob = inference_problem((6, 6, 2), (1.0, 1.0, 0.2))
    res = run_inference(prob, bimodal, n_obs=1, seed=0, max_iters=400, observe_all=True)
    assert np.abs(res.u_pred[res.obs_indices] - res.u_true[res.obs_indices]).max() < 1e-6
    assert res.objective_history[-1] < 1e-10


def test_inference_error_improves_with_observations():
    _, prob = inference_problem((10, 10, 2), (1.0, 1.0, 0.2))
    few = run_inference(prob, bimodal, n_obs=20, seed=3, max_iters=60)
    _, prob2 = inference_problem((10, 10, 2), (1.0, 1.0, 0.2))
    many = run_inference(prob2, bimodal, n_obs=80, seed=3, max_iters=60)
    assert many.relative_l2_error < few.relative_l2_error


def test_inference_rejects_bad_obs_count():
    _, prob = inference_problem((3, 3, 2), (1, 1, 0.4))
    with pytest.raises(ValueError):
        run_inference(prob, bimodal, n_obs=0, seed=0)
    with pytest.raises(ValueError):
        run_inference(prob, bimodal, n_obs=10 ** 6, seed=0)


def test_simp_floor_keeps_system_solvable():
    mesh, prob = simp_cantilever((2, 2, 2), (1.0, 1.0, 1.0), fem.LinearElastic(ALU))
    prob.set_theta(np.full(mesh.n_cells, 1e-3))
    U, rep = fem.newton_solve(prob)
    assert rep.converged and np.all(np.isfinite(U))


def test_compliance_values():
    mesh, prob = simp_cantilever((2, 2, 1), (2.0, 2.0, 1.0))
    assert compliance(prob, np.zeros(prob.n_dofs)) == 0.0
    d = np.array([0.1, -0.2, 0.3])
    U = np.tile(d, mesh.n_nodes)
    assert np.isclose(compliance(prob, U), float(d @ np.array([0.0, 0.0, -1.0])) * 2.0, rtol=1e-12)


def test_compliance_uniform_density_scaling():
    mesh, prob = simp_cantilever((4, 2, 1), (4.0, 2.0, 1.0))
    prob.set_theta(np.ones(mesh.n_cells))
    c_full = compliance(prob, fem.newton_solve(prob)[0])
    prob.set_theta(np.full(mesh.n_cells, 0.5))
    c_half = compliance(prob, fem.newton_solve(prob)[0])
    assert np.isclose(c_half, c_full / 0.125, rtol=1e-8)


def test_zero_traction_compliance(rng):
    _, prob = simp_cantilever((2, 2, 1), (1.0, 1.0, 1.0), fem.LinearElastic(ALU), neumann=False)
    assert compliance(prob, rng.standard_normal(prob.n_dofs)) == 0.0


def test_density_filter_uniform_field_unchanged():
    mesh = fem.generate_box_mesh(4, 3, 2, 4.0, 3.0, 2.0)
    x = np.full(mesh.n_cells, 0.37)
    assert np.allclose(density_filter(mesh, radius=1.6)(x), x, rtol=1e-14)


def test_density_filter_small_radius_is_identity(rng):
    mesh = fem.generate_box_mesh(4, 3, 2, 4.0, 3.0, 2.0)
    x = rng.standard_normal(mesh.n_cells)
    assert np.array_equal(density_filter(mesh, radius=0.5)(x), x)


def test_density_filter_matches_brute_force(rng):
    mesh = fem.generate_box_mesh(3, 3, 2, 3.0, 3.0, 2.0)
    r = 1.7
    x = rng.standard_normal(mesh.n_cells)
    cent = element_centroids(mesh)
    expect = np.zeros(mesh.n_cells)
    for i in range(mesh.n_cells):
        w = np.maximum(0.0, r - np.linalg.norm(cent - cent[i], axis=1))
        expect[i] = (w * x).sum() / w.sum()
    assert np.allclose(density_filter(mesh, radius=r)(x), expect, rtol=1e-12)


def test_density_filter_linearity(rng):
    mesh = fem.generate_box_mesh(3, 3, 1, 3.0, 3.0, 1.0)
    f = density_filter(mesh, radius=1.4)
    x, y = rng.standard_normal(mesh.n_cells), rng.standard_normal(mesh.n_cells)
    rhs = 2.5 * f(x) - 1.25 * f(y)
    assert np.abs(f(2.5 * x - 1.25 * y) - rhs).max() <= 1e-12 * max(1.0, np.abs(rhs).max())


def test_density_filter_rejects_bad_radius():
    mesh = fem.generate_box_mesh(2, 2, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        density_filter(mesh, radius=0.0)


def test_filter_sensitivities_uniform_theta(rng):
    mesh = fem.generate_box_mesh(3, 3, 1, 3.0, 3.0, 1.0)
    f = density_filter(mesh, radius=1.4)
    s = rng.standard_normal(mesh.n_cells)
    assert np.allclose(filter_sensitivities(f, np.full(mesh.n_cells, 0.5), s), f(s), rtol=1e-12)


def test_mma_zero_gradient_inactive_constraint():
    x = np.linspace(0.2, 0.8, 10)
    xn = mma_update(MmaState.fresh(10), x, np.zeros(10), -0.1, np.full(10, 0.1), 1e-3, 1.0)
    assert np.abs(xn - x).max() < 1e-12


def test_mma_uniform_sensitivity_hits_volume_target():
    x = np.full(10, 0.6)
    xn = mma_update(MmaState.fresh(10), x, -np.ones(10), 0.6 - 0.5, np.full(10, 0.1), 1e-3, 1.0)
    assert abs(xn.mean() - 0.5) < 1e-6
    assert np.ptp(xn) < 1e-12


def test_mma_respects_move_limit_and_bounds(rng):
    x = rng.uniform(0.2, 0.9, 20)
    xn = mma_update(MmaState.fresh(20, move_limit=0.2), x, -rng.uniform(0.5, 2.0, 20), -1.0, np.full(20, 0.05), 1e-3,
                    1.0)
    assert np.all(xn <= 1.0 + 1e-12) and np.all(xn >= 1e-3 - 1e-12)
    assert np.abs(xn - x).max() <= 0.2 * (1.0 - 1e-3) + 1e-12


def test_mma_device_tensors_stay_on_device(rng):
    x = D.to_device(rng.uniform(0.2, 0.9, 30))
    xn = mma_update(MmaState.fresh(30), x, D.to_device(rng.standard_normal(30)), 0.1, np.full(30, 1 / 30), 1e-3, 1.0)
    assert D.is_device_tensor(xn)


def test_optimize_mma_stationary_feasible_point():
    from paper_2212_00964_b200.adjoint import optimize

    theta0 = np.full(6, 0.5)
    theta, hist = optimize(lambda t: (1.0, np.zeros(t.shape[0])), theta0, method="mma", max_iters=3,
                           bounds=(1e-3, 1.0), volume_constraint=lambda t: (float(t.mean() - 0.9),
                                                                            np.full(t.shape[0], 1.0 / t.shape[0])))
    assert np.abs(theta - theta0).max() < 1e-9
    assert hist.objective[1] <= hist.objective[0]


def test_run_topopt_smoke_properties():
    _, prob = simp_cantilever()
    res = run_topopt(prob, volume_fraction=0.5, n_steps=5)
    assert len(res.compliance_history) == 5 and len(res.volume_history) == 5
    for v in res.volume_history + [res.final_volume]:
        assert v <= 0.5 + 1e-6
    env = np.minimum.accumulate(res.compliance_history + [res.final_compliance])
    assert np.all(np.diff(env) <= 0)
    assert res.final_compliance < res.compliance_history[0]


def test_run_topopt_design_mask_pins_elements():
    mesh, prob = simp_cantilever((4, 2, 1), (4.0, 2.0, 1.0))
    mask = np.ones(mesh.n_cells, dtype=bool)
    mask[:2] = False
    res = run_topopt(prob, volume_fraction=0.5, n_steps=3, design_mask=mask)
    assert np.allclose(res.theta[:2], 1.0)
