"""Ports of the reference's constitutive-law tests (reference pkg/tests/test_materials.py) to
the device flux kernels.  The reference calls its host flux functions on a grad u; here the
same grad u G is imposed as the affine field u = G x on one unit HEX8 cell, where it is
exact at every quadrature point, and the flux comes back through `quad_point_stress`
(k_qp, csrc/element.cu) -- so every law is evaluated by the code the forward solve uses."""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem

pytestmark = pytest.mark.gpu


@pytest.fixture
def aluminum():
    return fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)


def device_flux(cls, c, G, problem=None):
    """Flux at the 8 quadrature points of the unit cell under u = G x (all equal)."""
    mesh = fem.generate_box_mesh(1, 1, 1, 1.0, 1.0, 1.0)
    prob = problem or cls(mesh, c, [])
    U = (mesh.nodes @ np.asarray(G).T).ravel()
    P = fem.quad_point_stress(prob, U)[0]
    assert np.abs(P - P[0]).max() <= 1e-10 * max(1.0, np.abs(P).max())  # round-off x moduli
    return P[0], prob, U


def test_linear_elastic_closed_form():
    """test_materials.py:38-42"""
    c = fem.ElasticConstants(E=1.0, nu=0.25)
    assert np.allclose(device_flux(fem.LinearElasticityProblem, c, np.zeros((3, 3)))[0], 0.0)
    sig = device_flux(fem.LinearElasticityProblem, c, np.diag([0.01, 0.0, 0.0]))[0]
    assert np.allclose(sig, np.diag([0.012, 0.004, 0.004]))


def test_linear_elastic_kills_skew_part(aluminum, rng):
    """test_materials.py:45-49"""
    W = rng.standard_normal((3, 3))
    sig = device_flux(fem.LinearElasticityProblem, aluminum, 0.5 * (W - W.T))[0]
    assert np.abs(sig).max() < 1e-12 * 70e3


def nh_flux_closed_form(grad_u, c):  # test_materials.py:70-77
    F = grad_u + np.eye(3)
    J = np.linalg.det(F)
    Fit = np.linalg.inv(F).T
    I1 = np.trace(F.T @ F)
    return c.G * J ** (-2.0 / 3.0) * (F - I1 / 3.0 * Fit) + c.kappa * (J - 1.0) * J * Fit


def test_neo_hookean_reference_state(aluminum):
    """test_materials.py:80-82"""
    assert np.abs(device_flux(fem.NeoHookeanProblem, aluminum, np.zeros((3, 3)))[0]).max() < 1e-10


def test_neo_hookean_dilation_isotropic(aluminum):
    """test_materials.py:85-87"""
    P = device_flux(fem.NeoHookeanProblem, aluminum, 0.03 * np.eye(3))[0]
    assert np.allclose(P, P[0, 0] * np.eye(3), atol=1e-9 * abs(P[0, 0]))


def test_neo_hookean_matches_closed_form_oracle(aluminum, rng):
    """test_materials.py:105-111"""
    n = 0
    while n < 5:
        gu = 0.1 * rng.standard_normal((3, 3))
        if np.linalg.det(gu + np.eye(3)) < 0.3:
            continue
        assert np.allclose(device_flux(fem.NeoHookeanProblem, aluminum, gu)[0], nh_flux_closed_form(gu, aluminum),
                           rtol=1e-10)
        n += 1


def test_neo_hookean_rejects_inversion(aluminum):
    """test_materials.py:122-124 (through the residual, which names the element and point)"""
    mesh = fem.generate_box_mesh(1, 1, 1, 1.0, 1.0, 1.0)
    prob = fem.NeoHookeanProblem(mesh, aluminum, [])
    with pytest.raises(fem.InvertedDeformationError, match="element 0"):
        fem.assemble_residual(prob, (mesh.nodes @ (-1.5 * np.eye(3)).T).ravel())


def test_j2_elastic_branch(aluminum, rng):
    """test_materials.py:127-131"""
    gu = 1e-5 * rng.standard_normal((3, 3))
    sig = device_flux(fem.J2PlasticityProblem, aluminum, gu)[0]
    assert np.allclose(sig, device_flux(fem.LinearElasticityProblem, aluminum, gu)[0], atol=1e-12)


def test_j2_pure_shear_lands_on_yield_surface(aluminum):
    """test_materials.py:134-148"""
    gamma = 0.01
    gu = np.zeros((3, 3))
    gu[0, 1] = gu[1, 0] = gamma
    sig = device_flux(fem.J2PlasticityProblem, aluminum, gu)[0]
    s = sig - np.trace(sig) / 3.0 * np.eye(3)
    assert np.sqrt(3.0) * 2.0 * aluminum.mu * gamma > aluminum.sigma_yield
    assert np.isclose(np.sqrt(1.5 * (s * s).sum()), aluminum.sigma_yield, rtol=1e-12)
    assert np.isclose(np.trace(sig), 0.0, atol=1e-9)


def test_j2_admissibility(aluminum, rng):
    """test_materials.py:151-157 (random grad u in [-0.05, 0.05])"""
    for _ in range(20):
        sig = device_flux(fem.J2PlasticityProblem, aluminum, rng.uniform(-0.05, 0.05, (3, 3)))[0]
        s = sig - np.trace(sig) / 3.0 * np.eye(3)
        assert np.sqrt(1.5 * (s * s).sum()) <= aluminum.sigma_yield + 1e-9


def test_j2_path_dependence_against_scalar_oracle(aluminum):
    """test_materials.py:160-192: proportional loading and unloading with the history committed
    on the device after every step (J2PlasticityProblem.commit)."""
    E0 = np.diag([0.0, 0.0, 0.012])
    amplitudes = list(np.linspace(0.1, 1.0, 10)) + list(np.linspace(0.9, 0.0, 10))
    dev0 = E0 - np.trace(E0) / 3.0 * np.eye(3)
    dev_mag = np.sqrt(1.5 * (dev0 * dev0).sum())
    c_dev = press = a_prev = 0.0
    mesh = fem.generate_box_mesh(1, 1, 1, 1.0, 1.0, 1.0)
    prob = fem.J2PlasticityProblem(mesh, aluminum, [])
    for a in amplitudes:
        da = a - a_prev
        c_trial = c_dev + 2.0 * aluminum.mu * da
        s_eff = abs(c_trial) * dev_mag
        c_dev = c_trial if s_eff <= aluminum.sigma_yield else c_trial * aluminum.sigma_yield / s_eff
        press += (aluminum.lam + 2.0 * aluminum.mu / 3.0) * np.trace(E0) * da
        a_prev = a
        sig, _, U = device_flux(None, aluminum, a * E0, problem=prob)
        assert np.allclose(sig, c_dev * dev0 + press * np.eye(3), atol=1e-10)
        prob.commit(U)
    assert np.abs(sig).max() > 1.0  # residual stress after unloading to zero strain


def test_linear_elastic_symmetric_output(rng):
    """test_materials.py:52-56 (25 random grad u in [-0.05, 0.05])"""
    c = fem.ElasticConstants(E=70e3, nu=0.3)
    for _ in range(25):
        sig = device_flux(fem.LinearElasticityProblem, c, rng.uniform(-0.05, 0.05, (3, 3)))[0]
        assert np.abs(sig - sig.T).max() <= 1e-12 * max(1.0, np.abs(sig).max())


def test_linear_elastic_tangent_constant(rng):
    """test_materials.py:59-67 (the device tangent of LE does not depend on the state)"""
    c = fem.ElasticConstants(E=70e3, nu=0.3)
    mesh = fem.generate_box_mesh(2, 1, 1, 2.0, 1.0, 1.0)
    prob = fem.LinearElasticityProblem(mesh, c, [])
    Ks = [fem.assemble_jacobian(prob, 0.01 * rng.standard_normal(prob.n_dofs)).data for _ in range(3)]
    assert np.allclose(Ks[0], Ks[1], rtol=1e-12, atol=0) and np.allclose(Ks[1], Ks[2], rtol=1e-12, atol=0)


def neo_hookean_energy(F, c):  # W = G/2 (J^(-2/3) tr(F^T F) - 3) + kappa/2 (J - 1)^2 (materials.py:80-84)
    J = np.linalg.det(F)
    return 0.5 * c.G * (J ** (-2.0 / 3.0) * np.trace(F.T @ F) - 3.0) + 0.5 * c.kappa * (J - 1.0) ** 2


def test_neo_hookean_matches_fd_of_energy(aluminum, rng):
    """test_materials.py:90-103: the device flux against central differences of the energy"""
    gu = 1e-3 * rng.standard_normal((3, 3))
    P = device_flux(fem.NeoHookeanProblem, aluminum, gu)[0]
    h = 1e-6
    F = gu + np.eye(3)
    P_fd = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            d = np.zeros((3, 3))
            d[i, j] = h
            P_fd[i, j] = (neo_hookean_energy(F + d, aluminum) - neo_hookean_energy(F - d, aluminum)) / (2 * h)
    assert np.abs(P - P_fd).max() / np.abs(P_fd).max() < 1e-6


def test_neo_hookean_objectivity(aluminum, rng):
    """test_materials.py:114-120 states it on the energy, W(QF) = W(F); the device evaluates
    the flux, for which it reads P(QF) = Q P(F) (10 random rotations)."""
    from scipy.spatial.transform import Rotation

    F = np.eye(3) + 0.05 * rng.standard_normal((3, 3))
    P0 = device_flux(fem.NeoHookeanProblem, aluminum, F - np.eye(3))[0]
    for q in Rotation.random(10, rng).as_matrix():
        Pq = device_flux(fem.NeoHookeanProblem, aluminum, q @ F - np.eye(3))[0]
        assert np.allclose(Pq, q @ P0, rtol=1e-10, atol=1e-10 * np.abs(P0).max())


def test_j2_tangent_finite_at_zero_deviator(aluminum):
    """test_materials.py:193-196: the consistent tangent at a zero deviator (pure dilation and
    the reference state) is finite"""
    mesh = fem.generate_box_mesh(1, 1, 1, 1.0, 1.0, 1.0)
    prob = fem.J2PlasticityProblem(mesh, aluminum, [])
    for G in (np.zeros((3, 3)), 0.01 * np.eye(3)):
        U = (mesh.nodes @ G.T).ravel()
        assert np.all(np.isfinite(fem.assemble_jacobian(prob, U).data))
        assert np.all(np.isfinite(fem.assemble_residual(prob, U)))


def test_j2_at_exact_yield_uses_elastic_branch():
    """test_materials.py:199-211: at f == 0 exactly (yield stress = the device's own trial
    s_eff) the return map keeps the elastic branch: flux and tangent equal the elastic ones"""
    base = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=1.0)
    gu = 0.003 * np.diag([1.0, 0.0, 0.0])
    sig_tr = device_flux(fem.LinearElasticityProblem, base, gu)[0]
    s = sig_tr - np.trace(sig_tr) / 3.0 * np.eye(3)
    c = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=float(np.sqrt(1.5 * (s * s).sum())))
    out, pj, U = device_flux(fem.J2PlasticityProblem, c, gu)
    ref, pl, _ = device_flux(fem.LinearElasticityProblem, c, gu)
    assert np.allclose(out, ref, rtol=1e-14, atol=0)
    assert np.allclose(fem.assemble_jacobian(pj, U).data, fem.assemble_jacobian(pl, U).data, rtol=1e-13, atol=1e-9)


def test_commit_state(aluminum, rng):
    """test_materials.py:214-228, through J2PlasticityProblem.commit on the device"""
    mesh = fem.generate_box_mesh(1, 1, 1, 1.0, 1.0, 1.0)
    prob = fem.J2PlasticityProblem(mesh, aluminum, [])
    prob.commit(np.zeros(prob.n_dofs))
    st = prob.state
    assert np.array_equal(st.eps_prev, np.zeros_like(st.eps_prev))
    assert np.array_equal(st.sig_prev, np.zeros_like(st.sig_prev))
    gu = 1e-5 * rng.standard_normal((3, 3))  # elastic range
    U = (mesh.nodes @ gu.T).ravel()
    prob.commit(U)
    st1 = prob.state
    sig_le = device_flux(fem.LinearElasticityProblem, aluminum, gu)[0]
    assert np.allclose(st1.sig_prev, np.broadcast_to(sig_le, st1.sig_prev.shape), atol=1e-12)
    prob.commit(U)  # zero increment is a fixed point
    st2 = prob.state
    assert np.array_equal(st2.eps_prev, st1.eps_prev) and np.array_equal(st2.sig_prev, st1.sig_prev)


def test_flux_zero_for_all_models(aluminum):
    """test_materials.py:231-239"""
    z = np.zeros((3, 3))
    assert np.abs(device_flux(fem.LinearElasticityProblem, aluminum, z)[0]).max() == 0.0
    assert np.abs(device_flux(fem.NeoHookeanProblem, aluminum, z)[0]).max() < 1e-10
    assert np.abs(device_flux(fem.J2PlasticityProblem, aluminum, z)[0]).max() == 0.0
    mesh = fem.generate_box_mesh(1, 1, 1, 1.0, 1.0, 1.0)
    pois = fem.PoissonProblem(mesh, 2.0, [])
    assert np.abs(fem.quad_point_stress(pois, np.zeros(pois.n_dofs))).max() == 0.0
