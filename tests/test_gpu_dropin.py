"""Drop-in semantics of mutable problem inputs and kernel-error localisation.

* The reference re-reads ``problem.theta`` and the J2 ``problem.state`` at every assembly
  (problems.py:76-93, 150-157): in-place edits and attribute reassignment must reach the device.
* A non-finite flux raises KernelEvaluationError naming the first element and quadrature
  point (assembly.py:216-233), not InvertedDeformationError: NaN det F is not "det F <= 0".
"""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem

pytestmark = pytest.mark.gpu
ALU = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)


def simp_problem():
    mesh = fem.generate_box_mesh(4, 2, 2, 2.0, 1.0, 1.0)
    specs = [fem.DirichletSpec(fem.BoundaryLocator.plane(0, 0.0), c, lambda p: 0.0) for c in range(3)]
    neu = [fem.NeumannSpec(fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, 2.0)),
                           lambda p: np.broadcast_to([0.0, 0.0, -1.0], np.asarray(p).shape[:-1] + (3,)))]
    return fem.SimpElasticityProblem(mesh, fem.LinearElastic(ALU), specs, neu)


def test_theta_edited_in_place_reaches_the_device():
    rng = np.random.default_rng(0)
    p = simp_problem()
    p.set_theta(rng.uniform(0.3, 0.9, p.mesh.n_cells))
    U = 1e-3 * rng.standard_normal(p.n_dofs)
    R0 = fem.assemble_residual(p, U)
    K0 = fem.assemble_jacobian(p, U).data
    p.theta[3] = 0.123  # in place, no set_theta (the reference reads problem.theta every time)
    R1 = fem.assemble_residual(p, U)
    K1 = fem.assemble_jacobian(p, U).data
    q = simp_problem()
    q.set_theta(p.theta.copy())
    assert not np.array_equal(R0, R1) and not np.array_equal(K0, K1)
    assert np.array_equal(R1, fem.assemble_residual(q, U))
    assert np.array_equal(K1, fem.assemble_jacobian(q, U).data)
    p.theta = np.full(p.mesh.n_cells, 0.5)  # attribute reassignment
    q.set_theta(np.full(p.mesh.n_cells, 0.5))
    assert np.array_equal(fem.assemble_residual(p, U), fem.assemble_residual(q, U))


def j2_problem(n=3):
    mesh = fem.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    bot, top = fem.BoundaryLocator.plane(2, 0.0), fem.BoundaryLocator.plane(2, 1.0)
    specs = [fem.DirichletSpec(bot, c, lambda p: 0.0) for c in range(3)] + [
        fem.DirichletSpec(top, 2, lambda p: 0.012)]
    return fem.J2PlasticityProblem(mesh, ALU, specs)


def test_j2_state_edited_in_place_reaches_the_device():
    p = j2_problem()
    h = fem.incremental_solve(p, fem.LoadSchedule.ramp(3))  # plastic: state committed 3 times
    U = h.steps[-1].U
    R0 = fem.assemble_residual(p, U)
    st = p.state
    assert np.abs(st.sig_prev).max() > 1.0
    st.sig_prev[2, 5, 0, 1] += 7.0  # in place on the object the problem handed out
    st.eps_prev[0, 0] *= 0.5
    R1 = fem.assemble_residual(p, U)
    q = j2_problem()
    q.state = fem.QuadPointState(st.eps_prev.copy(), st.sig_prev.copy())
    assert not np.array_equal(R0, R1)
    assert np.array_equal(R1, fem.assemble_residual(q, U))
    assert np.array_equal(fem.assemble_jacobian(p, U).data, fem.assemble_jacobian(q, U).data)
    # commit starts from the edited state, then the old view goes stale (a new object)
    p.commit(U)
    q.commit(U)
    assert p.state is not st
    assert np.array_equal(p.state.sig_prev, q.state.sig_prev)


def test_j2_state_edited_before_first_assembly():
    p = j2_problem()
    p.state.sig_prev[:] = 10.0  # before the device context exists
    q = j2_problem()
    q.state = fem.QuadPointState(np.zeros((q.mesh.n_cells, 8, 3, 3)), np.full((q.mesh.n_cells, 8, 3, 3), 10.0))
    U = np.zeros(p.n_dofs)
    assert np.array_equal(fem.assemble_residual(p, U), fem.assemble_residual(q, U))


@pytest.mark.parametrize("kind", ["le", "nh", "j2", "poisson"])
def test_nonfinite_u_raises_kernel_evaluation_error_naming_the_element(kind):
    mesh = fem.generate_box_mesh(3, 2, 2, 1.0, 1.0, 1.0)
    if kind == "poisson":
        prob = fem.PoissonProblem(mesh, 1.0, [])
    else:
        cls = {"le": fem.LinearElasticityProblem, "nh": fem.NeoHookeanProblem, "j2": fem.J2PlasticityProblem}[kind]
        prob = cls(mesh, ALU, [])
    node = 7  # (i, j, k) = (3, 1, 0): cells 2 and 5 share it; cell 2 is the first
    first = int(np.flatnonzero((mesh.cells == node).any(axis=1))[0])
    U = np.zeros(prob.n_dofs)
    U[node * prob.vec] = np.nan
    msg = f"non-finite value in flux kernel \\[element {first}, quad point 0\\]"
    with pytest.raises(fem.KernelEvaluationError, match=msg):
        fem.assemble_residual(prob, U)
    with pytest.raises(fem.KernelEvaluationError, match=msg):
        fem.assemble_jacobian(prob, U)
    # the context stays usable after the error
    assert np.all(np.isfinite(fem.assemble_residual(prob, np.zeros(prob.n_dofs))))


def test_large_host_results_are_plain_writable_numpy():
    """Host arrays in give host arrays out: results of >= 1 MiB come back through a pinned
    buffer (_device.to_host) but are ordinary float64 numpy arrays, equal to the device
    values, writable, and independent of later solves."""
    import torch

    from paper_2212_00964_b200 import _device as D

    x = torch.arange(300_000, dtype=torch.float64, device="cuda") * 0.5
    a = D.to_host(x)
    b = D.to_host(x[:10])
    assert isinstance(a, np.ndarray) and a.dtype == np.float64 and a.shape == (300_000,)
    assert np.array_equal(a, np.arange(300_000) * 0.5) and np.array_equal(b, a[:10])
    a[0] = 7.0
    assert float(x[0]) == 0.0
    x.fill_(1.0)
    c = D.to_host(x)
    assert a[1] == 0.5 and np.all(c == 1.0)
