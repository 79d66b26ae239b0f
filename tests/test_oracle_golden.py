"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/*.npz).

Bit-exact: mesh, CSR pattern, scatter map, diagonal slots, Dirichlet tables.
FP64: R and K at a seeded U to 1e-12 relative (hand tangents vs the reference's AD),
solutions to 1e-8 relative L2 (the north_star bar), known answers as published.
"""

import numpy as np
import pytest

import oracle as orc
from cases import CASES, schedule_factors
from conftest import load_golden
from oracle_cases import build_oracle

FAST = [n for n in CASES if n != "j2_8"]


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", list(CASES))
def test_integer_maps_bit_exact(name):
    g = load_golden(name)
    prob, _ = build_oracle(name)
    assert np.array_equal(prob.nodes, g["nodes"])
    assert np.array_equal(prob.cells, g["cells"])
    assert np.array_equal(prob.indptr, g["indptr"])
    assert np.array_equal(prob.indices, g["indices"])
    assert np.array_equal(prob.dest, g["dest"])
    assert np.array_equal(prob.diag, g["diag_slots"])
    assert np.array_equal(prob.dir_dofs, g["dir_dofs"])
    assert np.array_equal(prob.dir_values, g["dir_values"])


@pytest.mark.parametrize("name", FAST)
def test_loads(name):
    g = load_golden(name)
    prob, _ = build_oracle(name)
    assert np.allclose(prob.f_neumann, g["f_neumann"], rtol=1e-13, atol=1e-15)
    assert np.allclose(prob.f_body, g["f_body"], rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("name", FAST)
def test_residual_and_jacobian(name):
    g = load_golden(name)
    prob, U = build_oracle(name)
    if "state_eps" in g:
        prob.eps_prev, prob.sig_prev = g["state_eps"], g["state_sig"]
        U = g["U_test"]
    if "theta" in g and prob.simp_theta is not None:
        assert np.array_equal(prob.simp_theta, g["theta"])
    R = orc.residual(prob, U)
    assert rel(R, g["R_test"]) < 1e-12
    if "R_test_nodir" in g:
        assert rel(orc.residual(prob, U, apply_dirichlet=False), g["R_test_nodir"]) < 1e-12
    K = orc.jacobian(prob, U)
    assert rel(K, g["K_test"]) < 1e-12


@pytest.mark.parametrize("name", [n for n in FAST if "schedule" not in CASES[n]])
def test_newton_solution(name):
    g = load_golden(name)
    prob, _ = build_oracle(name)
    kw = dict(rel_tol=1e-10, abs_tol=1e-12, lin_rel=1e-11, lin_abs=1e-14)
    U, norms, _ = orc.newton(prob, **kw)
    assert rel(U, g["U_tight"]) < 1e-8
    prob2, _ = build_oracle(name)
    ncfg = CASES[name].get("newton", {})
    Ud, nd, _ = orc.newton(prob2, **ncfg)
    assert len(nd) == len(g["norms_default"])
    assert rel(Ud, g["U_default"]) < 1e-6


def test_c1_known_answers():
    """Newton its 1, reaction ~16 N, |U| = 0.32318."""
    prob, _ = build_oracle("c1")
    U, norms, its = orc.newton(prob)
    assert its == 1 and len(norms) == 2
    assert abs(norms[0] - 3.5) < 1e-12
    assert abs(np.linalg.norm(U) - 0.3231822390393) < 1e-9
    left = np.flatnonzero(np.abs(prob.nodes[:, 0]) <= 1e-5)
    assert abs(orc.reaction(prob, U, left, 2) - 16.0) < 1e-6


def test_nh_criterion6_history():
    """pkg/test_output.txt:213 — the reference's published history, to 1e-6 relative."""
    prob, _ = build_oracle("nh_crit6")
    _, norms, _ = orc.newton(prob, rel_tol=1e-9, abs_tol=1e-10)
    pub = [0.060000000000000005, 7.457066921927957, 0.0012056401689689693, 3.471924728500236e-11]
    assert len(norms) == 4
    assert np.allclose(norms[:3], pub[:3], rtol=1e-9)
    assert norms[3] < 1e-9


def test_j2_block_incremental():
    g = load_golden("j2_block")
    prob, _ = build_oracle("j2_block")
    top = np.flatnonzero(np.abs(prob.nodes[:, 2] - 1.0) <= 1e-5)
    hist = orc.incremental(prob, schedule_factors(CASES["j2_block"]["schedule"]), top, 2,
                           rel_tol=1e-10, abs_tol=1e-12, lin_rel=1e-11, lin_abs=1e-14)
    react = np.array([h["reaction"] for h in hist])
    assert np.allclose(react, g["reactions"], rtol=1e-8, atol=1e-8)
    assert rel(hist[-1]["U"], g["U_final"]) < 1e-8


@pytest.mark.slow
def test_j2_8_incremental_reactions():
    g = load_golden("j2_8")
    prob, _ = build_oracle("j2_8")
    top = np.flatnonzero(np.abs(prob.nodes[:, 2] - 1.0) <= 1e-5)
    hist = orc.incremental(prob, schedule_factors(CASES["j2_8"]["schedule"]), top, 2,
                           rel_tol=1e-10, abs_tol=1e-12, lin_rel=1e-11, lin_abs=1e-14)
    assert np.allclose([h["reaction"] for h in hist], g["reactions"], rtol=1e-7, atol=1e-7)


def test_bicgstab_matches_dense(rng):
    """Reference tests/test_solvers.py:45-69 restated on the oracle."""
    d = rng.uniform(0.5, 4.0, 23)
    ip = np.arange(24, dtype=np.int32)
    ix = np.arange(23, dtype=np.int32)
    b = rng.standard_normal(23)
    assert np.allclose(orc.bicgstab(ip, ix, d, b), b / d, rtol=1e-10)
    assert np.array_equal(orc.bicgstab(ip, ix, d, np.zeros(23)), np.zeros(23))
