"""Pin the oracle's adjoint row to the reference's own outputs
(tests/golden/*_adjoint.npz, generic_transpose.npz; see make_golden_adjoint.py).

Bit-exact: transposes (pure permutations).  FP64: design VJP to 1e-12 relative, adjoint
solution and total derivative to 1e-8 relative L2 (the north_star bar)."""

import numpy as np
import pytest

import oracle as orc
from conftest import load_golden
from oracle_cases import build_oracle

DESIGN = ["poisson_design", "simp", "simp_nh"]
TIGHT = dict(rel_tol=1e-11, abs_tol=1e-14)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", DESIGN)
def test_param_vjp(name):
    g = load_golden(f"{name}_adjoint")
    prob, U = build_oracle(name)
    assert np.array_equal(U, g["U_test"])
    v = orc.param_vjp(prob, U, g["theta_vjp"], g["w_test"])
    assert rel(v, g["vjp"]) < 1e-12


@pytest.mark.parametrize("name", DESIGN)
def test_transpose_bit_exact(name):
    g, ga = load_golden(name), load_golden(f"{name}_adjoint")
    ipt, ixt, dt = orc.csr_transpose(g["indptr"], g["indices"], g["K_test"])
    assert np.array_equal(ipt, ga["KT_indptr"]) and np.array_equal(ixt, ga["KT_indices"])
    assert np.array_equal(dt, ga["KT_data"])
    # structurally symmetric pattern: A^T keeps A's indptr / indices
    assert np.array_equal(ipt, g["indptr"]) and np.array_equal(ixt, g["indices"])


@pytest.mark.parametrize("name", DESIGN)
def test_adjoint_and_total_derivative(name):
    g = load_golden(f"{name}_adjoint")
    prob, _ = build_oracle(name)
    lam = orc.adjoint_solve(prob, g["U_tight"], g["dj_du"], **TIGHT)
    assert rel(lam, g["lam_tight"]) < 1e-8
    grad = -orc.param_vjp(prob, g["U_tight"], g["theta"], lam)
    assert rel(grad, g["grad_tight"]) < 1e-8


def test_generic_transpose():
    g = load_golden("generic_transpose")
    ipt, ixt, dt = orc.csr_transpose(g["indptr"], g["indices"], g["data"])
    assert np.array_equal(ipt, g["t_indptr"]) and np.array_equal(ixt, g["t_indices"])
    assert np.array_equal(dt, g["t_data"])
