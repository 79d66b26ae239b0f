"""BiCGSTAB on the GRID3 matvec pair (csrc/spmv.cu k_grid3_pair, krylov.cu
enqueue_iteration_pair): one matrix pass computes v = M p, q = M r and the lagging
w = M v, and t = q - alpha w replaces M (r - alpha v).  The iterates must follow the
two-matvec iteration up to rounding, the solves must match it, and the cross-CTA
dependency waits must never read a stale v (which would show up as O(1) differences)."""

import os

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from cases import CASES
from pkg_cases import build

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in ("B200FEM_PAIR", "B200FEM_GRID_SLAB")}

    def set_(**kw):
        for k, v in kw.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)
    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def grid_system(dims, seed=0):
    import torch
    from paper_2212_00964_b200.sparse import GridOperator
    _, prob, U = build("nh_block", dict(CASES["nh_block"], dims=dims))
    rng = np.random.default_rng(seed)
    U = (U if U is not None else np.zeros(prob.n_dofs)) + 1e-3 * rng.standard_normal(prob.n_dofs)
    ws = fem.workspace(prob)
    G = GridOperator(ws)
    ws.jacobian_grid(prob, torch.tensor(U, device="cuda"), G.device_data)
    b = torch.tensor(rng.standard_normal(prob.n_dofs), device="cuda")
    return G, b


def run_iters(G, b, iters, pair, env, slab=None):
    import torch
    env(B200FEM_PAIR=1 if pair else 0, B200FEM_GRID_SLAB=slab)
    x = torch.zeros_like(b)
    cfg = fem.LinearSolveConfig(rel_tol=1e-300, abs_tol=1e-300, max_iters=iters)
    with pytest.raises(fem.LinearSolverError):
        fem.solvers._bicgstab_device(G, b, x, False, cfg, method="bicgstab")
    return x.cpu().numpy()


# (12, 7, 9): one slab; slab rows 1/2/3 force many slabs, halo rows and ragged last slabs;
# (31, 2, 6) / (5, 1, 40): flat and thin lattices
@pytest.mark.parametrize("dims,slab", [((12, 7, 9), None), ((12, 7, 9), 2), ((12, 11, 9), 3),
                                       ((9, 14, 10), 1), ((31, 2, 6), 1), ((5, 1, 40), None)])
def test_pair_iterates_follow_two_matvec_iteration(dims, slab, env):
    G, b = grid_system(dims)
    for iters in (1, 3, 25):
        x2 = run_iters(G, b, iters, False, env, slab)
        xp = run_iters(G, b, iters, True, env, slab)
        assert rel(xp, x2) < (1e-9 if iters < 25 else 1e-7), (iters, rel(xp, x2))


def test_pair_first_iterate_bit_exact_v(env):
    """After one iteration x = alpha p + omega s: alpha comes from v = M p, which the pair
    kernel computes in the two-matvec kernel's order, so alpha is bit-identical and x
    differs from the two-matvec x only through omega (t = q - alpha w)."""
    G, b = grid_system((10, 9, 8), seed=4)
    x2 = run_iters(G, b, 1, False, env, 2)
    xp = run_iters(G, b, 1, True, env, 2)
    assert rel(xp, x2) < 1e-12


@pytest.mark.parametrize("slab", [None, 2])
def test_pair_newton_matches_two_matvec_newton(slab, env):
    dims = (11, 10, 12)
    env(B200FEM_GRID_SLAB=slab)
    out = {}
    for pair in (0, 1):
        env(B200FEM_PAIR=pair)
        _, p, _ = build("nh_block", dict(CASES["nh_block"], dims=dims))
        out[pair] = fem.newton_solve(p, cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-11),
                                     lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14, operator="grid"))
    (U0, r0), (U1, r1) = out[0], out[1]
    assert r0.n_iterations == r1.n_iterations
    assert rel(U1, U0) < 1e-9


def test_pair_deterministic(env):
    env(B200FEM_PAIR=1, B200FEM_GRID_SLAB=3)
    outs = []
    for _ in range(2):
        _, p, _ = build("nh_block", dict(CASES["nh_block"], dims=(10, 12, 11)))
        U, _ = fem.newton_solve(p, lin_cfg=fem.LinearSolveConfig(operator="grid"))
        outs.append(U)
    assert np.array_equal(outs[0], outs[1])
