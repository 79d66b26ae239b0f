"""Slab-major traversal of the GRID3 matvec (csrc/spmv.cu SlabWalk): the order in which
warps visit nodes must not change any result.  Every node's rows are computed by one
thread in a fixed order, so y = A x is bit-identical for every slab height, including
segments whose chunks straddle two segments, ragged last slabs, and the node sub-ranges
of partitioned parts (interior / halo bands)."""

import os

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from cases import CASES
from paper_2212_00964_b200.distributed import PartitionedSolver
from pkg_cases import build

pytestmark = pytest.mark.gpu
TIGHT = dict(cfg=fem.NewtonConfig(rel_tol=1e-10, abs_tol=1e-11),
             lin_cfg=fem.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-13))


@pytest.fixture
def slab():
    saved = os.environ.get("B200FEM_GRID_SLAB")

    def set_(rows):
        if rows is None:
            os.environ.pop("B200FEM_GRID_SLAB", None)
        else:
            os.environ["B200FEM_GRID_SLAB"] = str(rows)
    yield set_
    set_(None if saved is None else int(saved))


def grid_of(prob, U):
    import torch
    from paper_2212_00964_b200.sparse import GridOperator
    ws = fem.workspace(prob)
    G = GridOperator(ws)
    ws.jacobian_grid(prob, torch.tensor(U, device="cuda"), G.device_data)
    return G


@pytest.mark.parametrize("dims", [(12, 7, 9), (31, 2, 6), (9, 14, 10), (5, 1, 40), (40, 3, 3)])
def test_matvec_bit_identical_for_every_slab_height(dims, slab, rng):
    _, prob, U = build("nh_block", dict(CASES["nh_block"], dims=dims))
    U = (U if U is not None else np.zeros(prob.n_dofs)) + 1e-3 * rng.standard_normal(prob.n_dofs)
    G = grid_of(prob, U)
    x = rng.standard_normal(prob.n_dofs)
    slab(0)
    y0 = G @ x
    K = fem.assemble_jacobian(prob, U)
    assert np.linalg.norm(y0 - K @ x) <= 1e-14 * np.linalg.norm(K @ x)
    for rows in (1, 2, 3, 5, dims[1] + 1, 1000):
        slab(rows)
        assert np.array_equal(G @ x, y0), rows


@pytest.mark.parametrize("rows", [1, 2])
def test_newton_and_partitioned_parts_with_slabs(rows, slab):
    """Newton through the Krylov graph loop and the partitioned solve (interior rows and the
    two halo bands are separate node ranges of the same kernel) with forced slabs equal the
    plain-order solves (to rounding: the fused Krylov dots accumulate in visiting order)."""
    case = dict(CASES["nh_block"], dims=(7, 6, 12))
    out = {}
    for r in (0, rows):
        slab(r)
        _, p1, _ = build("nh_block", case)
        U1, _ = fem.newton_solve(p1, **TIGHT)
        _, p2, _ = build("nh_block", case)
        s = PartitionedSolver(p2, nparts=3, mode="local")
        assert all(p.grid for p in s.parts)
        s.newton_solve(**TIGHT)
        out[r] = (U1, s.gather_U())
    for a, b in zip(out[0], out[rows]):
        assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(a)
