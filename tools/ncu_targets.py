"""One launch of each config-3 hot kernel for ncu (run under ncu with a -k filter):

    ncu --set full --clock-control none --import-source on -k regex:'k_jacobian_v2|k_grid_pull' \
        -c 2 -o gpurun_out/r02_tangent python tools/ncu_targets.py tangent

modes: tangent (k_jacobian_v2 + k_grid_pull), residual (k_residual + gather), spmv (GRID3
matvec plain + the two Jacobi modes through a 2-iteration BiCGSTAB), all.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fullsize_cases as fc  # noqa: E402
import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200 import _device as D  # noqa: E402
from paper_2212_00964_b200.sparse import GridOperator  # noqa: E402


def main(mode, n=136):
    prob = fc.c3(fem, n)
    ws = fem.workspace(prob)
    U = D.to_device(1e-3 * np.random.default_rng(1).standard_normal(prob.n_dofs))
    G = GridOperator(ws)
    if mode in ("tangent", "all", "spmv"):
        ws.jacobian_grid(prob, U, G.device_data)
    if mode in ("residual", "all"):
        R = D.empty(prob.n_dofs)
        ws.residual(prob, U, R)
    if mode in ("spmv", "all"):
        x = D.to_device(np.random.default_rng(0).standard_normal(prob.n_dofs))
        G.matvec(x)
        b = D.to_device(np.ones(prob.n_dofs))
        try:
            fem.bicgstab_jacobi(G, b, cfg=fem.LinearSolveConfig(rel_tol=1e-30, abs_tol=1e-300, max_iters=2))
        except fem.LinearSolverError:
            pass
    torch.cuda.synchronize()
    print("done", mode)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
