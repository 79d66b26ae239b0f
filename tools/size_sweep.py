"""SpMV / Krylov / assembly throughput against the mesh size (NH box n^3, config-3 boundary
conditions): where the operator leaves L2 (126 MB) and the kernels become HBM-bound.

    python tools/size_sweep.py [--sizes 24,32,48,64,96,136,160]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200 import _device as D  # noqa: E402
from paper_2212_00964_b200 import _lib  # noqa: E402
from paper_2212_00964_b200.sparse import GridOperator  # noqa: E402


def ev_time(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def run(n):
    mesh = fem.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    bot, top = fem.BoundaryLocator.plane(2, 0.0), fem.BoundaryLocator.plane(2, 1.0)
    specs = [fem.DirichletSpec(bot, c, lambda p: 0.0) for c in range(3)] + [
        fem.DirichletSpec(top, 2, lambda p: np.full(np.asarray(p).shape[:-1], 0.02) if np.ndim(p) > 1 else 0.02)]
    prob = fem.NeoHookeanProblem(mesh, fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0), specs)
    ws = fem.workspace(prob)
    N, nn = prob.n_dofs, mesh.n_nodes
    U = D.zeros(N)
    K = fem.assemble_jacobian(prob, U)
    G = GridOperator(ws)
    ws.jacobian_grid(prob, U, G.device_data)
    x = D.to_device(np.random.default_rng(0).standard_normal(N))
    y = D.empty(N)
    lib = _lib.lib()
    reps = max(5, int(2e9 / (ws.nnz * 8)))
    t_csr = ev_time(lambda: lib.b200fem_matvec(K._device_handle(), D.ptr(x), D.ptr(y)), reps)
    t_grid = ev_time(lambda: lib.b200fem_matvec(G._device_handle(), D.ptr(x), D.ptr(y)), reps)
    b_csr = 8 * ws.nnz + 4 * (ws.nnz // 9) + 4 * (nn + 1) + 16 * N
    b_grid = 14 * 72 * nn + 16 * N + N
    t_jac = ev_time(lambda: ws.jacobian_grid(prob, U, G.device_data), 3)
    R = D.empty(N)
    t_res = ev_time(lambda: ws.residual(prob, U, R), 5)
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    Us, rep = fem.newton_solve(prob, D.zeros(N))
    torch.cuda.synchronize()
    t_newton = time.perf_counter() - t0
    its = sum(s.iterations for s in rep.linear_stats)
    return {"n": n, "n_dofs": N, "grid_MB": b_grid / 1e6, "csr_MB": b_csr / 1e6,
            "spmv_grid_us": t_grid * 1e6, "spmv_grid_gbs": b_grid / t_grid / 1e9,
            "spmv_csr_us": t_csr * 1e6, "spmv_csr_gbs": b_csr / t_csr / 1e9,
            "tangent_ms": t_jac * 1e3, "tangent_mcells_s": mesh.n_cells / t_jac / 1e6,
            "residual_ms": t_res * 1e3, "residual_mcells_s": mesh.n_cells / t_res / 1e6,
            "newton_s": t_newton, "newton_its": rep.n_iterations, "bicgstab_its": its,
            "s_per_bicgstab_it": t_newton / max(its, 1)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="24,32,48,64,96,136,160")
    a = ap.parse_args()
    for n in [int(v) for v in a.sizes.split(",")]:
        print(json.dumps(run(n)), flush=True)
        torch.cuda.empty_cache()
