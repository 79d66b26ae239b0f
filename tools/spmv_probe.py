"""Kernel probe: SpMV GB/s and BiCGSTAB time/iteration on the config-3 matrix (short; ncu-friendly).

    python tools/spmv_probe.py [--n 136] [--reps 20] [--iters 40] [--material nh|le|poisson]
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


def problem(n, material):
    mesh = fem.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    if material == "poisson":
        onb = fem.BoundaryLocator(lambda p: (np.abs(p - 0.5) >= 0.5 - 1e-9).any(axis=-1))
        return fem.PoissonProblem(mesh, 1.0, [fem.DirichletSpec(onb, 0, lambda p: 0.0)],
                                  source=lambda p: np.ones(np.asarray(p).shape[:-1] + (1,)))
    alu = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)
    bot, top = fem.BoundaryLocator.plane(2, 0.0), fem.BoundaryLocator.plane(2, 1.0)
    specs = [fem.DirichletSpec(bot, c, lambda p: 0.0) for c in range(3)] + [
        fem.DirichletSpec(top, 2, lambda p: 0.02)]
    cls = fem.NeoHookeanProblem if material == "nh" else fem.LinearElasticityProblem
    return cls(mesh, alu, specs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=136)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--material", default="nh")
    ap.add_argument("--operator", default="csr", choices=["csr", "sym", "grid"])
    a = ap.parse_args()
    prob = problem(a.n, a.material)
    ws = fem.workspace(prob)
    N = prob.n_dofs
    U = D.zeros(N)
    K = fem.assemble_jacobian(prob, U)
    if a.operator == "sym":
        from paper_2212_00964_b200.sparse import SymOperator
        K = SymOperator(ws)
        ws.jacobian_sym(prob, U, K.device_data)
    if a.operator == "grid":
        from paper_2212_00964_b200.sparse import GridOperator
        K = GridOperator(ws)
        ws.jacobian_grid(prob, U, K.device_data)
    x = D.to_device(np.random.default_rng(0).standard_normal(N))
    y = D.empty(N)
    lib = _lib.lib()
    h = K._device_handle()
    for _ in range(3):
        lib.b200fem_matvec(h, D.ptr(x), D.ptr(y))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        lib.b200fem_matvec(h, D.ptr(x), D.ptr(y))
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / a.reps / 1e3
    nnz, nn = ws.nnz, prob.mesh.n_nodes
    vec = prob.vec
    b_fem = 8 * nnz + (4 * (nnz // 9) + 4 * (nn + 1) if vec == 3 else 4 * nnz + 4 * (N + 1)) + 16 * N
    b_csr = 12 * nnz + 4 * (N + 1) + 16 * N
    # BiCGSTAB cost per iteration: a fixed number of iterations (tolerance unreachable)
    R = D.empty(N)
    ws.residual(prob, U, R)
    b = -R
    xs = D.zeros(N)
    def solve_ms(iters):
        cfg = fem.LinearSolveConfig(rel_tol=1e-300, abs_tol=1e-300, max_iters=iters)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            fem.solvers._bicgstab_device(K, b, xs, False, cfg)
        except fem.LinearSolverError:
            pass
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    solve_ms(2)
    t_a, t_b = solve_ms(a.iters), solve_ms(2 * a.iters)
    t_it = (t_b - t_a) / a.iters / 1e3  # marginal cost of one iteration
    e0.record()
    for _ in range(3):
        if a.operator == "sym":
            ws.jacobian_sym(prob, U, K.device_data)
        elif a.operator == "grid":
            ws.jacobian_grid(prob, U, K.device_data)
        else:
            ws.jacobian(prob, U, K.device_data)
    e1.record()
    torch.cuda.synchronize()
    t_jac = e0.elapsed_time(e1) / 3 / 1e3
    e0.record()
    for _ in range(5):
        ws.residual(prob, U, R)
    e1.record()
    torch.cuda.synchronize()
    t_res = e0.elapsed_time(e1) / 5 / 1e3
    if a.operator == "sym":  # DRAM bytes of the symmetric storage: upper blocks + lower block ids
        nsym = ws.sym_size()
        b_fem = 8 * nsym + 4 * (nnz // 9 - nsym // 9) + 4 * (nnz // 9) + 4 * (nn + 1) * 2 + 16 * N
    if a.operator == "grid":  # GRID values: 14 blocks of vec^2 values per node + x + y (+ 1 B/row flags)
        b_fem = 14 * 8 * vec * vec * nn + 16 * N + N
    print(json.dumps({"n": a.n, "material": a.material, "operator": a.operator, "nnz": nnz, "spmv_us": t * 1e6,
                      "spmv_gbs_fem": b_fem / t / 1e9, "spmv_gbs_csr12": b_csr / t / 1e9,
                      "bicgstab_ms_per_iter": t_it * 1e3, "jacobian_ms": t_jac * 1e3,
                      "residual_ms": t_res * 1e3, "mcells": prob.mesh.n_cells / 1e6}))


if __name__ == "__main__":
    main()
