"""Throughput of the other BASELINE configs on one B200 (device-timed, CUDA events).

    python tools/config_bench.py [--only c1,c2,c4,c5] [--c4n 40]

c1: LE cantilever 20x4x4, incremental_solve(ramp(1))              (CPU-reference config)
c2: Poisson 100^3 (1.03M DOF), source 1, zero on all faces        one Newton step, BiCGSTAB and PCG
c4: J2 n^3, z=0 clamped, u_z = 0.012 ramp_and_back(10)            20 load steps with history commit
c5: SIMP-LE 176x88x22, theta ~ U(0.3, 0.9) seeds 0..9             one Newton solve per design (warm start)
c5adj: the adjoint half of one config-5 design iteration: K assembly + K^T,
       adjoint BiCGSTAB on the compliance load, design VJP; plus the K^T kernel's GB/s
c5topo: full topology-optimisation iterations on the config-5 mesh, per phase:
        forward, compliance, adjoint, VJP, density filter (build once + apply), MMA update
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

ALU = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0


def c1():
    mesh = fem.generate_box_mesh(20, 4, 4, 20.0, 4.0, 4.0)
    x0 = fem.BoundaryLocator.plane(0, 0.0)
    specs = [fem.DirichletSpec(x0, c, lambda p: 0.0) for c in range(3)]
    neu = [fem.NeumannSpec(fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, 20.0)),
                           lambda p: np.broadcast_to([0.0, 0.0, -1.0], np.asarray(p).shape[:-1] + (3,)))]
    prob = fem.LinearElasticityProblem(mesh, ALU, specs, neu)
    fem.incremental_solve(prob, fem.LoadSchedule.ramp(1), reaction_locator=x0)  # warm-up incl. setup
    prob2 = fem.LinearElasticityProblem(mesh, ALU, specs, neu)
    h, dev, wall = timed(lambda: fem.incremental_solve(prob2, fem.LoadSchedule.ramp(1), reaction_locator=x0))
    r = h.steps[0]
    return {"config": "c1 LE cantilever 20x4x4", "n_dofs": prob.n_dofs, "wall_s_incl_setup": wall,
            "device_s": dev, "newton_its": r.newton_iterations, "reaction_z": r.reaction,
            "norm_U": float(np.linalg.norm(r.U)), "reference_cpu_s": "2.31 (SURVEY Appendix B, reference package)"}


def c2():
    n = 100
    mesh = fem.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    onb = fem.BoundaryLocator(lambda p: (np.abs(np.asarray(p) - 0.5) >= 0.5 - 1e-9).any(axis=-1))
    out = {"config": "c2 Poisson 100^3", "n_cells": mesh.n_cells}
    for method in ("bicgstab", "pcg"):
        prob = fem.PoissonProblem(mesh, 1.0, [fem.DirichletSpec(onb, 0, lambda p: 0.0)],
                                  source=lambda p: np.ones(np.asarray(p).shape[:-1] + (1,)))
        _, setup, _ = timed(lambda: fem.workspace(prob))
        lin = fem.LinearSolveConfig(method=method)
        fem.newton_solve(prob, D.zeros(prob.n_dofs), lin_cfg=lin)  # warm-up (K cached: jacobian_constant)
        prob._jac_cache = None
        (U, rep), dev, _ = timed(lambda: fem.newton_solve(prob, D.zeros(prob.n_dofs), lin_cfg=lin))
        out[method] = {"newton_s": dev, "setup_s": setup, "linear_iterations": [s.iterations for s in rep.linear_stats],
                       "matvecs": sum(s.matvecs for s in rep.linear_stats), "max_u": float(U.max()),
                       "norms": rep.residual_norms, "phase_s": getattr(rep, "timings", None)}
    out["n_dofs"] = prob.n_dofs
    out["reference_max_u"] = "5.622140e-02 (SURVEY 8(d), reference BiCGSTAB, 200 matvecs)"
    return out


def c4(n):
    mesh = fem.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    bot, top = fem.BoundaryLocator.plane(2, 0.0), fem.BoundaryLocator.plane(2, 1.0)
    specs = [fem.DirichletSpec(bot, c, lambda p: 0.0) for c in range(3)] + [
        fem.DirichletSpec(top, 2, lambda p: 0.012)]
    prob = fem.J2PlasticityProblem(mesh, ALU, specs)
    fem.workspace(prob)
    sched = fem.LoadSchedule.ramp_and_back(10)
    h, dev, wall = timed(lambda: fem.incremental_solve(prob, sched, reaction_locator=top))
    return {"config": f"c4 J2 {n}^3 ramp_and_back(10)", "n_dofs": prob.n_dofs, "device_s": dev, "wall_s": wall,
            "newton_its": [r.newton_iterations for r in h.steps], "reactions": [r.reaction for r in h.steps]}


def c5(method="bicgstab"):
    mesh = fem.generate_box_mesh(176, 88, 22, 8.0, 4.0, 1.0)
    x0 = fem.BoundaryLocator.plane(0, 0.0)
    specs = [fem.DirichletSpec(x0, c, lambda p: 0.0) for c in range(3)]
    neu = [fem.NeumannSpec(fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, 8.0)),
                           lambda p: np.broadcast_to([0.0, 0.0, -1.0], np.asarray(p).shape[:-1] + (3,)))]
    prob = fem.SimpElasticityProblem(mesh, fem.LinearElastic(ALU), specs, neu, penalty=3.0)
    fem.workspace(prob)
    lin = fem.LinearSolveConfig(method=method)
    U = D.zeros(prob.n_dofs)
    times, its = [], []
    for k in range(10):
        prob.set_theta(np.random.default_rng(k).uniform(0.3, 0.9, mesh.n_cells))
        (U, rep), dev, _ = timed(lambda: fem.newton_solve(prob, U, lin_cfg=lin))
        times.append(dev)
        its.append([s.iterations for s in rep.linear_stats])
    return {"config": f"c5 SIMP-LE 176x88x22 ({method})", "n_dofs": prob.n_dofs, "per_design_s": times,
            "mean_design_s": float(np.mean(times[1:])), "linear_iterations": its}


def c5adj():
    from paper_2212_00964_b200 import _lib
    from paper_2212_00964_b200.adjoint import adjoint_solve, total_derivative
    from paper_2212_00964_b200.inverse import compliance_load_vector

    mesh = fem.generate_box_mesh(176, 88, 22, 8.0, 4.0, 1.0)
    x0 = fem.BoundaryLocator.plane(0, 0.0)
    specs = [fem.DirichletSpec(x0, c, lambda p: 0.0) for c in range(3)]
    neu = [fem.NeumannSpec(fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, 8.0)),
                           lambda p: np.broadcast_to([0.0, 0.0, -1.0], np.asarray(p).shape[:-1] + (3,)))]
    prob = fem.SimpElasticityProblem(mesh, fem.LinearElastic(ALU), specs, neu, penalty=3.0)
    ws = fem.workspace(prob)
    prob.set_theta(np.random.default_rng(0).uniform(0.3, 0.9, mesh.n_cells))
    U, _ = fem.newton_solve(prob, D.zeros(prob.n_dofs), lin_cfg=fem.LinearSolveConfig(method="pcg"))
    f = D.to_device(compliance_load_vector(prob))
    th = D.to_device(prob.theta)
    out = {"config": "c5adj SIMP-LE 176x88x22 adjoint half (pcg split)", "n_dofs": prob.n_dofs, "nnz": ws.nnz}
    for rep in range(2):  # second pass is the timed one (first includes lazy allocations)
        KT, t_kt, _ = timed(lambda: fem.tangent_transpose(prob, U))
        lam, t_adj, _ = timed(lambda: adjoint_solve(prob, U, f, lin_cfg=fem.LinearSolveConfig(method="pcg")))
        g, t_vjp, _ = timed(lambda: total_derivative(prob, U, lam, th))
    K = fem.assemble_jacobian(prob, U)
    dt = D.empty(ws.nnz)
    lib = _lib.lib()
    _, t_t, _ = timed(lambda: [lib.b200fem_transpose_fem(ws.ctx, D.ptr(K.device_data), D.ptr(dt)) for _ in range(5)])
    t_t /= 5
    nb = 16 * ws.nnz + 4 * (ws.nnz // 9) + 8 * (mesh.n_nodes + 1)
    out.update({"tangent_transpose_s": t_kt, "adjoint_solve_s": t_adj, "vjp_s": t_vjp,
                "adjoint_half_s": t_kt + t_adj + t_vjp, "transpose_kernel_ms": t_t * 1e3,
                "transpose_kernel_gbs": nb / t_t / 1e9, "grad_norm": float(torch.linalg.norm(g))})
    return out


def c5topo(steps=3):
    from paper_2212_00964_b200.adjoint import adjoint_solve, total_derivative
    from paper_2212_00964_b200.inverse import (MmaState, compliance, compliance_load_vector, density_filter,
                                               filter_sensitivities, mma_update)

    mesh = fem.generate_box_mesh(176, 88, 22, 8.0, 4.0, 1.0)
    x0 = fem.BoundaryLocator.plane(0, 0.0)
    specs = [fem.DirichletSpec(x0, c, lambda p: 0.0) for c in range(3)]
    neu = [fem.NeumannSpec(fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, 8.0)),
                           lambda p: np.broadcast_to([0.0, 0.0, -1.0], np.asarray(p).shape[:-1] + (3,)))]
    prob = fem.SimpElasticityProblem(mesh, fem.LinearElastic(ALU), specs, neu, penalty=3.0)
    fem.workspace(prob)
    lin = fem.LinearSolveConfig(method="pcg")
    edge = 8.0 / 176
    filt, t_fb, _ = timed(lambda: density_filter(mesh, 1.5 * edge))
    n = mesh.n_cells
    theta = D.to_device(np.full(n, 0.5))
    st = MmaState.fresh(n)
    c_grad = D.to_device(np.full(n, 1.0 / n))
    f = D.to_device(compliance_load_vector(prob))
    U = D.zeros(prob.n_dofs)
    rows = []
    for k in range(steps):
        prob.set_theta(D.to_host(theta))
        (U, rep), t_fw, _ = timed(lambda: fem.newton_solve(prob, U, lin_cfg=lin))
        c, t_c, _ = timed(lambda: compliance(prob, U))
        lam, t_adj, _ = timed(lambda: adjoint_solve(prob, U, f, lin_cfg=lin))
        th = D.to_device(prob.theta)
        sens, t_vjp, _ = timed(lambda: total_derivative(prob, U, lam, th))
        sens, t_f, _ = timed(lambda: filter_sensitivities(filt, th, sens, prob.theta_min))
        gv = float(theta.mean()) - 0.5
        theta, t_mma, _ = timed(lambda: mma_update(st, theta, sens, gv, c_grad, prob.theta_min, 1.0))
        rows.append({"compliance": c, "forward_s": t_fw, "compliance_s": t_c, "adjoint_s": t_adj, "vjp_s": t_vjp,
                     "filter_s": t_f, "mma_s": t_mma, "pcg_iters": [s.iterations for s in rep.linear_stats]})
    return {"config": "c5topo SIMP-LE 176x88x22 topology optimisation (pcg)", "n_cells": n, "filter_nnz": filt.nnz,
            "filter_build_s": t_fb, "steps": rows}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c4,c5")
    ap.add_argument("--c4n", type=int, default=40)
    a = ap.parse_args()
    runs = {"c1": lambda: [c1()], "c2": lambda: [c2()], "c4": lambda: [c4(a.c4n)],
            "c5": lambda: [c5("bicgstab"), c5("pcg")], "c5adj": lambda: [c5adj()], "c5topo": lambda: [c5topo()]}
    for name in a.only.split(","):
        for r in runs[name]():
            print(json.dumps(r), flush=True)
