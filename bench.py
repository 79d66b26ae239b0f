#!/usr/bin/env python
"""Benchmark: Newton-solve wall time of the 7.7M-DOF Neo-Hookean tensile box (BASELINE config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 136]

A step is one full ``newton_solve`` from U = 0 (default reference tolerances) on
generate_box_mesh(n, n, n, 1, 1, 1), z=0 clamped, u_z = 0.02 on z=1 (2 % stretch):
residual + CSR Jacobian assembly + device BiCGSTAB per Newton iteration, all inputs
resident in HBM.  `e2e` is the same solve through the public API with host buffers
(U0 from pinned host memory in, U to host out).  Inputs (CSR values 4.9 GB) are far
larger than the 126 MB L2, so no explicit flush is needed between steps.

--impl reference times the reference package itself (gradfem, pip-installed into
baseline/_ref) on the host CPU with all host threads: every phase rate is measured live
(Jacobian / residual at a small mesh, matvec and BiCGSTAB on the full 136^3 sparsity) and
composed to the config-3 solve; it prints the same metric.
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # BLAS oversubscription
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Newton-solve wall time @7.7M DOF HEX8 (NH tensile box 136^3)"
UNIT = "s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=136)
    p.add_argument("--stretch", type=float, default=0.02)
    p.add_argument("--ref-cell-n", type=int, default=10,
                   help="reference arm: mesh edge of the live Jacobian / residual sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--linear", default="bicgstab", choices=["bicgstab", "pcg"],
                   help="Krylov method of the timed Newton solve (reference default: bicgstab)")
    p.add_argument("--no-alt", action="store_true", help="skip the one-solve measurement of the other method")
    p.add_argument("--partitioned", action="store_true",
                   help="use the partitioned (multi-GPU) solver even on one rank (path check)")
    p.add_argument("--spawn", action="store_true",
                   help="launch the ranks through torch.distributed.run even for --gpus 1 (spawn-path check)")
    return p.parse_args()


def spawn_ranks(args):
    """`python bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one
    process per GPU, NCCL), exactly as the driver's torchrun command does, and pass rank 0's
    JSON line through.  Returns the exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    argv = [a for a in sys.argv[1:] if a != "--spawn"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def config(n, stretch):
    nn = (n + 1) ** 3
    return {"workload": f"NeoHookean tensile box {n}^3 HEX8, {stretch:.0%} stretch, newton_solve default tol",
            "n_cells": n ** 3, "n_dofs": 3 * nn, "nnz": 9 * (3 * n + 1) ** 3, "material": "E=70e3 nu=0.3",
            "l2_flush": "inputs (CSR values) >> 126 MB L2"}


# ------------------------------------------------------------------ CPU reference sample
def cpu_reference_sample(n_target, n_csr=64, n_cell=8):
    """Bounded cpu_baseline of our arm (~20 s): the reference package itself (baseline/_ref),
    composed to n_target^3 from live phase rates (tools/cpu_reference.py ReferenceComposer)
    with the Krylov phase measured on a 64^3 full-pattern system and scaled by nnz."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import cpu_reference as cr

    t0 = time.perf_counter()
    comp = cr.ReferenceComposer(n_target=n_target, n_csr=n_csr, n_cell=n_cell)
    r = comp.step()
    info = cr.host_info()
    return {"value": r["value"], "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
            "sample": (f"gradfem (baseline/_ref, unmodified) on {info.get('cpu')} x {os.cpu_count()} threads: "
                       f"Jacobian / residual rates at {n_cell}^3, workspace rate at 24^3, bicgstab_jacobi and "
                       f"CsrMatrix.matvec on the full {n_csr}^3 pattern (scaled by nnz to {n_target}^3), "
                       f"{r['krylov_iterations']} Krylov iterations; composed estimate (DESIGN.md section 4)"),
            "parts_s": r["parts"], "sample_wall_s": time.perf_counter() - t0}


# ----------------------------------------------------------------------- clocks sampler
class Clocks:
    def __init__(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-i", os.environ.get("LOCAL_RANK", "0"), "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_allreduces(world):
    """Allreduces per partitioned BiCGSTAB iteration: 2 with the fused dot group (on by default
    from 4 NCCL ranks, krylov_dist.cu dist_fused_dots), else 3."""
    e = os.environ.get("B200FEM_DIST_FUSED_DOTS", "")
    return 2 if (e != "0" if e else world >= 4) else 3


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# FP64 (non-tensor) DFMA peak measured on the pool's B200 (tools/fp64_peak.cu ->
# profiles/r01_fp64_peak.json): the roofline denominator of the FP64-bound assembly kernels.
FP64_PEAK_TFLOPS = 34.23
# Algorithmic FLOPs per cell of the NH kernels (FMA = 2), counted from the factored algorithm
# (DESIGN.md section 3): tangent = 8 points x ~960 (geometry, grad u, F, H, per-node vectors)
# + 36 pairs x 8 points x 63 (block update); residual = 8 points x ~770.
NH_TANGENT_FLOPS_PER_CELL = 8 * 960 + 36 * 8 * 63
NH_RESIDUAL_FLOPS_PER_CELL = 8 * 770


def jacobi_roofline(kprof, plain_bytes, rows, peak):
    """GB/s of the two Jacobi-mode matvecs the BiCGSTAB iteration runs (k_spmv_grid3_pf, 85 % of
    the bench step's kernel time), from the iteration profile (kernels timed one by one).
    Algorithmic bytes over the plain matvec: v = D^-1 A p reads D^-1 and r0 (r0.v), 16 B per row;
    t = D^-1 A s reads D^-1, 8 B per row (its t.s operand s is the matvec's own input)."""
    if not kprof:
        return None
    out = {}
    for k, extra in (("spmv_jacobi_r0", 16), ("spmv_jacobi_tt", 8)):
        us = kprof["kernels_us"].get(k)
        if us:
            b = plain_bytes + extra * rows
            gbs = b / (us * 1e-6) / 1e9
            out[k] = {"bytes_per_launch": b, "launch_us": us, "achieved_gbs": gbs, "frac": gbs / peak}
    return out


def ncu_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "spmv_traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


# -------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2212_00964_b200 as fem
    from paper_2212_00964_b200 import _device as D
    from paper_2212_00964_b200 import _lib
    from paper_2212_00964_b200.solvers import _tangent_matrix

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.partitioned:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n = args.n
    mesh = fem.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    alu = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)
    bot, top = fem.BoundaryLocator.plane(2, 0.0), fem.BoundaryLocator.plane(2, 1.0)
    s = args.stretch
    specs = [fem.DirichletSpec(bot, c, lambda p: 0.0) for c in range(3)] + [
        fem.DirichletSpec(top, 2, lambda p, s=s: np.full(np.asarray(p).shape[:-1], s) if np.ndim(p) > 1 else s)]
    prob = fem.NeoHookeanProblem(mesh, alu, specs)
    N = prob.n_dofs
    lin = fem.LinearSolveConfig(method=args.linear)
    t0 = time.perf_counter()
    if world == 1 and not args.partitioned:
        ws = fem.workspace(prob)
        U0 = D.zeros(N)
        sub, part = prob, None

        def step(lin=lin):
            return fem.newton_solve(prob, U0, lin_cfg=lin)

        def e2e_step(U0_host):
            U, _ = fem.newton_solve(prob, U0_host, lin_cfg=lin)  # pinned host in, numpy out
            return U
    else:
        from paper_2212_00964_b200.distributed import PartitionedSolver

        solver = PartitionedSolver(prob, nparts=world, mode="nccl")
        part = solver.parts[0]
        ws, sub = part.ws, part.problem

        def step(lin=lin):
            return None, solver.newton_solve(lin_cfg=lin)

        def e2e_step(U0_host):
            solver.newton_solve(U0_host, lin_cfg=lin)
            lo, hi = part.own_dofs
            return D.to_host(part.U[lo:hi])
    torch.cuda.synchronize()
    setup_s = max_over_ranks(time.perf_counter() - t0)

    for _ in range(args.warmup):
        step()
    barrier()
    clocks = Clocks()
    l0 = _lib.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    reports = []
    ev[0].record()
    for k in range(args.steps):
        U, rep = step()
        ev[k + 1].record()
        reports.append(rep)
    barrier()
    launches = _lib.launch_count() - l0
    ck = clocks.stop()
    per_step = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    total_ms = max_over_ranks(ev[0].elapsed_time(ev[-1]))
    ms = total_ms / args.steps
    rep = reports[-1]
    lin_iters = [s_.iterations for s_ in rep.linear_stats]
    matvecs = sum(s_.matvecs for s_ in rep.linear_stats)
    lin_s = (getattr(rep, "timings", None) or {}).get("linear_s")
    # one Krylov iteration inside the timed solve (restart residuals included), device time
    in_solve_iter_ms = (lin_s / max(sum(lin_iters), 1) * 1e3) if lin_s else None

    # ---------------- kernel-level evidence (after the timed region, same stream, CUDA events)
    if part is None:
        K = _tangent_matrix(prob, U, lin.operator)
        Uk = U
        n_rows_nodes, row_lo = mesh.n_nodes, 0
    else:
        K, Uk = part.K, part.U
        row_lo, row_hi = part.plan.own_local
        n_rows_nodes = row_hi - row_lo
    Nl = sub.n_dofs
    x = D.to_device(np.random.default_rng(0).standard_normal(Nl))
    y = D.empty(Nl)
    h = K._device_handle()
    lib = _lib.lib()
    for _ in range(3):
        lib.b200fem_matvec(h, D.ptr(x), D.ptr(y))
    reps = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.b200fem_matvec(h, D.ptr(x), D.ptr(y))
    e1.record()
    torch.cuda.synchronize()
    t_spmv = e0.elapsed_time(e1) / reps / 1e3
    from paper_2212_00964_b200.sparse import GridOperator
    grid_op = isinstance(K, GridOperator)
    # one BiCGSTAB iteration inside the while-graph vs its kernels timed one by one
    kprof = None
    if part is None:
        import ctypes as C

        prof = (C.c_double * 8)()
        xb = D.empty(Nl)
        if lib.b200fem_bicgstab_profile(h, D.ptr(x), D.ptr(xb), 60, prof) == 0:
            names = ["update_p", "spmv_jacobi_r0", "update_s", "spmv_jacobi_tt", "update_xr", "loop_cond"]
            kprof = {"graph_iter_us": prof[0], "kernels_us": dict(zip(names, prof[1:7])), "kernel_sum_us": prof[7],
                     "gap_us": prof[0] - prof[7], "iterations": 60}
        del xb
    ip = ws.indptr
    nnz_rows = int(ip[3 * (row_lo + n_rows_nodes)] - ip[3 * row_lo])
    rows = 3 * n_rows_nodes
    bytes_fem = 8 * nnz_rows + 4 * (nnz_rows // 9) + 4 * (n_rows_nodes + 1) + 8 * Nl + 8 * rows
    bytes_csr = 12 * nnz_rows + 4 * (rows + 1) + 8 * Nl + 8 * rows
    # GRID3: self + 13 upper-offset 3x3 blocks per node, x read once, y written, 1 B/row Dirichlet flag
    bytes_grid = 14 * 72 * n_rows_nodes + 8 * Nl + 8 * rows + rows
    bytes_alg = bytes_grid if grid_op else bytes_fem
    R = D.empty(Nl)
    e0.record()
    for _ in range(5):
        ws.residual(sub, Uk, R)
    e1.record()
    torch.cuda.synchronize()
    t_res = e0.elapsed_time(e1) / 5 / 1e3

    def time_jac(fn, reps=3):
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    if grid_op:  # the Newton loop's tangent (GRID3) and the reference-layout CSR (assemble_jacobian)
        t_jac = time_jac(lambda: ws.jacobian_grid(sub, Uk, K.device_data))
        Kc = D.empty(ws.nnz)
        t_jac_csr = time_jac(lambda: ws.jacobian(sub, Uk, Kc))
        del Kc
    else:
        t_jac = t_jac_csr = time_jac(lambda: ws.jacobian(sub, Uk, K.device_data))
    n_cells_l, n_nodes_l = sub.mesh.n_cells, sub.mesh.n_nodes

    # ---------------- e2e through the public API with host buffers
    U0_host = torch.zeros(N, dtype=torch.float64).pin_memory()
    e2e_step(U0_host)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step(U0_host)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    d2h = 8 * N if part is None else 8 * (part.own_dofs[1] - part.own_dofs[0])

    # ---------------- the other Krylov method, one device-timed solve (same problem, same tolerances)
    alt = None
    if not args.no_alt and part is None:
        other = "pcg" if args.linear == "bicgstab" else "bicgstab"
        olin = fem.LinearSolveConfig(method=other)
        barrier()
        e0.record()
        _, orep = step(olin)
        e1.record()
        torch.cuda.synchronize()
        alt = {"method": other, "newton_s": e0.elapsed_time(e1) / 1e3, "newton_iterations": orep.n_iterations,
               "linear_iterations": [s_.iterations for s_ in orep.linear_stats],
               "matvecs": sum(s_.matvecs for s_ in orep.linear_stats), "residual_norms": orep.residual_norms}

    # ---------------- opt-in inexact Newton (operator "grid32": FP32-stored tangent values, FP64
    # everything else), one device-timed solve per method; NOT the headline (the reference's
    # operator is FP64) -- reported with its distance to the FP64 solution of the timed steps
    mixed = None
    if not args.no_alt and part is None and grid_op:
        mixed = {"operator": "grid32", "note": "tangent values rounded to FP32 for the Krylov matvecs; FP64 "
                 "vectors, sums, residual and Newton test; not the reference operator, not the headline"}
        U64 = U.clone()
        for meth in ("bicgstab", "pcg"):
            mlin = fem.LinearSolveConfig(method=meth, operator="grid32")
            step(mlin)  # warm: allocates the FP32 copy
            barrier()
            e0.record()
            Um, mrep = step(mlin)
            e1.record()
            torch.cuda.synchronize()
            mixed[meth] = {"newton_s": e0.elapsed_time(e1) / 1e3, "newton_iterations": mrep.n_iterations,
                           "linear_iterations": [s_.iterations for s_ in mrep.linear_stats],
                           "residual_norms": mrep.residual_norms,
                           "rel_l2_vs_fp64_U": float(torch.linalg.vector_norm(Um - U64) /
                                                     torch.linalg.vector_norm(U64))}
        K32 = _tangent_matrix(prob, U64, "grid32")
        h32 = K32._device_handle()
        for _ in range(3):
            lib.b200fem_matvec(h32, D.ptr(x), D.ptr(y))
        e0.record()
        for _ in range(reps):
            lib.b200fem_matvec(h32, D.ptr(x), D.ptr(y))
        e1.record()
        torch.cuda.synchronize()
        t32 = e0.elapsed_time(e1) / reps / 1e3
        b32 = 14 * 36 * n_rows_nodes + 8 * Nl + 8 * rows + rows
        mixed["spmv_us"] = t32 * 1e6
        mixed["spmv_gbs"] = b32 / t32 / 1e9
        mixed["spmv_bytes_per_launch"] = b32

    peak, peak_kind = peaks()
    traffic = (ncu_traffic() or {}).get("grid3" if grid_op else "fem3")
    achieved = bytes_alg / t_spmv / 1e9
    out = {
        "metric": METRIC, "value": ms / 1e3, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generated box mesh, 2% stretch BCs)",
        "config": dict(config(n, s), parallelism=(
            f"node-slab partition x{world} (NCCL halo + {dist_allreduces(world)} allreduces per BiCGSTAB iteration)"
            if part is not None else "single GPU")),
        "e2e": {"value": e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": {"kernel": ("k_spmv_grid3 (GRID3 symmetric offset-major storage: 14 upper 3x3 blocks per node, "
                                "lower blocks re-read from L2, thread per node)") if grid_op else
                               "k_spmv_fem3_tma2 (CSR SpMV, node-blocked columns, cp.async.bulk pipeline, half-warp per node)",
                     "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "bytes_per_launch": bytes_alg,
                     "traffic": (traffic or {}).get("bytes_per_launch") if world == 1 else None,
                     "fem3_equiv_gbs": bytes_fem / t_spmv / 1e9,
                     "csr12_equiv_gbs": bytes_csr / t_spmv / 1e9, "launch_us": t_spmv * 1e6,
                     # the two modes the BiCGSTAB iteration actually runs (85 % of the step's
                     # kernel time, profiles/r02_launches_bench_final_summary.json)
                     "in_solve_modes": jacobi_roofline(kprof, bytes_alg, rows, peak) if grid_op else None},
        "newton": {"linear_method": args.linear, "iterations": rep.n_iterations,
                   "phase_s": getattr(rep, "timings", None),
                   "residual_norms": rep.residual_norms, "linear_iterations": lin_iters, "matvecs": matvecs,
                   "in_solve_iter_ms": in_solve_iter_ms, "per_step_ms": per_step},
        "krylov_profile": kprof,
        "alt_linear": alt,
        "alt_mixed_precision": mixed,
        "assembly": {"residual_ms": t_res * 1e3, "residual_mcells_s": n_cells_l / t_res / 1e6,
                     "jacobian_ms": t_jac * 1e3, "jacobian_mcells_s": n_cells_l / t_jac / 1e6,
                     "jacobian_layout": "grid3" if grid_op else "csr",
                     "jacobian_csr_ms": t_jac_csr * 1e3, "jacobian_csr_mcells_s": n_cells_l / t_jac_csr / 1e6,
                     "jacobian_csr_hbm_gbs": (8 * ws.nnz + 32 * n_cells_l + 24 * n_nodes_l + 8 * Nl) / t_jac_csr / 1e9,
                     "fp64_roofline": {
                         "bound": "fp64", "peak_tflops": FP64_PEAK_TFLOPS, "peak_kind": "measured (tools/fp64_peak.cu)",
                         "residual_flops_per_cell": NH_RESIDUAL_FLOPS_PER_CELL,
                         "residual_tflops": NH_RESIDUAL_FLOPS_PER_CELL * n_cells_l / t_res / 1e12,
                         "residual_frac": NH_RESIDUAL_FLOPS_PER_CELL * n_cells_l / t_res / 1e12 / FP64_PEAK_TFLOPS,
                         # the Newton loop's tangent (GRID3 layout when the mesh is a lattice), at
                         # this algorithm's FLOP count and at SURVEY 8(d)'s 33k per cell; the
                         # reference-layout CSR assembly (assemble_jacobian) separately
                         "tangent_flops_per_cell": NH_TANGENT_FLOPS_PER_CELL,
                         "tangent_tflops": NH_TANGENT_FLOPS_PER_CELL * n_cells_l / t_jac / 1e12,
                         "tangent_frac": NH_TANGENT_FLOPS_PER_CELL * n_cells_l / t_jac / 1e12 / FP64_PEAK_TFLOPS,
                         "tangent_frac_at_survey_33k": 33e3 * n_cells_l / t_jac / 1e12 / FP64_PEAK_TFLOPS,
                         "tangent_csr_frac": NH_TANGENT_FLOPS_PER_CELL * n_cells_l / t_jac_csr / 1e12 / FP64_PEAK_TFLOPS},
                     "per_rank": world > 1},
        "setup_s": setup_s,
        "clocks": ck,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_reference_sample(n)
    if rank == 0:
        emit(out)
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args):
    """The reference arm: the UNMODIFIED reference package (pip-installed into baseline/_ref)
    timed on this host's cores, composed to the config-3 solve (tools/cpu_reference.py
    ReferenceComposer: every phase rate measured live each step; the full-pattern 136^3 system
    for the Krylov phase).  Rank 0 only; other ranks exit 0."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import cpu_reference as cr

    t0 = time.perf_counter()
    comp = cr.ReferenceComposer(n_target=args.n, n_csr=args.n, n_cell=args.ref_cell_n)
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        comp.step()
    vals, walls, last = [], [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        last = comp.step()
        walls.append(time.perf_counter() - t0)
        vals.append(last["value"])
    v = float(np.median(vals))
    info = cr.host_info()
    sample = (f"gradfem (baseline/_ref, unmodified) on {info.get('cpu')} x {os.cpu_count()} threads "
              f"(numba; OPENBLAS_NUM_THREADS=1): per step assemble_jacobian + assemble_residual at "
              f"{args.ref_cell_n}^3 and 4 CsrMatrix.matvec on the full {args.n}^3 pattern; setup once: workspace() "
              f"rate at 24^3, bicgstab_jacobi fixed + per-iteration cost on the full pattern; composed to "
              f"{args.n}^3 with {last['krylov_iterations']} Krylov iterations ({last['krylov_iterations_source']}), "
              f"3 Jacobians, 4 residuals (DESIGN.md section 4)")
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(walls)) * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": dict(config(args.n, args.stretch), parallelism="host CPU"),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                         "sample": sample, "estimate": "composed from live phase rates",
                         "parts_s": last["parts"], "rates": last["rates"], "setup_wall_s": setup_s,
                         "step_values_s": vals},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out)


_JSON_FD = None


def emit(obj):
    """The one JSON line, on the process's original stdout (see __main__)."""
    os.write(_JSON_FD if _JSON_FD is not None else sys.stdout.fileno(), (json.dumps(obj) + "\n").encode())


if __name__ == "__main__":
    a = parse()
    if "WORLD_SIZE" not in os.environ and (a.gpus > 1 or a.spawn):
        sys.exit(spawn_ranks(a))
    # stdout carries exactly the JSON line: anything else written to fd 1 -- NCCL's
    # "NCCL version" banner under NCCL_DEBUG=VERSION, library or Python prints -- goes to stderr
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    run_reference(a) if a.impl == "reference" else run_ours(a)
