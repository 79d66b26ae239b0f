"""CPU reference measurements on the GPU box's host.

    python tools/cpu_reference.py ladder [n ...]       # gradfem (baseline/_ref) NH newton_solve, phase-timed
    python tools/cpu_reference.py port136 [--n 136]     # oracle port at full size + the GPU solve, U compared

ladder: the UNMODIFIED reference package (pip-installed into baseline/_ref, not /root/reference,
which does not exist on the GPU box) runs the config-3 problem (NH tensile box n^3, 2 %
stretch, newton_solve at its default tolerances) with its numba kernels on all host threads and
OPENBLAS_NUM_THREADS=1.  Phases are timed by wrapping gradfem.solvers'
assemble_residual / assemble_jacobian / bicgstab_jacobi and counting CsrMatrix.matvec calls --
the pattern of the reference's own pkg/benchmarks/bench_backends.py:25-33.  One JSON line per n.

port136: the oracle port (oracle/gradfem_oracle.py: closed-form tangents instead of the
reference's AD, same pattern / scatter / numba matvec / BiCGSTAB / Newton) at 136^3 on the host,
then the B200 solve of the same problem through the package API; prints both timings and the
relative L2 difference of the two U fields (the config-3 parity check at full size that the
reference package itself cannot run in the 62 GB build container).

Outputs JSON lines on stdout (the gpurun call redirects them into gpurun_out/).
"""

import json
import os
import platform
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402


def host_info():
    info = {"cpu": platform.processor(), "threads": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    info["cpu"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            info["mem_gb"] = round(int(fh.readline().split()[1]) / 2**20, 1)
    except OSError:
        pass
    return info


def peak_rss_gb():
    import resource

    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20


def import_gradfem():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gradfem")):
        raise SystemExit(f"reference package not installed at {ref} (see DESIGN.md section 4)")
    sys.path.insert(0, ref)
    import gradfem

    return gradfem


class PhaseTimer:
    """Wrap the reference's phase functions where newton_solve looks them up (gradfem.solvers)."""

    def __init__(self, gf):
        import gradfem.solvers as S
        import gradfem.sparse as SP

        self.S, self.SP = S, SP
        self.t = {"residual": 0.0, "jacobian": 0.0, "bicgstab": 0.0}
        self.n = {"residual": 0, "jacobian": 0, "bicgstab": 0, "matvec": 0}
        self.orig = (S.assemble_residual, S.assemble_jacobian, S.bicgstab_jacobi, SP.CsrMatrix.matvec)

        def wrap(name, fn):
            def w(*a, **k):
                t0 = time.perf_counter()
                try:
                    return fn(*a, **k)
                finally:
                    self.t[name] += time.perf_counter() - t0
                    self.n[name] += 1
            return w

        S.assemble_residual = wrap("residual", S.assemble_residual)
        S.assemble_jacobian = wrap("jacobian", S.assemble_jacobian)
        S.bicgstab_jacobi = wrap("bicgstab", S.bicgstab_jacobi)
        mv = SP.CsrMatrix.matvec

        def counted(selfm, x):
            self.n["matvec"] += 1
            return mv(selfm, x)

        SP.CsrMatrix.matvec = counted

    def restore(self):
        S, SP = self.S, self.SP
        S.assemble_residual, S.assemble_jacobian, S.bicgstab_jacobi, SP.CsrMatrix.matvec = self.orig


def gradfem_newton(gf, n, threads):
    """One config-3-shaped gradfem solve at n^3 with phase times (reference API, stock path)."""
    import fullsize_cases as fc
    from gradfem.assembly import workspace

    gf.backend.set_num_threads(threads)
    prob = fc.c3(gf, n)
    t0 = time.perf_counter()
    workspace(prob)
    t_ws = time.perf_counter() - t0
    pt = PhaseTimer(gf)
    try:
        t0 = time.perf_counter()
        U, rep = gf.newton_solve(prob)
        t_newton = time.perf_counter() - t0
    finally:
        pt.restore()
    ws = prob._ws
    nnz = int(ws.indices.size)
    return {
        "n": n, "n_cells": n ** 3, "n_dofs": prob.n_dofs, "nnz": nnz, "threads": threads,
        "workspace_s": t_ws, "newton_s": t_newton, "total_s": t_ws + t_newton,
        "phase_s": dict(pt.t), "calls": dict(pt.n), "newton_iterations": rep.n_iterations,
        "residual_norms": rep.residual_norms,
        "jacobian_us_per_cell": pt.t["jacobian"] / max(pt.n["jacobian"], 1) / n ** 3 * 1e6,
        "residual_us_per_cell": pt.t["residual"] / max(pt.n["residual"], 1) / n ** 3 * 1e6,
        "bicgstab_s_per_matvec": pt.t["bicgstab"] / max(pt.n["matvec"], 1),
        "peak_rss_gb": peak_rss_gb(), "U_norm": float(np.linalg.norm(U)),
    }


def ladder(sizes):
    gf = import_gradfem()
    threads = os.cpu_count()
    info = host_info()
    print(json.dumps({"host": info, "backend": gf.backend.backend_name(), "numba_threads": threads,
                      "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}), flush=True)
    gradfem_newton(gf, 4, threads)  # numba JIT outside the series
    for n in sizes:
        r = gradfem_newton(gf, n, threads)
        r["host"] = info["cpu"]
        print(json.dumps(r), flush=True)
    # the 1-thread tie-back of acceptance criterion 9 (pkg/test_output.txt:222: 15 s, LE 32^3)
    gf.backend.set_num_threads(1)
    import fullsize_cases as fc

    mesh = gf.generate_box_mesh(32, 32, 32, 1.0, 1.0, 1.0)
    bot, top = gf.BoundaryLocator.plane(2, 0.0), gf.BoundaryLocator.plane(2, 1.0)
    specs = [gf.DirichletSpec(bot, c, fc._const(0.0)) for c in range(3)] + [
        gf.DirichletSpec(top, 2, fc._const(0.01))]
    prob = gf.LinearElasticityProblem(mesh, gf.ElasticConstants(**fc.ALU), specs)
    t0 = time.perf_counter()
    U0 = np.zeros(prob.n_dofs)
    R = gf.assemble_residual(prob, U0)
    K = gf.assemble_jacobian(prob, U0)
    gf.bicgstab_jacobi(K, -R, cfg=gf.LinearSolveConfig(rel_tol=1e-10))
    print(json.dumps({"criterion9_le32_1thread_s": time.perf_counter() - t0,
                      "published_s": 15.0, "published_ref": "pkg/test_output.txt:222"}), flush=True)


def port136(n):
    import oracle as orc

    try:
        import numba

        numba.set_num_threads(numba.config.NUMBA_NUM_THREADS)
        threads = numba.get_num_threads()
    except Exception:
        threads = 1
    info = host_info()
    nodes, cells = orc.box_mesh(n, n, n, 1.0, 1.0, 1.0)
    law = orc.Law("nh", E=70e3, nu=0.3, sigma_yield=250.0)
    bot = np.flatnonzero(np.abs(nodes[:, 2]) <= 1e-5)
    top = np.flatnonzero(np.abs(nodes[:, 2] - 1.0) <= 1e-5)
    dd = np.concatenate([bot * 3 + c for c in range(3)] + [top * 3 + 2])
    dv = np.concatenate([np.zeros(3 * bot.size), np.full(top.size, 0.02)])
    o = np.argsort(dd)
    t0 = time.perf_counter()
    prob = orc.OracleProblem(nodes, cells, law, dd[o], dv[o])
    t_setup = time.perf_counter() - t0
    stats = {}
    t0 = time.perf_counter()
    U_cpu, norms, its = orc.newton(prob, stats=stats)
    t_newton = time.perf_counter() - t0
    out = {"n": n, "n_dofs": prob.n_dofs, "host": info, "numba_threads": threads, "kind": "port",
           "setup_s": t_setup, "newton_s": t_newton, "total_s": t_setup + t_newton, "newton_iterations": its,
           "residual_norms": norms, "matvecs": stats.get("matvecs"), "peak_rss_gb": peak_rss_gb()}
    print(json.dumps(out), flush=True)
    del prob
    # the B200 solve of the same problem (package API, default tolerances)
    import torch

    import fullsize_cases as fc
    import paper_2212_00964_b200 as fem

    if torch.cuda.is_available():
        p = fc.c3(fem, n)
        fem.workspace(p)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U_gpu, rep = fem.newton_solve(p)
        t_gpu = time.perf_counter() - t0
        d = float(np.linalg.norm(U_gpu - U_cpu) / np.linalg.norm(U_cpu))
        print(json.dumps({"n": n, "gpu_newton_s": t_gpu, "gpu_residual_norms": rep.residual_norms,
                          "rel_l2_U_gpu_vs_port": d, "max_abs_diff": float(np.max(np.abs(U_gpu - U_cpu))),
                          "U_norm": float(np.linalg.norm(U_cpu))}), flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "ladder":
        ladder([int(a) for a in sys.argv[2:]] or [16, 24, 32, 48, 64])
    elif cmd == "port136":
        port136(int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 136)
    else:
        raise SystemExit(__doc__)
