"""CPU reference measurements on the GPU box's host.

    python tools/cpu_reference.py ladder [n ...]       # gradfem (baseline/_ref) NH newton_solve, phase-timed
    python tools/cpu_reference.py port136 [--n 136]     # oracle port at full size + the GPU solve, U compared
    python tools/cpu_reference.py fullphases [--n 136]  # gradfem at full size: workspace, R, K, 1st BiCGSTAB

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


def fullphases(n):
    """The reference package at the FULL config-3 size, phase by phase, inside one lease: its
    workspace(), one residual, one AD Jacobian and the first Newton step's BiCGSTAB solve (the
    whole solve -- three Jacobians and ~1750 Krylov iterations, ~77 min -- does not fit one
    60-minute lease); the Newton solve's time is these measured phases times their counts."""
    gf = import_gradfem()
    threads = os.cpu_count()
    gf.backend.set_num_threads(threads)
    import fullsize_cases as fc
    from gradfem.assembly import workspace

    info = host_info()
    prob = fc.c3(gf, n)
    out = {"n": n, "host": info, "threads": threads, "kind": "reference package, full size, per phase"}
    t0 = time.perf_counter()
    workspace(prob)
    out["workspace_s"] = time.perf_counter() - t0
    print(json.dumps(out), flush=True)
    U = np.zeros(prob.n_dofs)
    t0 = time.perf_counter()
    R = gf.assemble_residual(prob, U)
    out["residual_s"] = time.perf_counter() - t0
    print(json.dumps(out), flush=True)
    t0 = time.perf_counter()
    K = gf.assemble_jacobian(prob, U)
    out["jacobian_s"] = time.perf_counter() - t0
    out["jacobian_us_per_cell"] = out["jacobian_s"] / n ** 3 * 1e6
    print(json.dumps(out), flush=True)
    pt = PhaseTimer(gf)
    try:
        t0 = time.perf_counter()
        dU = gf.solvers.bicgstab_jacobi(K, -R)
        out["bicgstab1_s"] = time.perf_counter() - t0
    finally:
        pt.restore()
    out["bicgstab1_matvecs"] = pt.n["matvec"]
    out["bicgstab1_s_per_matvec"] = out["bicgstab1_s"] / max(pt.n["matvec"], 1)
    t0 = time.perf_counter()
    R1 = gf.assemble_residual(prob, U + dU)
    out["residual2_s"] = time.perf_counter() - t0
    out["newton_norms_0_1"] = [float(np.linalg.norm(R)), float(np.linalg.norm(R1))]
    out["peak_rss_gb"] = peak_rss_gb()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "ladder":
        ladder([int(a) for a in sys.argv[2:]] or [16, 24, 32, 48, 64])
    elif cmd == "fullphases":
        fullphases(int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 136)
    elif cmd == "port136":
        port136(int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 136)
    else:
        raise SystemExit(__doc__)


def lattice_csr(n, seed=0):
    """CSR of a vec-3 operator with the exact pattern the reference builds for an n^3 box mesh
    (sparse.py:75-108: node blocks of the 27-point lattice stencil, columns ascending), with
    diagonally dominant values (|off-diagonal row sum| < diagonal): a full-size system on which
    the reference's own Krylov code (CsrMatrix.matvec -> numba csr_matvec, bicgstab_jacobi) can
    be timed in seconds, without its ~5 min / 65 GB workspace build."""
    N1 = n + 1
    ii, jj = np.meshgrid(np.arange(N1), np.arange(N1), indexing="xy")
    ii, jj = ii.ravel(), jj.ravel()
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]  # ascending node id
    indptr_parts, cols, pself = [], [], []
    for k in range(N1):
        M = np.full((ii.size, 27), -1, dtype=np.int64)
        for t, (di, dj, dk) in enumerate(offs):
            i2, j2, k2 = ii + di, jj + dj, k + dk
            ok = (i2 >= 0) & (i2 < N1) & (j2 >= 0) & (j2 < N1) & (0 <= k2 < N1)
            M[ok, t] = i2[ok] + N1 * j2[ok] + N1 * N1 * k2
        valid = M >= 0
        cnt = valid.sum(axis=1)
        pself.append(valid[:, :13].sum(axis=1))
        indptr_parts.append(np.repeat(3 * cnt, 3))
        c3 = (3 * M[:, None, :, None] + np.arange(3)[None, None, None, :]).astype(np.int32)
        cols.append(np.broadcast_to(c3, (ii.size, 3, 27, 3))[np.broadcast_to(valid[:, None, :, None],
                                                                              (ii.size, 3, 27, 3))])
    indptr = np.zeros(3 * N1 ** 3 + 1, dtype=np.int64)
    np.cumsum(np.concatenate(indptr_parts), out=indptr[1:])
    indices = np.concatenate(cols)
    del cols
    data = np.random.default_rng(seed).uniform(-0.012, 0.0, indices.size)
    ps = np.concatenate(pself)
    rows = np.arange(3 * N1 ** 3)
    diag_pos = indptr[:-1] + 3 * np.repeat(ps, 3) + (rows % 3)
    data[diag_pos] = 1.0
    return indptr.astype(np.int32), indices, data


def reference_krylov_rates(gf, A, iters=(1, 5)):
    from gradfem.solvers import LinearSolverError

    """Wall time of the reference's bicgstab_jacobi on A at two iteration caps (each raises
    LinearSolverError at max_iters, after its explicit-residual check): per-iteration cost and
    the per-solve fixed cost (diagonal() + explicit residuals), plus one CsrMatrix.matvec."""
    b = np.ones(A.shape[0])
    x = A.matvec(b)  # numba JIT outside the timing
    t0 = time.perf_counter()
    A.matvec(b)
    t_mv = time.perf_counter() - t0
    ts = []
    for k in iters:
        t0 = time.perf_counter()
        try:
            gf.bicgstab_jacobi(A, b, cfg=gf.LinearSolveConfig(rel_tol=1e-300, abs_tol=1e-300, max_iters=k))
        except LinearSolverError:
            pass
        ts.append(time.perf_counter() - t0)
    per_it = (ts[1] - ts[0]) / (iters[1] - iters[0])
    return {"matvec_s": t_mv, "bicgstab_iter_s": per_it, "bicgstab_fixed_s": ts[0] - iters[0] * per_it,
            "raw": dict(zip(iters, ts)), "x_norm": float(np.linalg.norm(x))}


# ---------------------------------------------------------------- composed full-size estimate
C3_KRYLOV_ITERATIONS = 1763   # BiCGSTAB iterations of the config-3 Newton solve (3 solves; the B200
C3_NEWTON_SOLVES = 3          # run of the same algorithm, BENCH_r01.json; the port's CPU run at full
C3_RESIDUALS = 4              # size: profiles/r02_port136.json) and Newton residual evaluations


def measured_port_iterations():
    """Krylov iterations of the oracle port's full-size config-3 solve, if measured (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_port136.json")) as fh:
            d = json.load(fh)
        return int(d["port"]["krylov_iterations"]), "oracle port at 136^3 on the GPU box host (profiles/r02_port136.json)"
    except Exception:
        return C3_KRYLOV_ITERATIONS, "B200 solve of the same algorithm (BENCH_r01.json)"


class ReferenceComposer:
    """Wall time of the reference package's config-3 newton_solve at n_target^3, composed from
    phases of the UNMODIFIED reference (baseline/_ref) timed live on this host:

      setup    gradfem workspace() at n_ws^3, per cell  x N_e             (assembly.py:83-145)
      K        gradfem assemble_jacobian at n_cell^3, per cell x N_e      x 3 Newton solves
      R        gradfem assemble_residual at n_cell^3, per cell x N_e      x 4 evaluations
      Krylov   gradfem bicgstab_jacobi / CsrMatrix.matvec on a full-pattern n_csr^3 system
               (the reference's exact sparsity, sparse.py:75-108; scaled by nnz when n_csr <
               n_target): per-solve fixed cost (diagonal(), explicit residuals) x 3 + per-
               iteration cost x the config-3 iteration count.
    The Jacobian/residual are per-cell numpy work (chunks of 1024/8192 cells, assembly.py:28-29)
    and the matvec is memory-bound, so the per-unit rates transfer; profiles/r02_cpu_ladder.json
    holds full measured solves at 16^3-64^3 that validate the composition."""

    def __init__(self, n_target=136, n_csr=136, n_cell=10, n_ws=24):
        self.gf = import_gradfem()
        self.gf.backend.set_num_threads(os.cpu_count())
        import fullsize_cases as fc
        from gradfem.assembly import workspace
        from gradfem.sparse import CsrMatrix

        self.fc, self.n_target, self.n_csr, self.n_cell = fc, n_target, n_csr, n_cell
        t0 = time.perf_counter()
        workspace(fc.c3(self.gf, n_ws))
        self.ws_per_cell = (time.perf_counter() - t0) / n_ws ** 3
        self.prob = fc.c3(self.gf, n_cell)
        workspace(self.prob)
        self.U = 1e-4 * np.random.default_rng(1).standard_normal(self.prob.n_dofs)
        self.gf.assemble_jacobian(self.prob, self.U)  # numba / first-call costs outside the steps
        ip, ix, d = lattice_csr(n_csr)
        self.A = CsrMatrix(ip, ix, d)
        self.kry = reference_krylov_rates(self.gf, self.A)
        self.b = np.ones(self.A.shape[0])
        self.its, self.its_src = measured_port_iterations()

    def step(self):
        """One bounded live sample (~seconds): K and R at n_cell^3, four full-pattern matvecs."""
        gf, N_e = self.gf, self.n_cell ** 3
        t0 = time.perf_counter()
        gf.assemble_jacobian(self.prob, self.U)
        t_K = (time.perf_counter() - t0) / N_e
        t0 = time.perf_counter()
        gf.assemble_residual(self.prob, self.U)
        t_R = (time.perf_counter() - t0) / N_e
        t0 = time.perf_counter()
        for _ in range(4):
            self.A.matvec(self.b)
        t_mv = (time.perf_counter() - t0) / 4
        return self.compose(t_K, t_R, t_mv)

    def compose(self, t_K, t_R, t_mv):
        n = self.n_target
        Ne = n ** 3
        scale = 9 * (3 * n + 1) ** 3 / (9 * (3 * self.n_csr + 1) ** 3)  # nnz ratio
        k = self.kry
        t_vec = max(k["bicgstab_iter_s"] - 2 * k["matvec_s"], 0.0)  # BiCGSTAB vector work per iteration
        t_iter = (2 * t_mv + t_vec) * scale
        # BiCGSTAB iterations grow ~linearly with the mesh edge for other sizes
        its = self.its if n == 136 else self.its * n / 136.0
        parts = {"setup_s": self.ws_per_cell * Ne, "jacobian_s": C3_NEWTON_SOLVES * t_K * Ne,
                 "residual_s": C3_RESIDUALS * t_R * Ne,
                 "krylov_s": C3_NEWTON_SOLVES * k["bicgstab_fixed_s"] * scale + its * t_iter}
        return {"value": sum(parts.values()), "parts": parts,
                "rates": {"jacobian_us_per_cell": t_K * 1e6, "residual_us_per_cell": t_R * 1e6,
                          "matvec_s_at_n_csr": t_mv, "matvec_gbs": 12 * self.A.nnz / t_mv / 1e9,
                          "bicgstab_iter_s_at_target": t_iter,
                          "bicgstab_fixed_s_at_n_csr": k["bicgstab_fixed_s"],
                          "workspace_us_per_cell": self.ws_per_cell * 1e6},
                "krylov_iterations": its, "krylov_iterations_source": self.its_src}
