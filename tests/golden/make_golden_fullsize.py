"""Reference goldens for BASELINE configs C2, C4 and C5 at their stated sizes.

Runs the REFERENCE package (gradfem) in the build container (the GPU box has no /root/reference):

    OPENBLAS_NUM_THREADS=1 NUMBA_NUM_THREADS=2 python tests/golden/make_golden_fullsize.py maps|c2|c4|c5

* maps: SHA-256 of the reference workspace's integer maps (indptr, indices, dest, diag_slots,
  dir_dofs, dir_row_slots; reference sparse.py:75-108, assembly.py:83-145) at C2, C4 (40^3) and
  C5 (176x88x22) -> full_maps.json.
* c2: reference newton_solve at its default tolerances (U, residual norms) and the discrete
  solution of the reference's own Newton system (K, R from gradfem.assemble_jacobian /
  assemble_residual; free block solved by Jacobi-CG to rel 1e-13) -> full_c2.npz.
* c4: reference incremental_solve(ramp_and_back(10)) at tight tolerances (Newton 1e-10/1e-12,
  BiCGSTAB 1e-11/1e-14): reactions, volume-averaged stress, Newton iterations, U at the peak and
  final steps -> full_c4.npz.
* c5: designs k = 0..2: the reference's K and R at the warm start U_{k-1} (set_theta(theta_k)), and
  U_k = U_{k-1} + dU with K dU = -R solved to rel 1e-13 (Dirichlet rows are identity rows, so the
  free block K_ff is the SPD system CG needs) -> full_c5.npz.  The reference's BiCGSTAB cannot
  reach tight tolerances here (its tol sits at the round-off floor of ||b - Ax|| for design 0,
  DESIGN.md section 4), so the Newton system is solved outside it; SIMP-LE is linear, so U_k is
  the reference Newton step's exact target.
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem as gf  # noqa: E402
from gradfem.assembly import workspace  # noqa: E402
from gradfem.solvers import volume_averaged_stress  # noqa: E402, F401

import fullsize_cases as fc  # noqa: E402

TIGHT_NEWTON = dict(rel_tol=1e-10, abs_tol=1e-12)
TIGHT_LINEAR = dict(rel_tol=1e-11, abs_tol=1e-14)


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def exact_newton_step(prob, U, rtol=1e-13):
    """U + dU with K(U) dU = -R(U), from the reference's own K and R; free block by Jacobi-CG."""
    import scipy.sparse as sp
    from scipy.sparse.linalg import cg

    ws = workspace(prob)
    R = gf.assemble_residual(prob, U)
    K = gf.assemble_jacobian(prob, U)
    n = R.size
    A = sp.csr_matrix((K.data, K.indices, K.indptr), shape=(n, n))
    free = np.ones(n, bool)
    free[ws.dir_dofs] = False
    dU = np.zeros(n)
    dU[ws.dir_dofs] = -R[ws.dir_dofs]  # identity rows
    Aff = A[free][:, free]
    rhs = -R[free] - A[free][:, ~free] @ dU[~free]
    dinv = 1.0 / Aff.diagonal()
    M = sp.diags(dinv)
    its = [0]
    x, info = cg(Aff, rhs, rtol=rtol, atol=0.0, maxiter=200000, M=M,
                 callback=lambda _: its.__setitem__(0, its[0] + 1))
    assert info == 0, f"CG info {info}"
    dU[free] = x
    lin_res = float(np.linalg.norm(A @ dU + R) / np.linalg.norm(R))
    Un = U + dU
    R1 = gf.assemble_residual(prob, Un)
    return Un, {"norm_R0": float(np.linalg.norm(R)), "norm_R1": float(np.linalg.norm(R1)),
                "lin_rel_residual": lin_res, "cg_iterations": its[0]}


def make_maps():
    out = {}
    for name, build in (("c2", fc.c2), ("c4", fc.c4), ("c5", fc.c5)):
        t0 = time.perf_counter()
        prob = build(gf)
        ws = workspace(prob)
        out[name] = fc.map_hashes(ws)
        out[name]["workspace_s"] = time.perf_counter() - t0
        log(name, out[name]["indices"]["shape"], f"{out[name]['workspace_s']:.1f}s")
        del prob, ws
    with open(os.path.join(HERE, "full_maps.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def make_c2():
    prob = fc.c2(gf)
    t0 = time.perf_counter()
    workspace(prob)
    t_ws = time.perf_counter() - t0
    t0 = time.perf_counter()
    U_d, rep = gf.newton_solve(prob)
    t_solve = time.perf_counter() - t0
    log("c2 default", rep.residual_norms, f"{t_solve:.1f}s")
    U_x, info = exact_newton_step(prob, np.zeros(prob.n_dofs))
    log("c2 exact", info)
    np.savez_compressed(os.path.join(HERE, "full_c2.npz"), U_default=U_d, norms_default=np.array(rep.residual_norms),
                        U_exact=U_x, exact_info=json.dumps(info), timing=json.dumps(
                            {"workspace_s": t_ws, "newton_s": t_solve}))


def make_c4():
    prob = fc.c4(gf)
    workspace(prob)
    sched = gf.LoadSchedule.ramp_and_back(10)
    t0 = time.perf_counter()
    h = gf.incremental_solve(prob, sched, cfg=gf.NewtonConfig(**TIGHT_NEWTON),
                             lin_cfg=gf.LinearSolveConfig(**TIGHT_LINEAR), reaction_locator=fc.c4_top(gf))
    t = time.perf_counter() - t0
    its = [r.newton_iterations for r in h.steps]
    log("c4 tight", its, [round(r.reaction, 3) for r in h.steps], f"{t:.1f}s")
    np.savez_compressed(os.path.join(HERE, "full_c4.npz"),
                        reactions=np.array([r.reaction for r in h.steps]),
                        avg_stress=np.array([r.avg_stress for r in h.steps]),
                        newton_iterations=np.array(its),
                        final_norms=np.array([r.residual_norm for r in h.steps]),
                        scales=np.array(sched.factors), U_peak=h.steps[9].U, U_final=h.steps[-1].U,
                        timing=json.dumps({"incremental_s": t}))


def make_c5(designs=3):
    prob = fc.c5(gf)
    workspace(prob)
    U = np.zeros(prob.n_dofs)
    out, infos = {}, []
    for k in range(designs):
        prob.set_theta(fc.c5_theta(k, prob.mesh.n_cells))
        t0 = time.perf_counter()
        U, info = exact_newton_step(prob, U)
        info["s"] = time.perf_counter() - t0
        log("c5 design", k, info)
        out[f"U_{k}"] = U
        infos.append(info)
    np.savez_compressed(os.path.join(HERE, "full_c5.npz"), info=json.dumps(infos), **out)


if __name__ == "__main__":
    {"maps": make_maps, "c2": make_c2, "c4": make_c4, "c5": make_c5}[sys.argv[1]]()
