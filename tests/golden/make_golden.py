"""Generate tests/golden/<case>.npz by running the REFERENCE package (gradfem).

Run in the build container only (the GPU box has no /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [case ...]

Each fixture holds the reference's own outputs for one case of cases.py: the mesh,
the integer maps (indptr, indices, dest, diag_slots, dir_dofs), the loads, R and
K.data at a seeded U, and the Newton / incremental results.  Tight solver
tolerances are used for the solution fields so that parity compares solutions,
not Krylov round-off trajectories ("FP64 parity of U").
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem as gf  # noqa: E402
from gradfem.assembly import workspace  # noqa: E402
from gradfem.solvers import volume_averaged_stress  # noqa: E402

from cases import CASES, node_mask, schedule_factors, test_vectors, traction_fn, value_fn  # noqa: E402

TIGHT_NEWTON = dict(rel_tol=1e-10, abs_tol=1e-12)
TIGHT_LINEAR = dict(rel_tol=1e-11, abs_tol=1e-14)


def locator(loc):
    return gf.BoundaryLocator(lambda p, loc=loc: node_mask(loc, np.atleast_2d(p)) if np.ndim(p) > 1
                              else bool(node_mask(loc, np.atleast_2d(p))[0]))


def build(case):
    mesh = gf.generate_box_mesh(*case["dims"], *case["L"])
    kind, mat = case["law"]
    c = gf.ElasticConstants(**mat) if kind != "poisson" else None
    specs = [gf.DirichletSpec(locator(loc), comp, value_fn(val, comp)) for loc, comp, val in case["dirichlet"]]
    neu = [gf.NeumannSpec(gf.boundary_facets(mesh, locator(loc)), traction_fn(t)) for loc, t in case.get("neumann", [])]
    body = None
    if "body" in case:
        body = traction_fn(case["body"])
    if kind == "poisson":
        src = None
        if "source" in case:
            s = case["source"]
            src = lambda p, s=s: np.full(np.asarray(p).shape[:-1] + (1,), s)  # noqa: E731
        prob = gf.PoissonProblem(mesh, mat["alpha"], specs, neu, source=src,
                                 design_source=bool(case.get("design_source")))
    elif kind == "le":
        prob = gf.LinearElasticityProblem(mesh, c, specs, neu, body)
    elif kind == "nh":
        prob = gf.NeoHookeanProblem(mesh, c, specs, neu, body)
    elif kind == "j2":
        prob = gf.J2PlasticityProblem(mesh, c, specs, neu, body)
    elif kind == "simp_le":
        prob = gf.SimpElasticityProblem(mesh, gf.LinearElastic(c), specs, neu, penalty=3.0)
    elif kind == "simp_nh":
        prob = gf.SimpElasticityProblem(mesh, gf.NeoHookean(c), specs, neu, penalty=3.0)
    else:
        raise ValueError(kind)
    return mesh, prob


def run(name):
    case = CASES[name]
    t0 = time.perf_counter()
    mesh, prob = build(case)
    U, theta = test_vectors(case, mesh.n_nodes, mesh.n_cells, prob.vec)
    if theta is not None:
        prob.set_theta(theta)
    ws = workspace(prob)
    out = dict(
        nodes=mesh.nodes, cells=mesh.cells.astype(np.int32), indptr=ws.indptr, indices=ws.indices,
        dest=ws.dest.astype(np.int32), diag_slots=ws.diag_slots.astype(np.int32),
        dir_dofs=ws.dir_dofs, dir_values=ws.dir_values, dir_row_slots=ws.dir_row_slots,
        f_neumann=ws.f_neumann, f_body=ws.f_body, U_test=U,
    )
    if theta is not None:
        out["theta"] = prob.theta
    kind = case["law"][0]
    if "schedule" not in case:
        out["R_test"] = gf.assemble_residual(prob, U)
        out["R_test_nodir"] = gf.assemble_residual(prob, U, apply_dirichlet=False)
        out["K_test"] = gf.assemble_jacobian(prob, U).data
        ncfg = gf.NewtonConfig(**case.get("newton", {}))
        Ud, rep = gf.newton_solve(prob, cfg=ncfg)  # reference default linear tolerances
        out["U_default"] = Ud
        out["norms_default"] = np.array(rep.residual_norms)
        prob2 = build(case)[1]
        if theta is not None:
            prob2.set_theta(theta)
        Ut, rep2 = gf.newton_solve(prob2, cfg=gf.NewtonConfig(**TIGHT_NEWTON),
                                   lin_cfg=gf.LinearSolveConfig(**TIGHT_LINEAR))
        out["U_tight"] = Ut
        out["norms_tight"] = np.array(rep2.residual_norms)
        out["avg_stress"] = volume_averaged_stress(prob2, Ut)
        if "reaction" in case:
            loc, comp = case["reaction"]
            out["reaction"] = np.array(gf.reaction_force(prob2, Ut, locator(loc), comp))
    else:
        factors = schedule_factors(case["schedule"])
        loc, comp = case["reaction"]
        hist = gf.incremental_solve(prob, gf.LoadSchedule(tuple(factors)),
                                    cfg=gf.NewtonConfig(**TIGHT_NEWTON),
                                    lin_cfg=gf.LinearSolveConfig(**TIGHT_LINEAR),
                                    reaction_locator=locator(loc), reaction_component=comp)
        out["reactions"] = np.array([r.reaction for r in hist.steps])
        out["step_iters"] = np.array([r.newton_iterations for r in hist.steps])
        out["avg_stress_hist"] = np.array([r.avg_stress for r in hist.steps])
        out["U_final"] = hist.steps[-1].U
        out["U_peak"] = hist.steps[len(factors) // 2 - 1].U
        # R/K at a plastic state: committed state after the peak step, evaluated near the peak.
        prob_s = build(case)[1]
        half = factors[: len(factors) // 2]
        hs = gf.incremental_solve(prob_s, gf.LoadSchedule(tuple(half)), cfg=gf.NewtonConfig(**TIGHT_NEWTON),
                                  lin_cfg=gf.LinearSolveConfig(**TIGHT_LINEAR))
        Upk = hs.steps[-1].U
        Uev = 1.05 * Upk + U
        out["state_eps"] = prob_s.state.eps_prev
        out["state_sig"] = prob_s.state.sig_prev
        out["U_test"] = Uev
        out["R_test"] = gf.assemble_residual(prob_s, Uev)
        out["K_test"] = gf.assemble_jacobian(prob_s, Uev).data
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {time.perf_counter() - t0:.1f}s  n_dofs={prob.n_dofs} nnz={ws.indices.size}")


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        run(n)
