"""Generate tests/golden/<case>_adjoint.npz by running the REFERENCE package (gradfem):
the adjoint row on the design cases of cases.py.

Run in the build container only (the GPU box has no /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_adjoint.py

Each fixture holds, for one design case:
  * w_test, theta_vjp and vjp = assemble_param_vjp(prob, U_test, theta_vjp, w_test)
    (theta_vjp is drawn outside the SIMP clip range on purpose: the reference differentiates
    at the theta it is given);
  * KT_indptr / KT_indices / KT_data = assemble_jacobian(prob, U_test).transpose();
  * the objective's dj_du at U_tight, lam_tight = adjoint_solve(...) and the total
    derivative grad_tight, with tight solver tolerances;
  * value / gradient of ReducedObjective at theta (fresh objective, tight tolerances).
plus generic_transpose.npz: a random non-symmetric CSR and its reference transpose.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem as gf  # noqa: E402
from gradfem.adjoint import ReducedObjective, adjoint_solve, total_derivative  # noqa: E402
from gradfem.assembly import assemble_param_vjp, workspace  # noqa: E402
from gradfem.inverse import (compliance, compliance_load_vector, poisson_objective,  # noqa: E402
                             poisson_objective_gradient)
from gradfem.sparse import CsrMatrix  # noqa: E402

from cases import CASES, test_vectors  # noqa: E402
from make_golden import TIGHT_LINEAR, TIGHT_NEWTON, build  # noqa: E402

DESIGN_CASES = ["poisson_design", "simp", "simp_nh"]


def objective_for(name, prob, n_nodes, rng):
    if name == "poisson_design":
        ws = workspace(prob)
        free = np.setdiff1d(np.arange(prob.n_dofs), ws.dir_dofs)
        obs = np.sort(rng.choice(free, min(6, free.size), replace=False))
        vals = 0.01 * rng.standard_normal(obs.size)
        return (obs, vals, lambda U, t: poisson_objective(U, obs, vals),
                lambda U, t: poisson_objective_gradient(U, obs, vals))
    return (None, None, lambda U, t: compliance(prob, U), lambda U, t: compliance_load_vector(prob))


def run(name):
    case = CASES[name]
    mesh, prob = build(case)
    U, theta = test_vectors(case, mesh.n_nodes, mesh.n_cells, prob.vec)
    prob.set_theta(theta)
    rng = np.random.default_rng(1000 + case["seed"])
    w = rng.standard_normal(prob.n_dofs)
    if prob.design_layout == "element":
        theta_vjp = rng.uniform(0.2, 1.1, mesh.n_cells)
    else:
        theta_vjp = rng.standard_normal(mesh.n_nodes)
    out = dict(U_test=U, theta=theta, w_test=w, theta_vjp=theta_vjp,
               vjp=assemble_param_vjp(prob, U, theta_vjp, w))
    KT = gf.assemble_jacobian(prob, U).transpose()
    out.update(KT_indptr=KT.indptr, KT_indices=KT.indices, KT_data=KT.data)

    obs, vals, obj, djdu = objective_for(name, prob, mesh.n_nodes, rng)
    if obs is not None:
        out.update(obs=obs, obs_values=vals)
    ncfg, lcfg = gf.NewtonConfig(**TIGHT_NEWTON), gf.LinearSolveConfig(**TIGHT_LINEAR)
    Ut, _ = gf.newton_solve(prob, cfg=ncfg, lin_cfg=lcfg)
    dj = djdu(Ut, theta)
    lam = adjoint_solve(prob, Ut, dj, lin_cfg=lcfg)
    out.update(U_tight=Ut, dj_du=dj, lam_tight=lam, grad_tight=total_derivative(prob, Ut, lam, prob.theta),
               objective_tight=np.array(obj(Ut, theta)))

    prob2 = build(case)[1]
    if obs is not None:
        ro = ReducedObjective(prob2, objective=lambda U_, t: poisson_objective(U_, obs, vals),
                              dj_du=lambda U_, t: poisson_objective_gradient(U_, obs, vals),
                              newton_cfg=ncfg, lin_cfg=lcfg)
    else:
        ro = ReducedObjective(prob2, objective=lambda U_, t: compliance(prob2, U_),
                              dj_du=lambda U_, t: compliance_load_vector(prob2), newton_cfg=ncfg, lin_cfg=lcfg)
    v, g = ro.value_and_gradient(theta)
    out.update(ro_value=np.array(v), ro_grad=g)
    np.savez_compressed(os.path.join(HERE, f"{name}_adjoint.npz"), **out)
    print(f"{name}: n_dofs={prob.n_dofs} |vjp|={np.linalg.norm(out['vjp']):.3e} |grad|={np.linalg.norm(g):.3e}")


def generic_transpose():
    rng = np.random.default_rng(77)
    n = 40
    dense = np.where(rng.random((n, n)) < 0.15, rng.standard_normal((n, n)), 0.0)
    dense[5, :] = 0.0  # an empty row and an empty column
    dense[:, 9] = 0.0
    rows, cols = np.nonzero(dense)
    indptr = np.zeros(n + 1, dtype=np.int32)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    A = CsrMatrix(indptr=indptr, indices=cols.astype(np.int32), data=dense[rows, cols])
    T = A.transpose()
    np.savez_compressed(os.path.join(HERE, "generic_transpose.npz"), indptr=A.indptr, indices=A.indices, data=A.data,
                        t_indptr=T.indptr, t_indices=T.indices, t_data=T.data)
    print("generic_transpose: nnz", A.data.size)


if __name__ == "__main__":
    for n in sys.argv[1:] or DESIGN_CASES:
        run(n)
    generic_transpose()
