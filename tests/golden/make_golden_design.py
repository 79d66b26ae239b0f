"""Generate tests/golden/design.npz by running the REFERENCE package (gradfem): the design-loop
row -- density filter CSR and products, filtered sensitivities, an MMA
sequence (with asymptote history), the L2 field error, and short run_topopt / run_inference
histories with tight solver tolerances.

Run in the build container only (the GPU box has no /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_design.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem as gf  # noqa: E402
from gradfem.inverse import (MmaState, density_filter, filter_sensitivities, l2_field_error,  # noqa: E402
                             mma_update, run_inference, run_topopt)

FILTERS = [((4, 3, 2), (4.0, 3.0, 2.0), 1.6), ((3, 3, 2), (3.0, 3.0, 2.0), 1.7), ((6, 4, 3), (3.0, 2.0, 1.5), 0.8),
           ((5, 5, 1), (1.0, 1.0, 0.2), 0.45)]
TIGHT_N = dict(rel_tol=1e-10, abs_tol=1e-12)
TIGHT_L = dict(rel_tol=1e-11, abs_tol=1e-14)


def bimodal(x):
    x = np.asarray(x)
    return 10 * np.exp(-10 * np.sum((x - [0.25, 0.25, 0.1]) ** 2, axis=-1)) + 10 * np.exp(
        -10 * np.sum((x - [0.75, 0.75, 0.1]) ** 2, axis=-1))


def main():
    out = {}
    rng = np.random.default_rng(4242)
    for k, (dims, box, r) in enumerate(FILTERS):
        mesh = gf.generate_box_mesh(*dims, *box)
        f = density_filter(mesh, r)
        x = rng.standard_normal(mesh.n_cells)
        th = rng.uniform(0.0005, 1.0, mesh.n_cells)
        s = rng.standard_normal(mesh.n_cells)
        out.update({f"f{k}_indptr": f.matrix.indptr, f"f{k}_indices": f.matrix.indices, f"f{k}_data": f.matrix.data,
                    f"f{k}_x": x, f"f{k}_Hx": f(x), f"f{k}_theta": th, f"f{k}_sens": s,
                    f"f{k}_fs": filter_sensitivities(f, th, s)})
    # MMA: 5 steps (history from the third), mixed-sign sensitivities, active and inactive constraint
    n = 60
    st = MmaState.fresh(n, move_limit=0.2)
    x = rng.uniform(0.2, 0.9, n)
    out["mma_x0"] = x
    for k in range(5):
        dj = rng.standard_normal(n) * (1.0 + k)
        gv = float(x.mean() - 0.5) if k != 2 else -1.0
        c = np.full(n, 1.0 / n)
        xn = mma_update(st, x, dj, gv, c, 1e-3, 1.0)
        out.update({f"mma{k}_dj": dj, f"mma{k}_g": np.array(gv), f"mma{k}_x": xn, f"mma{k}_low": st.lower,
                    f"mma{k}_upp": st.upper})
        x = xn
    mesh = gf.generate_box_mesh(3, 3, 2, 1.0, 1.0, 0.4)
    up, ut = rng.standard_normal(mesh.n_nodes), rng.standard_normal(mesh.n_nodes)
    out.update(l2_up=up, l2_ut=ut, l2=np.array(l2_field_error(mesh, up, ut)))
    # run_topopt on the reference test's cantilever (tests/test_inverse.py:98-111)
    mesh = gf.generate_box_mesh(8, 4, 1, 8.0, 4.0, 1.0)
    right = gf.boundary_facets(mesh, gf.BoundaryLocator.plane(0, 8.0))
    t = np.array([0.0, 0.0, -1.0])
    left = gf.BoundaryLocator.plane(0, 0.0)
    prob = gf.SimpElasticityProblem(
        mesh, gf.LinearElastic(gf.ElasticConstants(E=70e3, nu=0.3)),
        [gf.DirichletSpec(left, c, lambda p: 0.0) for c in range(3)],
        [gf.NeumannSpec(right, lambda p: np.broadcast_to(t, np.asarray(p).shape[:-1] + (3,)))])
    res = run_topopt(prob, volume_fraction=0.5, n_steps=5, newton_cfg=gf.NewtonConfig(**TIGHT_N),
                     lin_cfg=gf.LinearSolveConfig(**TIGHT_L))
    out.update(topo_theta=res.theta, topo_comp=np.array(res.compliance_history), topo_vol=np.array(res.volume_history),
               topo_final=np.array(res.final_compliance))
    # run_inference, fully observed (tests/test_inverse.py:55-60, fewer iterations)
    mesh = gf.generate_box_mesh(6, 6, 2, 1.0, 1.0, 0.2)
    onb = gf.BoundaryLocator(lambda p: (np.abs(np.asarray(p)) < 1e-9).any(axis=-1)
                             | (np.abs(np.asarray(p) - np.array([1.0, 1.0, 0.2])) < 1e-9).any(axis=-1))
    pp = gf.PoissonProblem(mesh, 1.0, [gf.DirichletSpec(onb, 0, lambda p: 0.0)], design_source=True)
    inf = run_inference(pp, bimodal, n_obs=12, seed=0, max_iters=15,
                        lin_cfg=gf.LinearSolveConfig(**TIGHT_L))
    out.update(inf_obs=inf.obs_indices, inf_obj=np.array(inf.objective_history), inf_err=np.array(inf.error_history),
               inf_theta=inf.theta, inf_u_true=inf.u_true, inf_rel=np.array(inf.relative_l2_error))
    np.savez_compressed(os.path.join(HERE, "design.npz"), **out)
    print("design.npz:", len(out), "arrays; topopt compliance", res.compliance_history[0], "->", res.final_compliance)


if __name__ == "__main__":
    main()
