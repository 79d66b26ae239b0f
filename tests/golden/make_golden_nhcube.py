"""Reference goldens for the config-3 problem at reduced size ("NH n^3,
2 % stretch, default tolerances"): generate_box_mesh(n, n, n, 1, 1, 1), z=0 clamped, u_z = 0.02
on z=1.  Stores the Newton residual history at the reference's default tolerances and the
tight-tolerance solution.  Build container only (the reference is not on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_nhcube.py [n ...]
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem as gf  # noqa: E402


def problem(pk, n):
    mesh = pk.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    bot, top = pk.BoundaryLocator.plane(2, 0.0), pk.BoundaryLocator.plane(2, 1.0)
    v = lambda s: (lambda p: np.full(np.asarray(p).shape[:-1], s) if np.ndim(p) > 1 else s)  # noqa: E731
    specs = [pk.DirichletSpec(bot, c, v(0.0)) for c in range(3)] + [pk.DirichletSpec(top, 2, v(0.02))]
    return pk.NeoHookeanProblem(mesh, pk.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0), specs)


if __name__ == "__main__":
    for n in [int(a) for a in sys.argv[1:]] or [16]:
        t0 = time.perf_counter()
        _, rep_d = gf.newton_solve(problem(gf, n))
        Ut, rep_t = gf.newton_solve(problem(gf, n), cfg=gf.NewtonConfig(rel_tol=1e-10, abs_tol=1e-12),
                                    lin_cfg=gf.LinearSolveConfig(rel_tol=1e-11, abs_tol=1e-14))
        np.savez_compressed(os.path.join(HERE, f"nhcube_{n}.npz"), norms_default=np.array(rep_d.residual_norms),
                            norms_tight=np.array(rep_t.residual_norms), U_tight=Ut)
        print(n, rep_d.residual_norms, rep_t.n_iterations, f"{time.perf_counter() - t0:.1f}s")
