"""Small forward solves for compute-sanitizer runs (SURVEY.md section 5 sanitizers).

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Cases c1 (LE cantilever), nh_block (neo-Hookean) and j2_block (J2, incremental with history
commit) of tests/golden/cases.py: residual, CSR Jacobian, GRID tangent, both Krylov methods,
Newton, plus the partitioned (local) solve and the batch law entry point.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402

import paper_2212_00964_b200 as fem  # noqa: E402
from cases import CASES, schedule_factors  # noqa: E402
from paper_2212_00964_b200.distributed import newton_solve_partitioned  # noqa: E402
from pkg_cases import build  # noqa: E402


def main():
    for name in ("c1", "nh_block", "j2_block"):
        mesh, prob, U = build(name)
        R = fem.assemble_residual(prob, U)
        K = fem.assemble_jacobian(prob, U)
        assert np.all(np.isfinite(R)) and np.all(np.isfinite(K.data))
        if "schedule" in CASES[name]:
            h = fem.incremental_solve(prob, fem.LoadSchedule(tuple(schedule_factors(CASES[name]["schedule"]))))
            print(name, "steps", len(h.steps), "newton its", [r.newton_iterations for r in h.steps])
        else:
            for method in ("bicgstab", "pcg"):
                _, p2, _ = build(name)
                _, rep = fem.newton_solve(p2, lin_cfg=fem.LinearSolveConfig(method=method))
                print(name, method, "newton its", rep.n_iterations)
    case = dict(CASES["nh_block"], dims=(4, 3, 8))
    _, prob, _ = build("nh_block", case)
    _, rep = newton_solve_partitioned(prob, nparts=2, mode="local")
    print("partitioned nh", rep.n_iterations)
    g = 1e-3 * np.random.default_rng(0).standard_normal((16, 3, 3))
    c = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)
    fem.NeoHookean(c).tangent(g)
    fem.J2Plasticity(c).flux(g, fem.QuadPointState.fresh((16,)))
    print("sanitize cases done")


if __name__ == "__main__":
    main()
