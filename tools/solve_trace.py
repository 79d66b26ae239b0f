"""Where the config-3 Newton solve's linear time goes outside the Krylov while-loop: runs the
solve twice (warm-up, then traced) with B200FEM_KRYLOV_TRACE=1 set by the caller, and prints
the phase split next to the host timeline krylov.cu writes to stderr.

    B200FEM_KRYLOV_TRACE=1 python tools/solve_trace.py
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]

import torch  # noqa: E402

import fullsize_cases as fc  # noqa: E402
import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200 import _device as D  # noqa: E402

prob = fc.c3(fem, int(sys.argv[1]) if len(sys.argv) > 1 else 136)
fem.workspace(prob)
for k in range(2):
    print(f"[solve {k}]", file=sys.stderr, flush=True)
    U0 = D.zeros(prob.n_dofs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    U, rep = fem.newton_solve(prob, U0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    its = [s.iterations for s in rep.linear_stats]
    print(json.dumps({"solve": k, "wall_s": wall, "phase_s": rep.timings, "linear_iterations": its,
                      "restarts": [s.restarts for s in rep.linear_stats],
                      "linear_ms_per_it": 1e3 * rep.timings["linear_s"] / sum(its)}), flush=True)
