"""The N-part partitioned solve of config 3, run in "local" mode (all parts in this process on
one B200, exchanged by device copies and summed in part order): the same partition, halo plan,
overlap, captured batch graphs and Krylov code the N-rank NCCL run uses, checked against the
single-GPU solve at full size.

    python tools/dist_local_check.py [--n 136] [--parts 8] [--method bicgstab|pcg]
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fullsize_cases as fc  # noqa: E402
import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200.distributed import PartitionedSolver  # noqa: E402


def arg(name, default):
    return type(default)(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


n, parts, method = arg("--n", 136), arg("--parts", 8), arg("--method", "bicgstab")
lin = fem.LinearSolveConfig(method=method)
p1 = fc.c3(fem, n)
U1, r1 = fem.newton_solve(p1, lin_cfg=lin)
p2 = fc.c3(fem, n)
t0 = time.perf_counter()
s = PartitionedSolver(p2, nparts=parts, mode="local")
t_setup = time.perf_counter() - t0
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = s.newton_solve(lin_cfg=lin)
torch.cuda.synchronize()
t_solve = time.perf_counter() - t0
U2 = s.gather_U()
out = {"n": n, "parts": parts, "method": method, "setup_s": t_setup, "local_solve_s": t_solve,
       "newton_its": [r1.n_iterations, rep.n_iterations],
       "linear_iterations_single": [st.iterations for st in r1.linear_stats],
       "linear_iterations_parts": [st.iterations for st in rep.linear_stats],
       "norms_single": r1.residual_norms, "norms_parts": rep.residual_norms,
       "rel_l2_U_parts_vs_single": float(np.linalg.norm(U2 - U1) / np.linalg.norm(U1)),
       "ranges": [list(map(int, r)) for r in s.ranges]}
print(json.dumps(out), flush=True)
