"""BiCGSTAB iteration profile of the config-3 GRID3 operator (b200fem_bicgstab_profile): the
graph-loop iteration vs its kernels one by one.  A/B switches come from the environment, e.g.

    B200FEM_NO_GRAPH=1 python tools/krylov_profile.py
"""

import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402

import fullsize_cases as fc  # noqa: E402
import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200 import _device as D  # noqa: E402
from paper_2212_00964_b200 import _lib  # noqa: E402
from paper_2212_00964_b200.sparse import GridOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 136
prob = fc.c3(fem, n)
ws = fem.workspace(prob)
U = D.to_device(1e-3 * np.random.default_rng(1).standard_normal(prob.n_dofs))
G = GridOperator(ws)
ws.jacobian_grid(prob, U, G.device_data)
b = D.to_device(np.random.default_rng(0).standard_normal(prob.n_dofs))
x = D.empty(prob.n_dofs)
out = (C.c_double * 8)()
lib = _lib.lib()
for _ in range(2):
    st = lib.b200fem_bicgstab_profile(G._device_handle(), D.ptr(b), D.ptr(x), 60, out)
names = ["graph_iter", "update_p", "spmv_jacobi_r0", "update_s", "spmv_jacobi_tt", "update_xr", "loop_cond", "sum"]
env = {k: v for k, v in os.environ.items() if k.startswith("B200FEM_")}
print(json.dumps({"status": st, "env": env, **{k: round(out[i], 2) for i, k in enumerate(names)}}))
