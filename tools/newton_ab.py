"""Config-3 Newton solve under environment A/B switches (one subprocess per variant):

    python tools/newton_ab.py B200FEM_VEC_SCALAR=1 [more VAR=VALUE ...]

prints, per variant (the baseline first), the device-timed solve (CUDA events, after a warm-up
solve), Newton/Krylov iteration counts, the BiCGSTAB iteration profile and the relative
difference of U against the baseline variant.
"""

import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import ctypes as C, json, os, sys
import numpy as np
sys.path[:0] = [os.environ["ROOT"], os.path.join(os.environ["ROOT"], "tests", "golden")]
import torch
import fullsize_cases as fc
import paper_2212_00964_b200 as fem
from paper_2212_00964_b200 import _device as D, _lib
from paper_2212_00964_b200.solvers import _tangent_matrix
prob = fc.c3(fem, 136)
fem.workspace(prob)
U0 = D.zeros(prob.n_dofs)
fem.newton_solve(prob, U0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(3):
    e0.record(); U, rep = fem.newton_solve(prob, U0); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
K = _tangent_matrix(prob, U, "auto")
x = D.to_device(np.random.default_rng(0).standard_normal(prob.n_dofs)); xb = D.empty(prob.n_dofs)
prof = (C.c_double * 8)()
_lib.lib().b200fem_bicgstab_profile(K._device_handle(), D.ptr(x), D.ptr(xb), 60, prof)
np.save(sys.argv[1], D.to_host(U))
print(json.dumps({"newton_s": ts, "linear_iterations": [s.iterations for s in rep.linear_stats],
                  "norms": rep.residual_norms, "graph_iter_us": prof[0], "phase_s": rep.timings}))
'''


def main():
    import numpy as np

    variants = [("baseline", {})] + [(a, dict([a.split("=", 1)])) for a in sys.argv[1:]]
    ref = None
    with tempfile.TemporaryDirectory() as d:
        for name, extra in variants:
            f = os.path.join(d, "u.npy")
            p = subprocess.run([sys.executable, "-c", CHILD, f], env=dict(os.environ, ROOT=ROOT, **extra),
                               capture_output=True, text=True, timeout=900)
            if p.returncode:
                print(json.dumps({"variant": name, "error": p.stderr[-2000:]}), flush=True)
                continue
            r = json.loads(p.stdout.strip().splitlines()[-1])
            U = np.load(f)
            if ref is None:
                ref = U
            r["rel_l2_U_vs_baseline"] = float(np.linalg.norm(U - ref) / np.linalg.norm(ref))
            print(json.dumps({"variant": name, **r}), flush=True)


if __name__ == "__main__":
    main()
