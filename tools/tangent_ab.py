"""A/B of the lattice tangent assembly paths on the config-3 problem (or --n).

    python tools/tangent_ab.py [--n 136] [--reps 5]

Runs one subprocess per variant (the switches are read once per process):
  v2    : B200FEM_TANGENT=v2    -> k_jacobian_v2 (node-lane phase A) + k_grid_pull
  v1    : B200FEM_TANGENT=v1    -> k_jacobian (pair-per-lane phase A) + k_grid_pull
Each times ws.jacobian_grid at a perturbed U (CUDA events, after warm-up), the residual, and
saves y = G x for a fixed x; the parent prints the times, Mcells/s, FP64 TFLOP/s at the survey's
33k FLOP/cell and the builder's 25.8k count, and the relative difference of the y's.
"""

import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
import numpy as np
sys.path[:0] = [os.environ["ROOT"], os.path.join(os.environ["ROOT"], "tests", "golden")]
import torch
import fullsize_cases as fc
import paper_2212_00964_b200 as fem
from paper_2212_00964_b200 import _device as D
from paper_2212_00964_b200.sparse import GridOperator
n, reps, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
prob = fc.c3(fem, n)
ws = fem.workspace(prob)
U = D.to_device(1e-3 * np.random.default_rng(1).standard_normal(prob.n_dofs))
G = GridOperator(ws)
ws.jacobian_grid(prob, U, G.device_data)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ws.jacobian_grid(prob, U, G.device_data)
e1.record()
torch.cuda.synchronize()
t_jac = e0.elapsed_time(e1) / reps / 1e3
R = D.empty(prob.n_dofs)
ws.residual(prob, U, R)
e0.record()
for _ in range(reps):
    ws.residual(prob, U, R)
e1.record()
torch.cuda.synchronize()
t_res = e0.elapsed_time(e1) / reps / 1e3
x = D.to_device(np.random.default_rng(0).standard_normal(prob.n_dofs))
np.save(out, D.to_host(G.matvec(x)))
print(json.dumps({"jacobian_s": t_jac, "residual_s": t_res, "n_cells": prob.mesh.n_cells}))
'''

VARIANTS = {"v2": {"B200FEM_TANGENT": "v2"}, "v1": {"B200FEM_TANGENT": "v1"}}


def main():
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 136
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    import numpy as np

    res, ys = {}, {}
    with tempfile.TemporaryDirectory() as d:
        for name, extra in VARIANTS.items():
            env = dict(os.environ, ROOT=ROOT, **extra)
            f = os.path.join(d, f"{name}.npy")
            p = subprocess.run([sys.executable, "-c", CHILD, str(n), str(reps), f], env=env, capture_output=True,
                               text=True, timeout=900)
            if p.returncode:
                print(name, "FAILED", p.stderr[-3000:], file=sys.stderr)
                continue
            res[name] = json.loads(p.stdout.strip().splitlines()[-1])
            ys[name] = np.load(f)
    ref = ys.get("v1")
    for name, r in res.items():
        nc = r["n_cells"]
        r["jacobian_ms"] = r["jacobian_s"] * 1e3
        r["mcells_s"] = nc / r["jacobian_s"] / 1e6
        r["tflops_at_33k"] = 33e3 * nc / r["jacobian_s"] / 1e12
        r["frac_at_33k"] = r["tflops_at_33k"] / 34.23
        r["tflops_at_25.8k"] = 25824 * nc / r["jacobian_s"] / 1e12
        if ref is not None:
            r["rel_diff_Gx_vs_v1"] = float(np.linalg.norm(ys[name] - ref) / np.linalg.norm(ref))
        print(json.dumps({"variant": name, "n": n, **r}), flush=True)


if __name__ == "__main__":
    main()
