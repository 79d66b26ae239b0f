#!/bin/bash
# A/B of the z-slab pipelined lattice tangent (B200FEM_TANGENT_PIPE = slabs; 1 = off)
cd "$(dirname "$0")/.."
for P in 1 4 8 16; do
  B200FEM_TANGENT_PIPE=$P python - <<'PY'
import os, sys, json
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "tests", "golden")]
import numpy as np, torch
import fullsize_cases as fc, paper_2212_00964_b200 as fem
from paper_2212_00964_b200 import _device as D
from paper_2212_00964_b200.sparse import GridOperator
prob = fc.c3(fem, 136); ws = fem.workspace(prob)
U = D.to_device(1e-3 * np.random.default_rng(1).standard_normal(prob.n_dofs))
G = GridOperator(ws); ws.jacobian_grid(prob, U, G.device_data); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): ws.jacobian_grid(prob, U, G.device_data)
e1.record(); torch.cuda.synchronize()
x = D.to_device(np.random.default_rng(0).standard_normal(prob.n_dofs))
y = G.matvec(x)
print(json.dumps({"pipe": os.environ["B200FEM_TANGENT_PIPE"], "jacobian_ms": e0.elapsed_time(e1) / 5,
                  "Gx_norm": float(torch.linalg.vector_norm(y)), "Gx_sum": float(y.sum())}))
PY
done
