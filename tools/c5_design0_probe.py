import sys, os, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2212_00964_b200 as fem
from paper_2212_00964_b200 import _device as D
ALU = fem.ElasticConstants(E=70e3, nu=0.3, sigma_yield=250.0)
mesh = fem.generate_box_mesh(176, 88, 22, 8.0, 4.0, 1.0)
x0 = fem.BoundaryLocator.plane(0, 0.0)
specs = [fem.DirichletSpec(x0, c, lambda p: 0.0) for c in range(3)]
neu = [fem.NeumannSpec(fem.boundary_facets(mesh, fem.BoundaryLocator.plane(0, 8.0)),
                       lambda p: np.broadcast_to([0.0, 0.0, -1.0], np.asarray(p).shape[:-1] + (3,)))]
out = {}
for op in ("grid", "csr"):
    prob = fem.SimpElasticityProblem(mesh, fem.LinearElastic(ALU), specs, neu, penalty=3.0)
    prob.set_theta(np.random.default_rng(0).uniform(0.3, 0.9, mesh.n_cells))
    t0 = time.perf_counter()
    U, rep = fem.newton_solve(prob, D.zeros(prob.n_dofs), lin_cfg=fem.LinearSolveConfig(operator=op))
    torch.cuda.synchronize()
    out[op] = dict(s=time.perf_counter() - t0, stats=[(s.iterations, s.matvecs, s.restarts, s.residual, s.tol) for s in rep.linear_stats])
print(json.dumps(out))
