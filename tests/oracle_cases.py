"""Build the neutral cases of tests/golden/cases.py on the CPU oracle (test infrastructure)."""

import numpy as np

import oracle as orc
from cases import CASES, node_mask, test_vectors, traction_fn, value_fn


def build_oracle(name, case=None):
    case = case or CASES[name]
    nodes, cells = orc.box_mesh(*case["dims"], *case["L"])
    kind, mat = case["law"]
    if kind == "poisson":
        law = orc.Law("poisson", alpha=mat["alpha"])
    else:
        base = kind.replace("simp_", "")
        law = orc.Law(base, E=mat["E"], nu=mat["nu"], sigma_yield=mat.get("sigma_yield", np.inf))
    vec = law.vec
    specs = [(node_mask(loc, nodes), comp, value_fn(val, comp)) for loc, comp, val in case["dirichlet"]]
    dd, dv = orc.dirichlet_table(nodes, vec, specs)
    fn = np.zeros(nodes.shape[0] * vec)
    for loc, t in case.get("neumann", []):
        facets = orc.boundary_facets(nodes, cells, node_mask(loc, nodes))
        fn += orc.neumann_load(nodes, cells, vec, facets, traction_fn(t))
    body = None
    if "body" in case:
        body = traction_fn(case["body"])
    if "source" in case:
        s = case["source"]
        body = lambda p, s=s: np.full(np.asarray(p).shape[:-1] + (1,), s)  # noqa: E731
    fb = orc.body_load(nodes, cells, vec, body)
    U, theta = test_vectors(case, nodes.shape[0], cells.shape[0], vec)
    prob = orc.OracleProblem(nodes, cells, law, dd, dv, fn, fb,
                             jacobian_constant=kind in ("le", "poisson"))
    if kind.startswith("simp_"):
        prob.simp_theta = np.clip(theta, 1e-3, 1.0)
        prob.simp_penalty = 3.0
    if case.get("design_source"):
        prob.source_theta = theta
    return prob, U
