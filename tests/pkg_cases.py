"""Build the neutral cases of tests/golden/cases.py with paper_2212_00964_b200."""

import numpy as np

import paper_2212_00964_b200 as fem
from cases import CASES, node_mask, test_vectors, traction_fn, value_fn


def locator(loc):
    return fem.BoundaryLocator(lambda p, loc=loc: node_mask(loc, np.atleast_2d(p)) if np.ndim(p) > 1
                               else bool(node_mask(loc, np.atleast_2d(p))[0]))


def build(name, case=None):
    case = case or CASES[name]
    mesh = fem.generate_box_mesh(*case["dims"], *case["L"])
    kind, mat = case["law"]
    c = fem.ElasticConstants(**mat) if kind != "poisson" else None
    specs = [fem.DirichletSpec(locator(loc), comp, value_fn(val, comp)) for loc, comp, val in case["dirichlet"]]
    neu = [fem.NeumannSpec(fem.boundary_facets(mesh, locator(loc)), traction_fn(t))
           for loc, t in case.get("neumann", [])]
    body = traction_fn(case["body"]) if "body" in case else None
    if kind == "poisson":
        src = None
        if "source" in case:
            s = case["source"]
            src = lambda p, s=s: np.full(np.asarray(p).shape[:-1] + (1,), s)  # noqa: E731
        prob = fem.PoissonProblem(mesh, mat["alpha"], specs, neu, source=src,
                                  design_source=bool(case.get("design_source")))
    elif kind == "le":
        prob = fem.LinearElasticityProblem(mesh, c, specs, neu, body)
    elif kind == "nh":
        prob = fem.NeoHookeanProblem(mesh, c, specs, neu, body)
    elif kind == "j2":
        prob = fem.J2PlasticityProblem(mesh, c, specs, neu, body)
    elif kind == "simp_le":
        prob = fem.SimpElasticityProblem(mesh, fem.LinearElastic(c), specs, neu, penalty=3.0)
    elif kind == "simp_nh":
        prob = fem.SimpElasticityProblem(mesh, fem.NeoHookean(c), specs, neu, penalty=3.0)
    else:
        raise ValueError(kind)
    U, theta = test_vectors(case, mesh.n_nodes, mesh.n_cells, prob.vec)
    if theta is not None:
        prob.set_theta(theta)
    return mesh, prob, U
