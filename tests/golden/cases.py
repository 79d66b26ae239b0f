"""Neutral definitions of the parity cases shared by three consumers:

* tests/golden/make_golden.py builds them with the reference package (build container only),
* the oracle tests build them with oracle/ (numpy),
* the GPU parity tests build them with paper_2212_00964_b200.

Locators: ("plane", axis, value) with the reference default tolerance 1e-5 (mesh.py:32, 95-100),
("onbox", Lx, Ly, Lz) = all six faces with tol 1e-9 (reference tests/conftest.py:9-18),
("everywhere",).  Dirichlet values: a float, or ("affine", A) meaning u_c = (A x)_c.
"""

import numpy as np

ALU = dict(E=70e3, nu=0.3, sigma_yield=250.0)  # reference tests/conftest.py:35-37
PATCH_A = 1e-3 * np.array([[1.0, 0.4, 0.2], [0.0, -0.5, 0.3], [0.1, 0.0, 0.7]])


def _fixed(loc, vec=3):
    return [(loc, c, 0.0) for c in range(vec)]


CASES = {
    # BASELINE config 1: LE cantilever 20x4x4, clamped x=0, traction (0,0,-1) MPa on x=20.
    "c1": dict(dims=(20, 4, 4), L=(20.0, 4.0, 4.0), law=("le", ALU),
               dirichlet=_fixed(("plane", 0, 0.0)),
               neumann=[(("plane", 0, 20.0), (0.0, 0.0, -1.0))],
               reaction=(("plane", 0, 0.0), 2), seed=11, u_scale=1e-3),
    # Neo-Hookean tensile block, 2 % stretch on the top face, laterally free.
    "nh_block": dict(dims=(4, 3, 2), L=(1.0, 0.75, 0.5), law=("nh", ALU),
                     dirichlet=_fixed(("plane", 2, 0.0)) + [(("plane", 2, 0.5), 2, 0.01)],
                     seed=12, u_scale=2e-3),
    # Acceptance criterion 6 (reference tests/test_acceptance.py:219-230).
    "nh_crit6": dict(dims=(2, 2, 2), L=(1.0, 1.0, 1.0), law=("nh", ALU),
                     dirichlet=_fixed(("plane", 2, 0.0)) + [(("plane", 2, 1.0), 2, 0.02)],
                     newton=dict(rel_tol=1e-9, abs_tol=1e-10), seed=13, u_scale=1e-3),
    # J2 plasticity, load beyond yield and back.
    "j2_block": dict(dims=(3, 3, 3), L=(1.0, 1.0, 1.0), law=("j2", ALU),
                     dirichlet=_fixed(("plane", 2, 0.0)) + [(("plane", 2, 1.0), 2, 0.012)],
                     schedule=("ramp_and_back", 4), reaction=(("plane", 2, 1.0), 2),
                     seed=14, u_scale=1e-3),
    # J2 8^3 ramp_and_back(10) to u_z = 0.012.
    "j2_8": dict(dims=(8, 8, 8), L=(1.0, 1.0, 1.0), law=("j2", ALU),
                 dirichlet=_fixed(("plane", 2, 0.0)) + [(("plane", 2, 1.0), 2, 0.012)],
                 schedule=("ramp_and_back", 10), reaction=(("plane", 2, 1.0), 2),
                 seed=15, u_scale=1e-3),
    # Poisson with a constant source, zero on all faces (config 2 in miniature).
    "poisson": dict(dims=(5, 4, 3), L=(1.0, 1.0, 1.0), law=("poisson", dict(alpha=1.0)),
                    dirichlet=[(("onbox", 1.0, 1.0, 1.0), 0, 0.0)], source=1.0,
                    seed=16, u_scale=1e-2),
    # Poisson with a nodal design source (problems.py:100-130).
    "poisson_design": dict(dims=(3, 3, 3), L=(1.0, 1.0, 1.0), law=("poisson", dict(alpha=0.7)),
                           dirichlet=[(("onbox", 1.0, 1.0, 1.0), 0, 0.0)], design_source=True,
                           seed=17, u_scale=1e-2),
    # SIMP linear elasticity (config 5 in miniature).
    "simp": dict(dims=(6, 3, 2), L=(3.0, 1.5, 1.0), law=("simp_le", ALU),
                 dirichlet=_fixed(("plane", 0, 0.0)),
                 neumann=[(("plane", 0, 3.0), (0.0, 0.0, -1.0))],
                 theta=(0.3, 0.9), seed=18, u_scale=1e-3),
    # SIMP over a neo-Hookean base.
    "simp_nh": dict(dims=(4, 2, 2), L=(2.0, 1.0, 1.0), law=("simp_nh", ALU),
                    dirichlet=_fixed(("plane", 0, 0.0)),
                    neumann=[(("plane", 0, 2.0), (0.0, 0.0, -1.0))],
                    theta=(0.3, 0.9), seed=19, u_scale=1e-3),
    # Affine patch test with an LE body force (assembly.py:121-128).
    "le_body": dict(dims=(3, 2, 2), L=(1.0, 1.0, 1.0), law=("le", ALU),
                    dirichlet=[(("onbox", 1.0, 1.0, 1.0), c, ("affine", PATCH_A)) for c in range(3)],
                    body=(0.5, -1.0, 2.0), seed=20, u_scale=1e-3),
}


def node_mask(loc, nodes):
    """Boolean selection of mesh nodes by a neutral locator."""
    p = np.asarray(nodes)
    if loc[0] == "plane":
        _, axis, value = loc[:3]
        tol = loc[3] if len(loc) > 3 else 1e-5
        return np.abs(p[:, axis] - value) <= tol
    if loc[0] == "onbox":
        _, Lx, Ly, Lz = loc
        t = 1e-9
        return ((np.abs(p[:, 0]) < t) | (np.abs(p[:, 0] - Lx) < t) | (np.abs(p[:, 1]) < t)
                | (np.abs(p[:, 1] - Ly) < t) | (np.abs(p[:, 2]) < t) | (np.abs(p[:, 2] - Lz) < t))
    if loc[0] == "everywhere":
        return np.ones(p.shape[0], dtype=bool)
    raise ValueError(loc)


def value_fn(val, comp):
    """Vectorised value callable for a neutral Dirichlet value."""
    if isinstance(val, tuple) and val[0] == "affine":
        A = np.asarray(val[1], dtype=np.float64)
        return lambda p: (np.atleast_2d(p) @ A.T)[..., comp]
    v = float(val)
    return lambda p: np.full(np.asarray(p).shape[:-1], v) if np.ndim(p) > 1 else v


def traction_fn(t):
    t = np.asarray(t, dtype=np.float64)
    return lambda p: np.broadcast_to(t, np.asarray(p).shape[:-1] + (t.size,)).copy()


def schedule_factors(sched):
    kind, n = sched
    up = [(k + 1) / n for k in range(n)]
    if kind == "ramp":
        return up
    return up + [(n - 1 - k) / n for k in range(n)]


def test_vectors(case, n_nodes, n_cells, vec):
    """Seeded U for R/K evaluation and the SIMP/design theta (np.random.default_rng(seed))."""
    rng = np.random.default_rng(case["seed"])
    U = case["u_scale"] * rng.standard_normal(n_nodes * vec)
    theta = None
    if "theta" in case:
        lo, hi = case["theta"]
        theta = rng.uniform(lo, hi, n_cells)
    if case.get("design_source"):
        theta = rng.standard_normal(n_nodes)
    return U, theta
