"""Neutral output-writer fixtures shared by make_golden_io.py and tests/test_io_vtk.py."""

import numpy as np


def fields(mesh):
    """Point / cell fields with awkward values: -0.0, subnormals, 1e+-300 magnitudes, 1/3."""
    rng = np.random.default_rng(5)
    u = rng.standard_normal((mesh.n_nodes, 3)) * np.logspace(-300, 300, mesh.n_nodes)[:, None]
    u[0] = [-0.0, 1e-320, 1.0 / 3.0]
    p = rng.standard_normal(mesh.n_nodes)
    c = rng.uniform(0.0, 1.0, mesh.n_cells)
    return {"displacement": u, "phi": p}, {"density": c}
