"""BASELINE configs C2-C5 at the sizes BASELINE.json / SURVEY.md section 8(d) state, built with
either API (the reference package `gradfem`, or paper_2212_00964_b200: the same Problem API).

Shared by tests/golden/make_golden_fullsize.py (reference side, build container only) and
tests/test_gpu_fullsize_ref.py (device side).

* C2: generate_box_mesh(100,100,100, 1,1,1), PoissonProblem(alpha=1), u=0 on all six faces
  (on-box predicate, tol 1e-9, reference tests/conftest.py:9-18), source 1.
* C3: generate_box_mesh(136,136,136, 1,1,1), NeoHookeanProblem, z=0 clamped, u_z = 0.02 on z=1.
* C4: generate_box_mesh(40,40,40, 1,1,1), J2PlasticityProblem, z=0 clamped, u_z = 0.012 on z=1,
  LoadSchedule.ramp_and_back(10), reaction on z=1 (reference solvers.py:305-349).
* C5: generate_box_mesh(176,88,22, 8,4,1), SimpElasticityProblem(LinearElastic), p=3,
  x=0 clamped, traction (0,0,-1) on x=8; design k: theta ~ U(0.3, 0.9), default_rng(k)
  (reference inverse.py:402-405: set_theta, warm-started newton_solve per design).
"""

import numpy as np

ALU = dict(E=70e3, nu=0.3, sigma_yield=250.0)  # reference tests/conftest.py:35-37
C5_DIMS = (176, 88, 22, 8.0, 4.0, 1.0)


def _const(s):
    return lambda p: np.full(np.asarray(p).shape[:-1], s) if np.ndim(p) > 1 else s


def _onbox(p):
    return (np.abs(np.asarray(p) - 0.5) >= 0.5 - 1e-9).any(axis=-1)


def _traction(t):
    return lambda p: np.broadcast_to(np.asarray(t, float), np.asarray(p).shape[:-1] + (3,)).copy()


def c2(pk, n=100):
    mesh = pk.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    specs = [pk.DirichletSpec(pk.BoundaryLocator(_onbox), 0, _const(0.0))]
    return pk.PoissonProblem(mesh, 1.0, specs, source=lambda p: np.ones(np.asarray(p).shape[:-1] + (1,)))


def _tensile(pk, n, stretch, cls):
    mesh = pk.generate_box_mesh(n, n, n, 1.0, 1.0, 1.0)
    bot, top = pk.BoundaryLocator.plane(2, 0.0), pk.BoundaryLocator.plane(2, 1.0)
    specs = [pk.DirichletSpec(bot, c, _const(0.0)) for c in range(3)] + [pk.DirichletSpec(top, 2, _const(stretch))]
    return getattr(pk, cls)(mesh, pk.ElasticConstants(**ALU), specs)


def c3(pk, n=136):
    return _tensile(pk, n, 0.02, "NeoHookeanProblem")


def c4(pk, n=40):
    return _tensile(pk, n, 0.012, "J2PlasticityProblem")


def c4_top(pk):
    return pk.BoundaryLocator.plane(2, 1.0)


def c5(pk):
    mesh = pk.generate_box_mesh(*C5_DIMS)
    specs = [pk.DirichletSpec(pk.BoundaryLocator.plane(0, 0.0), c, _const(0.0)) for c in range(3)]
    neu = [pk.NeumannSpec(pk.boundary_facets(mesh, pk.BoundaryLocator.plane(0, 8.0)), _traction((0.0, 0.0, -1.0)))]
    return pk.SimpElasticityProblem(mesh, pk.LinearElastic(pk.ElasticConstants(**ALU)), specs, neu, penalty=3.0)


def c5_theta(k, n_cells):
    return np.random.default_rng(k).uniform(0.3, 0.9, n_cells)


MAP_FIELDS = (("indptr", np.int32), ("indices", np.int32), ("dest", np.int64), ("diag_slots", np.int64),
              ("dir_dofs", np.int64), ("dir_row_slots", np.int64))


def map_hashes(ws):
    """SHA-256 of each integer map of a workspace, in a canonical dtype (little-endian, C order)."""
    import hashlib

    out = {}
    for name, dt in MAP_FIELDS:
        a = np.ascontiguousarray(np.asarray(getattr(ws, name)).astype(dt, copy=False))
        out[name] = {"sha256": hashlib.sha256(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest(),
                     "shape": list(a.shape), "dtype": np.dtype(dt).name}
    return out
