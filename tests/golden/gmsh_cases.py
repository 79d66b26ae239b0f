"""Unstructured HEX8 test meshes written as Gmsh MSH v2.2 text (neutral: no package imports).

``ogrid_cylinder(m, r, nz)``: a cylinder (radius 1, height 2) meshed as an O-grid -- an m x m
core square plus four ring blocks of m x r quads -- extruded in nz layers.  The four core
corners are shared by 3 quads per layer (6 hexes per node instead of 8), so the node
coupling is not a lattice stencil; node ids are shuffled (seeded) the way a mesher
numbers them, and the file carries the point / line / quad boundary entities and one
orphan node that the importer must drop (reference mesh.py:216-285).
"""

import numpy as np


def _ogrid_2d(m, r, a=0.45, R=1.0):
    """2-D quads (counter-clockwise) of the O-grid; returns (points (P,2), quads (Q,4))."""
    key = {}
    pts = []

    def node(x, y):
        k = (round(x, 12), round(y, 12))
        if k not in key:
            key[k] = len(pts)
            pts.append((x, y))
        return key[k]

    quads = []

    def block(P):  # P(t, u) -> (x, y) on the (nt+1) x (nu+1) grid
        nt, nu = P.shape[0] - 1, P.shape[1] - 1
        ids = [[node(*P[t, u]) for u in range(nu + 1)] for t in range(nt + 1)]
        for t in range(nt):
            for u in range(nu):
                q = [ids[t][u], ids[t + 1][u], ids[t + 1][u + 1], ids[t][u + 1]]
                xy = np.array([pts[i] for i in q])
                area = 0.5 * np.sum(xy[:, 0] * np.roll(xy[:, 1], -1) - np.roll(xy[:, 0], -1) * xy[:, 1])
                quads.append(q if area > 0 else q[::-1])

    s = np.linspace(-a, a, m + 1)
    core = np.stack(np.meshgrid(s, s, indexing="ij"), axis=-1)  # (i, j) -> (x, y)
    block(core)
    for side in range(4):
        th = np.linspace(-np.pi / 4, np.pi / 4, m + 1)
        inner = np.stack([np.full(m + 1, a), np.linspace(-a, a, m + 1)], axis=-1)
        outer = R * np.stack([np.cos(th), np.sin(th)], axis=-1)
        u = np.linspace(0.0, 1.0, r + 1)
        P = (1 - u)[None, :, None] * inner[:, None, :] + u[None, :, None] * outer[:, None, :]
        c, s_ = np.cos(side * np.pi / 2), np.sin(side * np.pi / 2)
        rot = np.array([[c, -s_], [s_, c]])
        block(P @ rot.T)
    return np.array(pts), np.array(quads, dtype=np.int64)


def ogrid_cylinder(m=2, r=2, nz=3, H=2.0, seed=7):
    """(text, info): MSH v2.2 text of the extruded O-grid, and the geometric facts."""
    p2, q2 = _ogrid_2d(m, r)
    P = p2.shape[0]
    z = np.linspace(0.0, H, nz + 1)
    nodes = np.concatenate([np.column_stack([p2, np.full(P, zk)]) for zk in z])
    hexes = np.concatenate([np.column_stack([q2 + k * P, q2 + (k + 1) * P]) for k in range(nz)])
    rng = np.random.default_rng(seed)
    perm = rng.permutation(nodes.shape[0])          # file row f holds node perm[f]
    gid = np.empty(nodes.shape[0], dtype=np.int64)  # node -> gmsh id
    gid[perm] = np.arange(nodes.shape[0]) + 1
    orphan = nodes.shape[0] + 1
    lines = ["$MeshFormat", "2.2 0 8", "$EndMeshFormat", "$Nodes", str(nodes.shape[0] + 1)]
    for f in range(nodes.shape[0]):
        x, y, zz = nodes[perm[f]]
        lines.append(f"{f + 1} {float(x)!r} {float(y)!r} {float(zz)!r}")
    lines.append(f"{orphan} 5.0 5.0 5.0")
    lines.append("$EndNodes")
    elems = []
    elems.append(f"15 2 0 1 {gid[0]}")                                     # a point entity
    elems.append(f"1 2 0 2 {gid[0]} {gid[1]}")                             # a line entity
    for q in q2[:3]:                                                         # bottom quads
        elems.append("3 2 0 3 " + " ".join(str(gid[v]) for v in q))
    for h in hexes:
        elems.append("5 2 0 1 " + " ".join(str(gid[v]) for v in h))
    lines.append("$Elements")
    lines.append(str(len(elems)))
    lines += [f"{i + 1} {e}" for i, e in enumerate(elems)]
    lines.append("$EndElements")
    return "\n".join(lines) + "\n", {"n_hex": hexes.shape[0], "n_nodes": nodes.shape[0], "H": H}


ALU = dict(E=70e3, nu=0.3, sigma_yield=250.0)
# neutral case table: O-grid args, law, Dirichlet (plane z = value, components, value), top traction
GMSH_CASES = {
    "gmsh_le": dict(grid=(2, 2, 3), law="le", clamp=(0.0, (0, 1, 2), 0.0), top_traction=(0.1, 0.05, -1.0), seed=1),
    "gmsh_nh": dict(grid=(3, 2, 4), law="nh", clamp=(0.0, (0, 1, 2), 0.0), top_disp=(2, 0.02), seed=2),
    "gmsh_poisson": dict(grid=(2, 2, 3), law="poisson", clamp=(0.0, (0,), 0.0), top_disp=(0, 1.0), source=1.0,
                         seed=3),
}


def write_case_mesh(name, directory):
    import os
    text, _ = ogrid_cylinder(*GMSH_CASES[name]["grid"])
    path = os.path.join(directory, f"{name}.msh")
    with open(path, "w") as fh:
        fh.write(text)
    return path


def build_gmsh(pk, name, path):
    """The case built with package `pk` (gradfem or paper_2212_00964_b200): (mesh, problem, U_test)."""
    c = GMSH_CASES[name]
    mesh = pk.import_mesh(path)
    H = float(mesh.nodes[:, 2].max())
    z0, comps, v0 = c["clamp"]
    const = lambda v: (lambda p, v=v: np.full(np.asarray(p).shape[:-1], v) if np.ndim(p) > 1 else v)  # noqa: E731
    specs = [pk.DirichletSpec(pk.BoundaryLocator.plane(2, z0), k, const(v0)) for k in comps]
    if "top_disp" in c:
        k, v = c["top_disp"]
        specs.append(pk.DirichletSpec(pk.BoundaryLocator.plane(2, H), k, const(v)))
    neu = []
    if "top_traction" in c:
        t = np.array(c["top_traction"])
        neu.append(pk.NeumannSpec(pk.boundary_facets(mesh, pk.BoundaryLocator.plane(2, H)),
                                  lambda p, t=t: np.broadcast_to(t, np.asarray(p).shape[:-1] + (3,)).copy()))
    if c["law"] == "poisson":
        s = c["source"]
        prob = pk.PoissonProblem(mesh, 1.0, specs, neu, source=lambda p, s=s: np.full(np.asarray(p).shape[:-1] + (1,), s))
    else:
        cls = pk.LinearElasticityProblem if c["law"] == "le" else pk.NeoHookeanProblem
        prob = cls(mesh, pk.ElasticConstants(**ALU), specs, neu)
    U = 1e-3 * np.random.default_rng(c["seed"]).standard_normal(prob.n_dofs)
    return mesh, prob, U
