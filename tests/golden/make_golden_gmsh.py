"""Generate tests/golden/gmsh_*.npz with the REFERENCE package on imported O-grid meshes
(unstructured HEX8).  Build container only:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_gmsh.py
"""

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem as gf  # noqa: E402
from gradfem.assembly import workspace  # noqa: E402

from gmsh_cases import GMSH_CASES, build_gmsh, write_case_mesh  # noqa: E402

TIGHT_NEWTON = dict(rel_tol=1e-10, abs_tol=1e-12)
TIGHT_LINEAR = dict(rel_tol=1e-11, abs_tol=1e-14)


def run(name, d):
    path = write_case_mesh(name, d)
    mesh, prob, U = build_gmsh(gf, name, path)
    ws = workspace(prob)
    out = dict(nodes=mesh.nodes, cells=mesh.cells.astype(np.int32), indptr=ws.indptr, indices=ws.indices,
               dest=ws.dest.astype(np.int32), diag_slots=ws.diag_slots.astype(np.int32), dir_dofs=ws.dir_dofs,
               dir_values=ws.dir_values, f_neumann=ws.f_neumann, U_test=U,
               R_test=gf.assemble_residual(prob, U), K_test=gf.assemble_jacobian(prob, U).data)
    _, prob2, _ = build_gmsh(gf, name, path)
    Ut, rep = gf.newton_solve(prob2, cfg=gf.NewtonConfig(**TIGHT_NEWTON), lin_cfg=gf.LinearSolveConfig(**TIGHT_LINEAR))
    out["U_tight"] = Ut
    out["norms_tight"] = np.array(rep.residual_norms)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: n_dofs={prob.n_dofs} nnz={ws.indices.size} newton_its={rep.n_iterations}")


if __name__ == "__main__":
    with tempfile.TemporaryDirectory() as d:
        for n in sys.argv[1:] or list(GMSH_CASES):
            run(n, d)
