"""Generate tests/golden/vtk_ref.npz with the REFERENCE writers (build container only):
the reference's write_vtk output for a box mesh with point/cell fields and without, and its
LoadHistory CSV files, as raw bytes.

    python tests/golden/make_golden_io.py
"""

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import gradfem as gf  # noqa: E402
from gradfem.io_vtk import write_vtk  # noqa: E402
from gradfem.solvers import LoadHistory, StepRecord  # noqa: E402

from io_cases import fields  # noqa: E402  (the same field values as the test)


def raw(path):
    with open(path, "rb") as fh:
        return np.frombuffer(fh.read(), dtype=np.uint8)


if __name__ == "__main__":
    out = {}
    with tempfile.TemporaryDirectory() as d:
        mesh = gf.generate_box_mesh(5, 4, 3, 2.0, 1.5, 1.0)
        pd, cd = fields(mesh)
        write_vtk(mesh, pd, cd, path=os.path.join(d, "a.vtk"))
        out["with_fields"] = raw(os.path.join(d, "a.vtk"))
        write_vtk(mesh, path=os.path.join(d, "g.vtk"))
        out["geometry"] = raw(os.path.join(d, "g.vtk"))
        h = LoadHistory()
        for k, s in enumerate([0.5, 1.0]):
            h.steps.append(StepRecord(step=k + 1, scale=s, U=np.zeros(3), newton_iterations=k + 2,
                                      residual_norm=10.0 ** (-9 - k), residual_history=[1.0 / 3.0, 1e-5 * s],
                                      reaction=None if k == 0 else 2.0 / 3.0,
                                      avg_stress=np.arange(9.0).reshape(3, 3) * s))
        h.write_csv(os.path.join(d, "h.csv"))
        h.write_newton_csv(os.path.join(d, "n.csv"))
        out["history_csv"] = raw(os.path.join(d, "h.csv"))
        out["newton_csv"] = raw(os.path.join(d, "n.csv"))
    np.savez_compressed(os.path.join(HERE, "vtk_ref.npz"), **out)
    print({k: v.size for k, v in out.items()})
