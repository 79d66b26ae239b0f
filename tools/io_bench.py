"""Output-writer throughput: write_vtk ASCII / BINARY for a box mesh with a
displacement field, ours vs the reference writer (when /root/reference is importable).

    python tools/io_bench.py [--n 64] [--ref-n 32]
"""

import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200.io_vtk import write_vtk  # noqa: E402


def one(writer, mesh, d, name, **kw):
    U = np.random.default_rng(0).standard_normal((mesh.n_nodes, 3))
    path = os.path.join(d, name)
    t0 = time.perf_counter()
    writer(mesh, point_data={"displacement": U}, path=path, **kw)
    dt = time.perf_counter() - t0
    size = os.path.getsize(path)
    os.remove(path)
    return {"s": dt, "MB": size / 1e6, "MB_s": size / 1e6 / dt, "values": mesh.n_nodes * 6 + mesh.n_cells * 9}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--ref-n", type=int, default=32)
    a = ap.parse_args()
    out = {"threads": os.cpu_count()}
    with tempfile.TemporaryDirectory() as d:
        mesh = fem.generate_box_mesh(a.n, a.n, a.n, 1.0, 1.0, 1.0)
        out[f"ours_ascii_{a.n}"] = one(write_vtk, mesh, d, "a.vtk")
        out[f"ours_binary_{a.n}"] = one(write_vtk, mesh, d, "b.vtk", binary=True)
        try:
            sys.path.insert(0, "/root/reference/pkg/src")
            import gradfem as gf
            from gradfem.io_vtk import write_vtk as ref_write
            m2 = gf.generate_box_mesh(a.ref_n, a.ref_n, a.ref_n, 1.0, 1.0, 1.0)
            out[f"reference_ascii_{a.ref_n}"] = one(ref_write, m2, d, "r.vtk")
        except ImportError:
            out["reference"] = "not importable here"
    for k, v in out.items():
        if isinstance(v, dict):
            v["values_per_s"] = v["values"] / v["s"]
    print(json.dumps(out))
