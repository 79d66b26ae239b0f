"""Legacy VTK output of the mesh and solution fields (reference
io_vtk.py:1-94).

``write_vtk(..., binary=False)`` writes the reference's ASCII file byte for byte: the same
header, 17-significant-digit floats (io_vtk.py:18-19), cell type 12, the same field
validation and error messages.  The text of the large blocks (POINTS, CELLS, fields) is
produced by the library's multi-threaded host formatter (csrc/io.cu) instead of one Python
f-string per value: at config 3 (2.57M points, 2.52M cells) that is the difference between
minutes and seconds per VTK step.  ``binary=True`` writes the legacy BINARY variant
(big-endian float64 / int32 blocks, same header and fields) for steps that only need to be
read back by VTK/ParaView.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .mesh import Mesh

_VTK_HEX = 12


class VtkWriteError(ValueError):
    pass


def _fmt(x) -> str:
    return f"{x:.17g}"


def _rows_text(arr: np.ndarray, prefix: int = -1) -> bytes:
    """Rows of a 2-D array as lines of space-separated values (%.17g / integers)."""
    lib = _lib.host_lib()
    if arr.dtype.kind == "f":
        a = np.ascontiguousarray(arr, dtype=np.float64)
        cap = a.shape[0] * (a.shape[1] * 25 + 24) + 1
        buf = C.create_string_buffer(cap)
        n = lib.b200fem_format_f64_rows(a.ctypes.data, a.shape[0], a.shape[1], buf, cap)
    else:
        a = np.ascontiguousarray(arr, dtype=np.int64)
        cap = a.shape[0] * (a.shape[1] * 25 + 24) + 1
        buf = C.create_string_buffer(cap)
        n = lib.b200fem_format_i64_rows(a.ctypes.data, a.shape[0], a.shape[1], prefix, buf, cap)
    if n < 0:
        raise RuntimeError("output formatter buffer too small")
    return buf.raw[:n]


def _check_fields(mesh: Mesh, point_data: dict, cell_data: dict) -> None:
    for name, arr in point_data.items():
        arr = np.asarray(arr)
        if arr.shape not in ((mesh.n_nodes,), (mesh.n_nodes, 3)):
            raise VtkWriteError(
                f"point field {name!r} has shape {arr.shape}; expected "
                f"({mesh.n_nodes},) or ({mesh.n_nodes}, 3)"
            )
    for name, arr in cell_data.items():
        arr = np.asarray(arr)
        if arr.shape != (mesh.n_cells,):
            raise VtkWriteError(f"cell field {name!r} has shape {arr.shape}; expected ({mesh.n_cells},)")


def write_vtk(mesh: Mesh, point_data=None, cell_data=None, path=None, binary: bool = False) -> None:
    """Write the mesh plus named point / cell fields (io_vtk.py:22-82).

    point_data values may be (N,) scalars or (N, 3) vectors; cell_data values are (N_e,)
    scalars; CUDA tensors are accepted and copied to the host.  Field length mismatches are
    rejected (VtkWriteError) before anything is written."""
    def host(a):
        if hasattr(a, "detach"):
            a = a.detach().cpu().numpy()
        return np.asarray(a)

    point_data = {k: host(v) for k, v in dict(point_data or {}).items()}
    cell_data = {k: host(v) for k, v in dict(cell_data or {}).items()}
    _check_fields(mesh, point_data, cell_data)
    chunks = []
    head = ["# vtk DataFile Version 3.0", "gradfem output", "BINARY" if binary else "ASCII",
            "DATASET UNSTRUCTURED_GRID", f"POINTS {mesh.n_nodes} double"]
    chunks.append(("\n".join(head) + "\n").encode())

    def block(arr2d, dtype_be, prefix=-1):
        if binary:
            a = np.asarray(arr2d)
            if prefix >= 0:
                a = np.concatenate([np.full((a.shape[0], 1), prefix, dtype=a.dtype), a], axis=1)
            chunks.append(np.ascontiguousarray(a, dtype=dtype_be).tobytes() + b"\n")
        else:
            chunks.append(_rows_text(arr2d, prefix))

    block(mesh.nodes, ">f8")
    chunks.append(f"CELLS {mesh.n_cells} {mesh.n_cells * 9}\n".encode())
    block(mesh.cells, ">i4", prefix=8)
    chunks.append(f"CELL_TYPES {mesh.n_cells}\n".encode())
    if binary:
        chunks.append(np.full(mesh.n_cells, _VTK_HEX, dtype=">i4").tobytes() + b"\n")
    else:
        chunks.append(("12\n" * mesh.n_cells).encode())
    if point_data:
        chunks.append(f"POINT_DATA {mesh.n_nodes}\n".encode())
        for name, arr in point_data.items():
            arr = np.asarray(arr, dtype=np.float64)
            if arr.ndim == 1:
                chunks.append(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n".encode())
                block(arr[:, None], ">f8")
            else:
                chunks.append(f"VECTORS {name} double\n".encode())
                block(arr, ">f8")
    if cell_data:
        chunks.append(f"CELL_DATA {mesh.n_cells}\n".encode())
        for name, arr in cell_data.items():
            arr = np.asarray(arr, dtype=np.float64)
            chunks.append(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n".encode())
            block(arr[:, None], ">f8")
    try:
        with open(path, "wb") as fh:
            for c in chunks:
                fh.write(c)
    except OSError as err:
        raise IOError(f"cannot write VTK file {path}: {err}") from err


def read_vtk_points(path) -> np.ndarray:
    """Parse back the POINTS block of an ASCII or BINARY file (round-trip checks)."""
    with open(path, "rb") as fh:
        data = fh.read()
    head_end = data.find(b"POINTS")
    if head_end < 0:
        raise VtkWriteError(f"no POINTS block in {path}")
    binary = b"\nBINARY\n" in data[:head_end]
    eol = data.index(b"\n", head_end)
    n = int(data[head_end:eol].split()[1])
    if binary:
        return np.frombuffer(data, dtype=">f8", count=3 * n, offset=eol + 1).astype(np.float64).reshape(n, 3)
    vals = data[eol + 1:].split(b"\n", n)[:n]
    return np.array(b" ".join(vals).split(), dtype=np.float64).reshape(n, 3)
