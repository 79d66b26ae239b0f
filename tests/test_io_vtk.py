"""VTK / CSV output.  The ASCII writer is compared BYTE FOR BYTE with the
reference writer's output, regenerated as a committed fixture (tests/golden/vtk_ref.npz by
tests/golden/make_golden_io.py) -- the reference itself is not needed at test time."""

import numpy as np
import pytest

import paper_2212_00964_b200 as fem
from conftest import load_golden
from io_cases import fields
from paper_2212_00964_b200.io_vtk import VtkWriteError, read_vtk_points, write_vtk


def test_ascii_vtk_byte_identical_to_reference(tmp_path):
    g = load_golden("vtk_ref")
    mesh = fem.generate_box_mesh(5, 4, 3, 2.0, 1.5, 1.0)
    pd, cd = fields(mesh)
    path = tmp_path / "a.vtk"
    write_vtk(mesh, pd, cd, path=path)
    assert path.read_bytes() == g["with_fields"].tobytes()
    write_vtk(mesh, path=path)
    assert path.read_bytes() == g["geometry"].tobytes()


def test_binary_vtk_roundtrip(tmp_path):
    mesh = fem.generate_box_mesh(4, 3, 2, 1.0, 1.0, 1.0)
    pd, cd = fields(mesh)
    path = tmp_path / "b.vtk"
    write_vtk(mesh, pd, cd, path=path, binary=True)
    assert np.array_equal(read_vtk_points(path), mesh.nodes)
    data = path.read_bytes()
    assert b"\nBINARY\n" in data[:200]
    off = data.index(b"CELLS")
    eol = data.index(b"\n", off)
    cells = np.frombuffer(data, dtype=">i4", count=9 * mesh.n_cells, offset=eol + 1).reshape(-1, 9)
    assert (cells[:, 0] == 8).all() and np.array_equal(cells[:, 1:], mesh.cells)


def test_write_vtk_geometry_roundtrip(tmp_path):  # reference tests/test_io_cli.py:150-156
    mesh = fem.generate_box_mesh(2, 2, 2, 1.0, 2.0, 3.0)
    path = tmp_path / "mesh.vtk"
    write_vtk(mesh, path=path)
    assert np.array_equal(read_vtk_points(path), mesh.nodes)


def test_write_vtk_rejects_bad_field_lengths(tmp_path):  # reference tests/test_io_cli.py:159-164
    mesh = fem.generate_box_mesh(2, 2, 2, 1.0, 1.0, 1.0)
    with pytest.raises(VtkWriteError, match="cell field"):
        write_vtk(mesh, cell_data={"x": np.zeros(5)}, path=tmp_path / "x.vtk")
    with pytest.raises(VtkWriteError, match="point field"):
        write_vtk(mesh, point_data={"u": np.zeros(3)}, path=tmp_path / "y.vtk")


def test_load_history_csv_matches_reference_format(tmp_path):
    g = load_golden("vtk_ref")
    h = fem.LoadHistory()
    for k, s in enumerate([0.5, 1.0]):
        h.steps.append(fem.StepRecord(step=k + 1, scale=s, U=np.zeros(3), newton_iterations=k + 2,
                                      residual_norm=10.0 ** (-9 - k), residual_history=[1.0 / 3.0, 1e-5 * s],
                                      reaction=None if k == 0 else 2.0 / 3.0,
                                      avg_stress=np.arange(9.0).reshape(3, 3) * s))
    h.write_csv(tmp_path / "h.csv")
    h.write_newton_csv(tmp_path / "n.csv")
    assert (tmp_path / "h.csv").read_bytes() == g["history_csv"].tobytes()
    assert (tmp_path / "n.csv").read_bytes() == g["newton_csv"].tobytes()
