"""The reference's low seam on the device (paper_2212_00964_b200.kernels, csrc/lowseam.cu):
bit-identical to the reference's numba csr_matvec / scatter_add (goldens from
make_golden_lowseam.py), plus ports of the reference's tests/test_kernels.py."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2212_00964_b200 import kernels

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return load_golden("lowseam")


@pytest.mark.parametrize("name", ["small", "empty_row", "large"])
def test_csr_matvec_bit_identical_to_reference(g, name):
    ip, ix, d, x = (g[f"{name}_{k}"] for k in ("indptr", "indices", "data", "x"))
    assert np.array_equal(kernels.csr_matvec(ip, ix, d, x), g[f"{name}_y"])
    import torch
    yd = kernels.csr_matvec(torch.tensor(ip, device="cuda"), torch.tensor(ix, device="cuda"),
                            torch.tensor(d, device="cuda"), torch.tensor(x, device="cuda"))
    assert yd.is_cuda and np.array_equal(yd.cpu().numpy(), g[f"{name}_y"])


@pytest.mark.parametrize("name", ["scatter_small", "scatter_large"])
def test_scatter_add_bit_identical_to_reference(g, name):
    v = g[f"{name}_v0"].copy()
    kernels.scatter_add(v, g[f"{name}_dest"], g[f"{name}_contribs"])  # host array, in place
    assert np.array_equal(v, g[f"{name}_v"])
    import torch
    vd = torch.tensor(g[f"{name}_v0"], device="cuda")
    ptr = vd.data_ptr()
    kernels.scatter_add(vd, torch.tensor(g[f"{name}_dest"], device="cuda"), g[f"{name}_contribs"])
    assert vd.data_ptr() == ptr and np.array_equal(vd.cpu().numpy(), g[f"{name}_v"])


def random_csr(rng, n=60, per_row=7):  # reference tests/test_kernels.py:8-15
    indptr = np.zeros(n + 1, dtype=np.int32)
    indices = []
    for i in range(n):
        cols = np.unique(np.append(rng.choice(n, per_row), i))
        indices.extend(np.sort(cols))
        indptr[i + 1] = len(indices)
    return indptr, np.array(indices, dtype=np.int32), rng.standard_normal(len(indices))


def test_matvec_matches_dense(rng):
    """test_kernels.py:18-25"""
    indptr, indices, data = random_csr(rng)
    n = indptr.shape[0] - 1
    dense = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(indptr))
    dense[rows, indices] = data
    x = rng.standard_normal(n)
    assert np.allclose(kernels.csr_matvec(indptr, indices, data, x), dense @ x, rtol=1e-13)


def test_scatter_add_fixed_order_is_deterministic(rng):
    """test_kernels.py:48-56"""
    n = 40
    dest = rng.integers(0, n, 2000)
    contribs = rng.standard_normal(2000)
    a = np.zeros(n)
    b = np.zeros(n)
    kernels.scatter_add(a, dest, contribs)
    kernels.scatter_add(b, dest, contribs)
    assert np.array_equal(a, b)


def test_matvec_bit_identical_across_calls(rng):
    """test_kernels.py:59-68 (thread counts -> repeated launches)"""
    indptr, indices, data = random_csr(rng, n=5000, per_row=30)
    x = rng.standard_normal(indptr.shape[0] - 1)
    assert np.array_equal(kernels.csr_matvec(indptr, indices, data, x), kernels.csr_matvec(indptr, indices, data, x))


def test_scatter_add_rejects_out_of_range_and_mismatch():
    v = np.zeros(4)
    with pytest.raises(IndexError):
        kernels.scatter_add(v, np.array([0, 4]), np.ones(2))
    with pytest.raises(IndexError):
        kernels.scatter_add(v, np.array([-1]), np.ones(1))
    assert np.array_equal(v, np.zeros(4))  # nothing applied
    with pytest.raises(ValueError):
        kernels.scatter_add(v, np.array([0, 1]), np.ones(3))
    kernels.scatter_add(v, np.zeros(0, dtype=np.int64), np.zeros(0))  # empty: no-op
