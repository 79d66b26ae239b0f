"""Pin the oracle's low-seam restatement (oracle csr_matvec / scatter_add, reference
kernels.py:21-55) to the reference's numba kernels (tests/golden/lowseam.npz,
make_golden_lowseam.py): bit-exact."""

import numpy as np
import pytest

import oracle as orc
from conftest import load_golden


@pytest.fixture(scope="module")
def g():
    return load_golden("lowseam")


@pytest.mark.parametrize("name", ["small", "empty_row", "large"])
def test_oracle_csr_matvec_bit_exact(g, name):
    y = orc.csr_matvec(g[f"{name}_indptr"], g[f"{name}_indices"], g[f"{name}_data"], g[f"{name}_x"])
    assert np.array_equal(y, g[f"{name}_y"])


@pytest.mark.parametrize("name", ["scatter_small", "scatter_large"])
def test_oracle_scatter_add_bit_exact(g, name):
    v = g[f"{name}_v0"].copy()
    orc.scatter_add(v, g[f"{name}_dest"], g[f"{name}_contribs"])
    assert np.array_equal(v, g[f"{name}_v"])
