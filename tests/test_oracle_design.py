"""Pin the oracle's design-loop row to the reference's outputs
(tests/golden/design.npz, see make_golden_design.py).

Bit-exact: filter pattern, filter weights, filter products (row-sequential), the MMA
iterates and asymptotes.  FP64: the L2 field error to 1e-13."""

import numpy as np
import pytest

import oracle as orc
from conftest import load_golden

FILTERS = [((4, 3, 2), (4.0, 3.0, 2.0), 1.6), ((3, 3, 2), (3.0, 3.0, 2.0), 1.7), ((6, 4, 3), (3.0, 2.0, 1.5), 0.8),
           ((5, 5, 1), (1.0, 1.0, 0.2), 0.45)]


@pytest.fixture(scope="module")
def g():
    return load_golden("design")


@pytest.mark.parametrize("k", range(len(FILTERS)))
def test_density_filter_bit_exact(g, k):
    dims, box, r = FILTERS[k]
    nodes, cells = orc.box_mesh(*dims, *box)
    H = orc.density_filter(nodes, cells, r)
    assert np.array_equal(H[0], g[f"f{k}_indptr"]) and np.array_equal(H[1], g[f"f{k}_indices"])
    assert np.array_equal(H[2], g[f"f{k}_data"])
    assert np.array_equal(orc.filter_apply(H, g[f"f{k}_x"]), g[f"f{k}_Hx"])
    th = g[f"f{k}_theta"]
    assert np.array_equal(orc.filter_apply(H, g[f"f{k}_sens"], mul=th, div=th, floor=1e-3), g[f"f{k}_fs"])


def test_mma_sequence(g):
    n = g["mma_x0"].size
    st = dict(lower=None, upper=None, x_prev=None, x_prev2=None, iteration=0, move_limit=0.2, asym_init=0.5,
              asym_expand=1.2, asym_shrink=0.7)
    x = g["mma_x0"]
    for k in range(5):
        xn = orc.mma_update(st, x, g[f"mma{k}_dj"], float(g[f"mma{k}_g"]), np.full(n, 1.0 / n), 1e-3, 1.0)
        assert np.array_equal(st["lower"], g[f"mma{k}_low"]) and np.array_equal(st["upper"], g[f"mma{k}_upp"])
        assert np.abs(xn - g[f"mma{k}_x"]).max() <= 1e-12
        x = g[f"mma{k}_x"]


def test_l2_field_error(g):
    nodes, cells = orc.box_mesh(3, 3, 2, 1.0, 1.0, 0.4)
    e = orc.l2_field_error(nodes, cells, g["l2_up"], g["l2_ut"])
    assert abs(e - float(g["l2"])) <= 1e-13 * float(g["l2"])
