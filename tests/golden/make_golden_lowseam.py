"""Generate tests/golden/lowseam.npz with the REFERENCE low-seam kernels (build container only):
gradfem.kernels.csr_matvec and scatter_add (numba backend) on random CSR matrices and
scatters, including an empty row, duplicate destinations and a 5000-row matrix.

    python tests/golden/make_golden_lowseam.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import gradfem.kernels as kernels  # noqa: E402
from gradfem.backend import HAS_NUMBA  # noqa: E402


def random_csr(rng, n, per_row, empty_row=None):  # as the reference's tests/test_kernels.py:8-15
    indptr = np.zeros(n + 1, dtype=np.int32)
    indices = []
    for i in range(n):
        cols = [] if i == empty_row else np.unique(np.append(rng.choice(n, per_row), i))
        indices.extend(np.sort(cols))
        indptr[i + 1] = len(indices)
    return indptr, np.array(indices, dtype=np.int32), rng.standard_normal(len(indices))


if __name__ == "__main__":
    assert HAS_NUMBA, "goldens come from the numba kernels"
    rng = np.random.default_rng(11)
    out = {}
    for name, (n, per_row, empty) in {"small": (60, 7, None), "empty_row": (50, 5, 17),
                                      "large": (5000, 30, None)}.items():
        ip, ix, d = random_csr(rng, n, per_row, empty)
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)
        out[f"{name}_indptr"], out[f"{name}_indices"], out[f"{name}_data"], out[f"{name}_x"] = ip, ix, d, x
        out[f"{name}_y"] = kernels.csr_matvec(ip, ix, d, x)
    for name, (nv, nc) in {"scatter_small": (40, 2000), "scatter_large": (1000, 50_000)}.items():
        dest = rng.integers(0, nv, nc)
        contribs = rng.standard_normal(nc) * 10.0 ** rng.integers(-8, 8, nc)
        v0 = rng.standard_normal(nv)
        v = v0.copy()
        kernels.scatter_add(v, dest, contribs)
        out[f"{name}_v0"], out[f"{name}_dest"], out[f"{name}_contribs"], out[f"{name}_v"] = v0, dest, contribs, v
    np.savez_compressed(os.path.join(HERE, "lowseam.npz"), **out)
    print("wrote lowseam.npz", {k: v.shape for k, v in out.items()})
