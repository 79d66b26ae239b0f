"""CPU checks of the reference-arm measurement tools (tools/cpu_reference.py): the full-pattern
system the reference's Krylov phase is timed on has exactly the reference workspace's sparsity,
and the composition adds up its phases.  Needs the reference package (baseline/_ref, or
/root/reference in the build container); skipped otherwise."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def _gradfem():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "gradfem")):
            sys.path.insert(0, path)
            try:
                import gradfem

                return gradfem
            except Exception:
                return None
    return None


gf = _gradfem()
pytestmark = pytest.mark.skipif(gf is None, reason="reference package not installed")


@pytest.mark.parametrize("n", [1, 3, 5])
def test_lattice_csr_is_the_reference_pattern(n):
    import cpu_reference as cr
    import fullsize_cases as fc
    from gradfem.assembly import workspace

    ip, ix, data = cr.lattice_csr(n)
    ws = workspace(fc.c3(gf, n))
    assert np.array_equal(ip, ws.indptr) and np.array_equal(ix, ws.indices)
    from gradfem.sparse import CsrMatrix

    A = CsrMatrix(ip, ix, data)
    d = A.diagonal()
    assert np.all(d == 1.0)
    off = np.abs(data).sum() - d.sum()
    assert off < d.sum()  # diagonally dominant overall: the timed BiCGSTAB does not break down


def test_composition_adds_up():
    import cpu_reference as cr

    comp = cr.ReferenceComposer.__new__(cr.ReferenceComposer)
    comp.n_target, comp.n_csr, comp.ws_per_cell = 10, 10, 2e-6
    comp.kry = {"matvec_s": 0.01, "bicgstab_iter_s": 0.05, "bicgstab_fixed_s": 0.2}
    comp.its, comp.its_src = 136, "test"
    comp.A = type("A", (), {"nnz": 9 * 31 ** 3})()
    r = comp.compose(t_K=1e-3, t_R=1e-5, t_mv=0.01)
    p = r["parts"]
    assert r["value"] == pytest.approx(sum(p.values()))
    assert p["jacobian_s"] == pytest.approx(3 * 1e-3 * 1000)
    assert p["residual_s"] == pytest.approx(4 * 1e-5 * 1000)
    # Krylov: 3 solves x fixed cost + iterations (scaled to n = 10 from 136) x (2 matvecs + vector work)
    its = 136 * 10 / 136.0
    assert p["krylov_s"] == pytest.approx(3 * 0.2 + its * (2 * 0.01 + 0.03))
