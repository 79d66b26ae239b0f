"""The reference's low seam, on the device: ``gradfem.kernels.csr_matvec`` and
``scatter_add`` (reference kernels.py:1-55; SURVEY.md §8(b) seam 1).

Same signatures and the same fixed accumulation order, so the results are bit-identical to
the reference's numba kernels (csrc/lowseam.cu):

* ``csr_matvec(indptr, indices, data, x) -> y``: per row, ((0 + d0 x0) + d1 x1) + ... in
  storage order with separately rounded products and sums (kernels.py:21-28).
* ``scatter_add(values, dest, contribs)``: ``values[dest[k]] += contribs[k]`` in ascending k,
  in place (kernels.py:30-34, 50-55).

Host (numpy) arguments give host results (``values`` updated in place); CUDA tensors stay on
the device.  This seam serves user-built matrices and scatters; the Newton loop uses the
fused assembly and the FEM / GRID3 operators instead.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as D
from . import _lib
from .errors import raise_for


def csr_matvec(indptr, indices, data, x):
    """y = A @ x for a CSR matrix given by (indptr, indices, data) (kernels.py:37-47)."""
    host = not D.is_device_tensor(x)
    t = D.torch()
    ip = D.to_device(indptr, t.int32)
    ix = D.to_device(indices, t.int32)
    dv = D.to_device(data)
    xv = D.to_device(x)
    n = int(ip.shape[0]) - 1
    if int(ix.shape[0]) != int(dv.shape[0]):
        raise ValueError(f"indices ({int(ix.shape[0])}) and data ({int(dv.shape[0])}) lengths differ")
    y = D.empty(max(n, 0))
    raise_for(_lib.lib().b200fem_csr_matvec_seq(n, D.ptr(ip), D.ptr(ix), D.ptr(dv), D.ptr(xv), D.ptr(y),
                                                 D.stream()), None, "csr_matvec")
    return D.to_host(y) if host else y


def scatter_add(values, dest, contribs):
    """values[dest[k]] += contribs[k], accumulated in ascending k (kernels.py:50-55)."""
    t = D.torch()
    host = not D.is_device_tensor(values)
    if not host and (values.dtype != t.float64 or not values.is_contiguous()):
        raise TypeError("scatter_add on a CUDA tensor needs a contiguous float64 values tensor (updated in place)")
    v = D.to_device(values)  # the tensor itself on the device path, a copy of a host array
    d = D.to_device(dest, t.int64)
    c = D.to_device(contribs)
    if int(d.shape[0]) != int(c.shape[0]):
        raise ValueError(f"dest ({int(d.shape[0])}) and contribs ({int(c.shape[0])}) lengths differ")
    err = _lib.Error()
    st = _lib.lib().b200fem_scatter_add(D.ptr(v), int(v.shape[0]), D.ptr(d), D.ptr(c), int(d.shape[0]), D.stream(),
                                        C.byref(err))
    if st == _lib.E_INVALID:
        raise IndexError(err.message)
    raise_for(st, err, "scatter_add")
    if host:
        values[...] = D.to_host(v)
