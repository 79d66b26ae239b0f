"""Device-resident CSR matrix with the reference CsrMatrix interface (sparse.py:15-72).

``indptr`` (int32), ``indices`` (int32) and ``data`` (float64) are exposed as host numpy
arrays, downloaded lazily and cached, so reference-style code and parity tests work
unchanged; the operator itself (matvec, diagonal, Krylov) runs on the GPU.  A matrix
assembled on an FEM workspace keeps only its values on the device and reuses the
workspace's node-blocked pattern (no 4-byte-per-nonzero index array is needed).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as D
from . import _lib
from .errors import raise_for


class CsrMatrix:
    """CSR storage; column indices sorted and unique within each row."""

    def __init__(self, indptr, indices, data):
        t = D.torch()
        self._ws = None
        self._h_indptr = None if indptr is None else _host(indptr, np.int32)
        self._h_indices = None if indices is None else _host(indices, np.int32)
        self._h_data = None
        self._d_data = None
        if isinstance(data, t.Tensor) and data.is_cuda:
            self._d_data = data.contiguous().to(t.float64)
        else:
            self._h_data = _host(data, np.float64)
        self._d_indptr = self._d_indices = None
        self._handle = None
        n = (self._h_indptr.shape[0] - 1) if self._h_indptr is not None else 0
        self._n = n

    @classmethod
    def _from_workspace(cls, ws, data_dev):
        m = cls.__new__(cls)
        m._ws = ws
        m._h_indptr = m._h_indices = m._h_data = None
        m._d_data = data_dev
        m._d_indptr = m._d_indices = None
        m._handle = None
        m._n = ws.n_dofs
        return m

    # ------------------------------------------------------------ host views
    @property
    def indptr(self) -> np.ndarray:
        if self._h_indptr is None:
            self._h_indptr = self._ws.indptr
        return self._h_indptr

    @property
    def indices(self) -> np.ndarray:
        if self._h_indices is None:
            self._h_indices = self._ws.indices
        return self._h_indices

    @property
    def data(self) -> np.ndarray:
        if self._h_data is None:
            self._h_data = D.to_host(self._d_data)
        return self._h_data

    @data.setter
    def data(self, values):
        self._h_data = _host(values, np.float64)
        self._d_data = None
        if self._handle is not None:
            _lib.lib().b200fem_matrix_set_data(self._handle, D.ptr(self.device_data))

    @property
    def device_data(self):
        """CSR values as a CUDA float64 tensor (uploaded on first use)."""
        if self._d_data is None:
            self._d_data = D.to_device(self._h_data)
        return self._d_data

    @property
    def shape(self):
        return (self._n, self._n)

    @property
    def nnz(self) -> int:
        if self._ws is not None:
            return int(self._ws.nnz)
        return int(self._h_indices.shape[0])

    # --------------------------------------------------------- device handle
    def _device_handle(self):
        if self._handle is None:
            lib = _lib.lib()
            h = C.c_void_p()
            if self._ws is not None:
                st = lib.b200fem_matrix_fem(C.byref(h), self._ws.ctx, D.ptr(self.device_data))
            else:
                self._d_indptr = D.to_device(self._h_indptr, D.torch().int32)
                self._d_indices = D.to_device(self._h_indices, D.torch().int32)
                st = lib.b200fem_matrix_csr(C.byref(h), self._n, self._h_indices.shape[0], D.ptr(self._d_indptr),
                                            D.ptr(self._d_indices), D.ptr(self.device_data), D.stream())
            raise_for(st, None, "matrix handle")
            self._handle = h
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.b200fem_matrix_destroy(h)
            except Exception:
                pass

    # ------------------------------------------------------------- operator
    def matvec(self, x):
        as_host = not D.is_device_tensor(x)
        xd = D.to_device(x)
        if xd.shape != (self._n,):
            raise ValueError(f"x must have shape ({self._n},), got {tuple(xd.shape)}")
        y = D.empty(self._n)
        raise_for(_lib.lib().b200fem_matvec(self._device_handle(), D.ptr(xd), D.ptr(y)), None, "matvec")
        return D.to_host(y) if as_host else y

    def __matmul__(self, x):
        return self.matvec(x)

    def device_diagonal(self):
        d = D.empty(self._n)
        raise_for(_lib.lib().b200fem_diagonal(self._device_handle(), D.ptr(d)), None, "diagonal")
        return d

    def diagonal(self) -> np.ndarray:
        return D.to_host(self.device_diagonal())

    def row_keys(self) -> np.ndarray:
        n = self._n
        return np.repeat(np.arange(n, dtype=np.int64), np.diff(self.indptr)) * n + self.indices

    def todense(self) -> np.ndarray:
        n = self._n
        out = np.zeros((n, n))
        rows = np.repeat(np.arange(n), np.diff(self.indptr))
        out[rows, self.indices] = self.data
        return out

    def transpose(self) -> "CsrMatrix":
        """Explicit transpose on the device (sparse.py:53-62: stable by column).

        A workspace matrix keeps its (structurally symmetric) pattern and only permutes the
        values (csrc/transpose.cu); a generic CSR goes through a stable radix sort."""
        lib = _lib.lib()
        if self._ws is not None:
            data_t = D.empty(self._ws.nnz)
            raise_for(lib.b200fem_transpose_fem(self._ws.ctx, D.ptr(self.device_data), D.ptr(data_t)), None,
                      "transpose_fem")
            return CsrMatrix._from_workspace(self._ws, data_t)
        t = D.torch()
        n, nnz = self._n, int(self._h_indices.shape[0])
        ip = D.to_device(self._h_indptr, t.int32)
        ix = D.to_device(self._h_indices, t.int32)
        ip_t = D.empty(n + 1, t.int32)
        ix_t = D.empty(max(nnz, 1), t.int32)
        d_t = D.empty(max(nnz, 1))
        raise_for(lib.b200fem_csr_transpose(n, nnz, D.ptr(ip), D.ptr(ix), D.ptr(self.device_data), D.ptr(ip_t),
                                            D.ptr(ix_t), D.ptr(d_t), D.stream()), None, "csr_transpose")
        return CsrMatrix(D.to_host(ip_t), D.to_host(ix_t)[:nnz], d_t[:nnz])

    def copy_structure(self) -> "CsrMatrix":
        if self._ws is not None:
            return CsrMatrix._from_workspace(self._ws, D.zeros(self._ws.nnz))
        return CsrMatrix(self.indptr, self.indices, np.zeros_like(self.data))


def _host(a, dtype):
    t = D.torch()
    if isinstance(a, t.Tensor):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


class _NodeBlockOperator:
    """Base of the device-only tangent operators used inside the Newton loop."""

    _ctor = None
    _size = None

    def __init__(self, ws, data=None):
        """``data``: share an existing value buffer (e.g. the FP64 GRID3 values of the "grid"
        and "grid32" Newton operators; each re-assembles into it before use)."""
        self._ws = ws
        self._n = ws.n_dofs
        # zero-filled once: lattice slots of missing neighbours are never written (the matvec
        # masks them) and must not hold stale bits for value copies such as refresh_f32
        if data is None:
            with ws.on_stream():
                data = D.zeros(getattr(ws, self._size)())
        self.device_data = data
        self._handle = None

    @property
    def shape(self):
        return (self._n, self._n)

    def _device_handle(self):
        if self._handle is None:
            h = C.c_void_p()
            raise_for(getattr(_lib.lib(), self._ctor)(C.byref(h), self._ws.ctx, D.ptr(self.device_data)), None,
                      self._ctor)
            self._handle = h
        return self._handle

    def matvec(self, x):
        as_host = not D.is_device_tensor(x)
        xd = D.to_device(x)
        y = D.empty(self._n)
        raise_for(_lib.lib().b200fem_matvec(self._device_handle(), D.ptr(xd), D.ptr(y)), None, "matvec")
        return D.to_host(y) if as_host else y

    __matmul__ = matvec

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.b200fem_matrix_destroy(h)
            except Exception:
                pass


class GridOperator(_NodeBlockOperator):
    """The tangent of a box-lattice workspace in GRID storage (csrc/spmv.cu GRID3).

    Same linear operator as the CSR Jacobian (identity Dirichlet rows).  Only the self block
    and the 13 upper-offset node blocks (3x3 for vec 3, scalars for vec 1) are stored, tiled
    element streams, so a vec-3 matvec streams 14*72 B per node instead of 27*72 B + column
    ids, and the lower blocks are re-read from L2.  Used by the Newton loop's Krylov solves;
    ``assemble_jacobian`` still returns the reference CSR."""

    _ctor = "b200fem_matrix_fem_grid"
    _size = "grid_size"

    def refresh_f32(self):
        """Round the current values into the single-precision copy that the matvec then streams
        (operator "grid32", b200fem_matrix_set_f32); call after every re-assembly."""
        lib = _lib.lib()
        if getattr(self, "device_data32", None) is None:
            self.device_data32 = D.empty(self.device_data.numel(), D.torch().float32)
            raise_for(lib.b200fem_matrix_set_f32(self._device_handle(), D.ptr(self.device_data32)), None,
                      "matrix_set_f32")
        raise_for(lib.b200fem_grid_to_f32(D.ptr(self.device_data), D.ptr(self.device_data32), self.device_data.numel(),
                                     D.stream()), None, "grid_to_f32")

    def matvec_pre_dirichlet(self, x):
        """K0 x: the same values without the identity Dirichlet rows (device in, device out)."""
        h = getattr(self, "_raw", None)
        if h is None:
            h = C.c_void_p()
            raise_for(_lib.lib().b200fem_matrix_fem_grid_ex(C.byref(h), self._ws.ctx, D.ptr(self.device_data), 1),
                      None, "matrix_fem_grid_ex")
            self._raw = h
        xd = D.to_device(x)
        y = D.empty(self._n)
        raise_for(_lib.lib().b200fem_matvec(h, D.ptr(xd), D.ptr(y)), None, "matvec")
        return y

    def __del__(self):
        h = getattr(self, "_raw", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.b200fem_matrix_destroy(h)
            except Exception:
                pass
        super().__del__()


class SymOperator:
    """The tangent of a vec-3 workspace as a symmetric node-block operator (csrc SYM3).

    Same linear operator as the CSR Jacobian of the workspace (identity Dirichlet rows) with
    only the upper 3x3 node blocks stored: about half of the value bytes per matvec.  Used by
    the Newton loop's Krylov solves; ``assemble_jacobian`` still returns the full CSR."""

    def __init__(self, ws):
        self._ws = ws
        self._n = ws.n_dofs
        self.device_data = D.empty(ws.sym_size())
        self._handle = None

    @property
    def shape(self):
        return (self._n, self._n)

    def _device_handle(self):
        if self._handle is None:
            h = C.c_void_p()
            raise_for(_lib.lib().b200fem_matrix_fem_sym(C.byref(h), self._ws.ctx, D.ptr(self.device_data)), None,
                      "matrix_fem_sym")
            self._handle = h
        return self._handle

    def matvec(self, x):
        as_host = not D.is_device_tensor(x)
        xd = D.to_device(x)
        y = D.empty(self._n)
        raise_for(_lib.lib().b200fem_matvec(self._device_handle(), D.ptr(xd), D.ptr(y)), None, "matvec")
        return D.to_host(y) if as_host else y

    __matmul__ = matvec

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            try:
                _lib._lib.b200fem_matrix_destroy(h)
            except Exception:
                pass
