"""ctypes binding of libb200fem.so (include/b200fem.h).

The product path has NO CPU fallback: if the library is missing or no CUDA device is
visible, every device entry point raises ``DeviceUnavailableError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libb200fem.so")

OK = 0
E_INVERTED_ELEMENT = 1
E_INVERTED_DEFORMATION = 2
E_NONFINITE_VALUE = 3
E_NONFINITE_DERIV = 4
E_LINEAR_SOLVER = 5
E_BREAKDOWN = 6
E_ZERO_DIAGONAL = 7
E_INVALID = 8
E_CUDA = 9
E_UNSUPPORTED = 10

MAT_POISSON, MAT_LE, MAT_NH, MAT_J2 = 0, 1, 2, 3
FLAG_SIMP, FLAG_DESIGN_SOURCE = 1, 2


class DeviceUnavailableError(RuntimeError):
    """libb200fem.so is not built or no CUDA device is present (there is no CPU path)."""


class Error(C.Structure):
    _fields_ = [("code", C.c_int32), ("qp", C.c_int32), ("cell", C.c_int64), ("value", C.c_double),
                ("iterations", C.c_int64), ("msg", C.c_char * 256)]

    @property
    def message(self):
        return self.msg.decode(errors="replace")


class SolveInfo(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvecs", C.c_int64), ("restarts", C.c_int64),
                ("residual", C.c_double), ("tol", C.c_double)]


_vp = C.c_void_p
_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double
_pf64 = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)
_pi32 = C.POINTER(C.c_int32)
_perr = C.POINTER(Error)

# name -> (restype, argtypes)
SIGNATURES = {
    "b200fem_version": (C.c_int, []),
    "b200fem_launch_count": (_i64, []),
    "b200fem_stream_sync": (C.c_int, [_vp]),
    "b200fem_ctx_create": (C.c_int, [C.POINTER(_vp), _i64, _i64, _i32, _vp, _vp, _i32, _vp, _i32, _vp, _perr]),
    "b200fem_ctx_destroy": (C.c_int, [_vp]),
    "b200fem_ctx_info": (C.c_int, [_vp, _pi64, _pi64, _pi32]),
    "b200fem_copy_indptr": (C.c_int, [_vp, _vp]),
    "b200fem_copy_indices": (C.c_int, [_vp, _vp]),
    "b200fem_copy_dest": (C.c_int, [_vp, _i64, _i64, _vp]),
    "b200fem_copy_diag_slots": (C.c_int, [_vp, _vp]),
    "b200fem_set_dirichlet": (C.c_int, [_vp, _vp, _vp, _i64]),
    "b200fem_set_loads": (C.c_int, [_vp, _vp, _vp]),
    "b200fem_set_theta": (C.c_int, [_vp, _vp, _i64, _i32]),
    "b200fem_set_state": (C.c_int, [_vp, _vp, _vp, _i32]),
    "b200fem_get_state": (C.c_int, [_vp, _vp, _vp]),
    "b200fem_residual": (C.c_int, [_vp, _vp, _f64, _i32, _vp, _pf64, _perr]),
    "b200fem_jacobian": (C.c_int, [_vp, _vp, _vp, _perr]),
    "b200fem_qp_flux": (C.c_int, [_vp, _vp, _vp, _perr]),
    "b200fem_volume_average_flux": (C.c_int, [_vp, _vp, _vp, _perr]),
    "b200fem_commit_state": (C.c_int, [_vp, _vp]),
    "b200fem_geometry": (C.c_int, [_vp, _vp, _vp]),
    "b200fem_law_batch": (C.c_int, [_i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _perr]),
    "b200fem_nh_energy_batch": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "b200fem_param_vjp": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _perr]),
    "b200fem_transpose_fem": (C.c_int, [_vp, _vp, _vp]),
    "b200fem_csr_transpose": (C.c_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "b200fem_matrix_fem": (C.c_int, [C.POINTER(_vp), _vp, _vp]),
    "b200fem_matrix_csr": (C.c_int, [C.POINTER(_vp), _i64, _i64, _vp, _vp, _vp, _vp]),
    "b200fem_ctx_sym_size": (C.c_int, [_vp, _pi64]),
    "b200fem_jacobian_sym": (C.c_int, [_vp, _vp, _vp, _vp, _perr]),
    "b200fem_matrix_fem_sym": (C.c_int, [C.POINTER(_vp), _vp, _vp]),
    "b200fem_ctx_grid_size": (C.c_int, [_vp, _pi64, C.POINTER(C.c_int32)]),
    "b200fem_jacobian_grid": (C.c_int, [_vp, _vp, _vp, _vp, _perr]),
    "b200fem_matrix_fem_grid": (C.c_int, [C.POINTER(_vp), _vp, _vp]),
    "b200fem_matrix_fem_grid_ex": (C.c_int, [C.POINTER(_vp), _vp, _vp, C.c_int32]),
    "b200fem_matrix_set_data": (C.c_int, [_vp, _vp]),
    "b200fem_grid_to_f32": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "b200fem_matrix_set_f32": (C.c_int, [_vp, _vp]),
    "b200fem_matrix_destroy": (C.c_int, [_vp]),
    "b200fem_matvec": (C.c_int, [_vp, _vp, _vp]),
    "b200fem_diagonal": (C.c_int, [_vp, _vp]),
    "b200fem_bicgstab": (C.c_int, [_vp, _vp, _vp, _i32, _f64, _f64, _i64, C.POINTER(SolveInfo), _perr]),
    "b200fem_bicgstab_profile": (C.c_int, [_vp, _vp, _vp, _i32, _pf64]),
    "b200fem_pcg": (C.c_int, [_vp, _vp, _vp, _i32, _f64, _f64, _i64, C.POINTER(SolveInfo), _perr]),
    "b200fem_comm_unique_id": (C.c_int, [_vp]),
    "b200fem_comm_create_nccl": (C.c_int, [C.POINTER(_vp), _vp, _i32, _i32]),
    "b200fem_comm_create_local": (C.c_int, [C.POINTER(_vp)]),
    "b200fem_comm_destroy": (C.c_int, [_vp]),
    "b200fem_comm_allreduce": (C.c_int, [_vp, _vp, _i64, _vp]),
    "b200fem_part_create": (C.c_int, [C.POINTER(_vp), _vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "b200fem_part_destroy": (C.c_int, [_vp]),
    "b200fem_dist_bicgstab": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i32, _f64, _f64, _i64, C.POINTER(SolveInfo),
                                        _perr]),
    "b200fem_dist_pcg": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i32, _f64, _f64, _i64, C.POINTER(SolveInfo),
                                   _perr]),
    "b200fem_dist_halo": (C.c_int, [_vp, _i32, _vp, _vp]),
    "b200fem_dist_dot": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _pf64]),
    "b200fem_norm2": (C.c_int, [_vp, _i64, _pf64, _vp]),
    "b200fem_dot": (C.c_int, [_vp, _vp, _i64, _pf64, _vp]),
    "b200fem_filter_create": (C.c_int, [C.POINTER(_vp), _i64, _vp, _vp, C.c_double, _vp]),
    "b200fem_filter_info": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "b200fem_filter_copy": (C.c_int, [_vp, _vp, _vp, _vp]),
    "b200fem_filter_apply": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp]),
    "b200fem_filter_destroy": (C.c_int, [_vp]),
    "b200fem_mma_update": (C.c_int, [_i64, _vp, _vp, C.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                     C.c_double, C.c_double, C.c_double, C.c_double, _vp, _vp]),
    "b200fem_l2_field_error": (C.c_int, [_i64, _vp, _vp, _vp, _vp, _pf64, _vp]),
    "b200fem_format_f64_rows": (C.c_int64, [_vp, _i64, C.c_int32, _vp, _i64]),
    "b200fem_format_i64_rows": (C.c_int64, [_vp, _i64, C.c_int32, _i64, _vp, _i64]),
    "b200fem_gather_sum": (C.c_int, [_vp, _vp, _i64, _pf64, _vp]),
    "b200fem_axpy": (C.c_int, [_i64, _f64, _vp, _vp, _vp]),
    "b200fem_csr_matvec_seq": (C.c_int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "b200fem_scatter_add": (C.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, C.POINTER(Error)]),
    "b200fem_scale": (C.c_int, [_i64, _f64, _vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen libb200fem.so and declare every prototype (no device needed)."""
    if not os.path.exists(path):
        raise DeviceUnavailableError(
            f"{path} is not built; run `python -m paper_2212_00964_b200._build` (nvcc, sm_100a)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded library, after checking that a CUDA device is present."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch

                if not torch.cuda.is_available():
                    raise DeviceUnavailableError(
                        "no CUDA device: the forward-solve path runs only on the GPU (no CPU fallback)")
                _lib = load_library()
    return _lib


_host = None


def host_lib():
    """The library for its host-only entry points (output formatting): no device needed."""
    global _host
    if _host is None:
        with _lock:
            if _host is None:
                _host = _lib if _lib is not None else load_library()
    return _host


def launch_count() -> int:
    return int(lib().b200fem_launch_count())
