"""ctypes binding of libctsm_b200.so (include/ctsm_b200.h).

The library is the product: there is no CPU fallback. If the shared library is
missing the import of any projector function fails loudly.
"""
from __future__ import annotations

import ctypes
import os

from .geometry import CGeometry, CtsmError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libctsm_b200.so")

CTSM_F64 = 0
CTSM_F32 = 1

_P = ctypes.c_void_p
_I = ctypes.c_int
_U64 = ctypes.c_uint64
_GP = ctypes.POINTER(CGeometry)
_D = ctypes.c_double

CTSM_OP_CSR = 0
CTSM_OP_MATRIX_FREE = 1


class COperator(ctypes.Structure):
    """ctsm_operator (include/ctsm_b200.h)."""
    _fields_ = [("kind", ctypes.c_int), ("pad0", ctypes.c_int),
                ("n_rows", ctypes.c_uint64), ("n_cols", ctypes.c_uint64),
                ("row_start", ctypes.c_void_p), ("col", ctypes.c_void_p), ("val", ctypes.c_void_p),
                ("geom", _GP), ("scale", ctypes.c_double),
                ("col_start", ctypes.c_void_p), ("trow", ctypes.c_void_p),
                ("tval", ctypes.c_void_p)]


_OP = ctypes.POINTER(COperator)

# name -> (restype, argtypes); mirrors include/ctsm_b200.h
SIGNATURES = {
    "ctsm_create": (_I, [_I, ctypes.POINTER(_P)]),
    "ctsm_destroy": (_I, [_P]),
    "ctsm_last_error": (ctypes.c_char_p, []),
    "ctsm_version": (ctypes.c_char_p, []),
    "ctsm_launch_count": (_U64, []),
    "ctsm_validate_geometry": (_I, [_GP]),
    "ctsm_csr_count": (_I, [_P, _GP, _I, _I, _U64, _P, ctypes.POINTER(_U64), _P]),
    "ctsm_csr_fill": (_I, [_P, _GP, _I, _I, _P, _P, _P, _P]),
    "ctsm_weights_batch": (_I, [_P, _GP, _U64, _P, _P, _P, _P, _I, _P, _P, _P, _P]),
    "ctsm_angle_block_entries": (_I, [_P, _GP, _I, _I, _I, _U64, _P, _P, _P,
                                      ctypes.POINTER(_U64), _P]),
    "ctsm_shard_angles": (_I, [_GP, _I, _I, _P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "ctsm_multi_create": (_I, [_P, _I, ctypes.POINTER(_P)]),
    "ctsm_multi_destroy": (_I, [_P]),
    "ctsm_multi_size": (_I, [_P]),
    "ctsm_multi_nccl_version": (_I, [_P]),
    "ctsm_multi_forward_project_matrix_free_host": (_I, [_P, _GP, _I, _P, _P]),
    "ctsm_multi_back_project_matrix_free_host": (_I, [_P, _GP, _I, _P, _P]),
    "ctsm_multi_sirt_host": (_I, [_P, _GP, _I, _P, _P, _I]),
    "ctsm_mc_volume_3d": (_I, [_P, _U64, _P, _P, _D, _D, _D, _D, _P, _P, _U64, _U64, _P, _P, _P]),
    "ctsm_multiline_volume_3d": (_I, [_P, _U64, _P, _P, _D, _D, _D, _D, _P, _P, _I, _P]),
    "ctsm_gauss_legendre": (None, [_I, _P, _P]),
    "ctsm_selftest_division": (_I, [_P, _U64, _U64, ctypes.POINTER(_U64)]),
    "ctsm_csr_angle_nnz": (_I, [_P, _GP, _I, ctypes.POINTER(_U64), _P]),
    "ctsm_csr_build": (_I, [_P, _GP, _I, _I, _U64, _P, _P, _P, _U64, ctypes.POINTER(_U64), _P]),
    "ctsm_spmv": (_I, [_P, _U64, _U64, _P, _P, _P, _P, _P, _P]),
    "ctsm_spmv_t": (_I, [_P, _U64, _U64, _P, _P, _P, _P, _P, _P]),
    "ctsm_csr_colsum_max": (_I, [_P, _U64, _U64, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "ctsm_spmv_t_bound": (_I, [_P, _U64, _U64, _P, _P, _P, _D, _P, _P, _P]),
    "ctsm_csc_build": (_I, [_P, _U64, _U64, _P, _P, _P, _P, _P, _P, _P]),
    "ctsm_spmv_t_csc": (_I, [_P, _U64, _U64, _P, _P, _P, _D, _P, _P, _P]),
    "ctsm_fwd_mf": (_I, [_P, _GP, _I, _I, _I, _I, _P, _P, _P]),
    "ctsm_bwd_mf": (_I, [_P, _GP, _I, _I, _I, _I, _P, _P, _P]),
    "ctsm_last_update_count": (_U64, [_P]),
    "ctsm_last_kernel_path": (_I, [_P]),
    "ctsm_quarter_symmetric": (_I, [_GP]),
    "ctsm_symmetry_order": (_I, [_GP]),
    "ctsm_fwd_mf_orbits": (_I, [_P, _GP, _I, _I, _I, _P, _P, _P]),
    "ctsm_bwd_mf_orbits": (_I, [_P, _GP, _I, _I, _I, _P, _P, _P]),
    "ctsm_invert_nonzero": (_I, [_P, _I, _U64, _P, _P]),
    "ctsm_sirt_residual": (_I, [_P, _GP, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ctsm_sirt_update": (_I, [_P, _I, _U64, _P, _P, _P, _P]),
    "ctsm_sirt": (_I, [_P, _GP, _I, _P, _P, _I, _P]),
    "ctsm_csr_count_mode": (_I, [_P, _GP, _I, _I, _I, _I, _U64, _P, ctypes.POINTER(_U64), _P]),
    "ctsm_csr_fill_mode": (_I, [_P, _GP, _I, _I, _I, _I, _P, _P, _P, _P]),
    "ctsm_fwd_mf_mode": (_I, [_P, _GP, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ctsm_bwd_mf_mode": (_I, [_P, _GP, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ctsm_forward_project_matrix_free_host": (_I, [_P, _GP, _P, _P]),
    "ctsm_back_project_matrix_free_host": (_I, [_P, _GP, _P, _P]),
    "ctsm_forward_project_matrix_free_host_f32": (_I, [_P, _GP, _P, _P]),
    "ctsm_back_project_matrix_free_host_f32": (_I, [_P, _GP, _P, _P]),
    "ctsm_spectral_norm_power": (_I, [_P, _OP, _I, _P, ctypes.POINTER(_D), _P]),
    "ctsm_nag_tikhonov": (_I, [_P, _OP, _P, _D, _I, _D, _P, _P, ctypes.POINTER(_I),
                               ctypes.POINTER(_I), _P]),
    "ctsm_scale_values": (_I, [_P, _U64, _P, _D, _P]),
    "ctsm_normal_samples": (None, [_U64, _U64, _P]),
    "ctsm_write_csm1_device": (_I, [_P, ctypes.c_char_p, _U64, _U64, _P, _P, _P, ctypes.c_char_p,
                                    _U64, _P]),
    "ctsm_csm1_header": (_I, [ctypes.c_char_p, ctypes.POINTER(_U64), ctypes.POINTER(_U64),
                              ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
    "ctsm_read_csm1_device": (_I, [_P, ctypes.c_char_p, _P, _P, _P, _P, _P]),
    "ctsm_write_ctt1": (_I, [ctypes.c_char_p, _P, _I, _P]),
    "ctsm_ctt1_header": (_I, [ctypes.c_char_p, _P, ctypes.POINTER(_I)]),
    "ctsm_read_ctt1": (_I, [ctypes.c_char_p, _P, _U64]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Loads the CUDA library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().ctsm_last_error().decode(errors="replace")
        if status == 100:
            raise CtsmError("CudaError", msg)
        raise CtsmError.from_status(status, msg.split(": ", 1)[-1])


def launch_count() -> int:
    return int(lib().ctsm_launch_count())
