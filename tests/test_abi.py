"""The C-ABI library loads and exports every entry point include/ctsm_b200.h
declares (no GPU needed: only symbol resolution, no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2511_12235_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ctsm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(ctsm_\w+)\s*\(", src, re.M)))


def test_header_declares_the_api():
    names = declared_functions()
    for must in ("ctsm_create", "ctsm_csr_count", "ctsm_csr_fill", "ctsm_spmv", "ctsm_spmv_t",
                 "ctsm_fwd_mf", "ctsm_bwd_mf", "ctsm_sirt"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    names = set(declared_functions())
    bound = set(_lib.SIGNATURES) | {"ctsm_bench_dfma"}
    assert names <= bound, names - bound


def test_no_cpu_fallback_symbols():
    """The product library links no oracle code."""
    L = ctypes.CDLL(_lib.LIB_PATH)
    for n in ("ref_build_system_matrix", "orc_crm_eval", "ref_forward_project_matrix_free"):
        assert not hasattr(L, n)


def test_errors_without_gpu_are_loud():
    """Without a device the API raises instead of computing on the CPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    h = ctypes.c_void_p()
    st = _lib.lib().ctsm_create(0, ctypes.byref(h))
    assert st != 0
