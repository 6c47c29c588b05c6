"""ctypes binding of libocmg_b200.so (the C ABI in include/ocmg_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every device entry point raises.  ``build()`` compiles the library
in-tree with nvcc for sm_100a.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libocmg_b200.so")
# developer A/B builds (scripts/): load another build of the same CUDA library
LIB_PATH = os.environ.get("OCMG_LIB", LIB_PATH)
CSRC = os.path.join(HERE, "csrc")

OCMG_OK = 0
OCMG_E_ARG = -1
OCMG_E_CUDA = -2
OCMG_E_SINGULAR = -3
OCMG_E_STATE = -4

POISSON, STOKES = 0, 1
SMOOTHER_IDS = {"normal": 0, "lsgs": 1, "slsgs": 2, "cgs": 3, "vanka": 4}
GS_MODES = {"reference": 0, "wavefront": 1, "multicolour": 2}

# table sizes, mirrored from csrc/ocmg_p1.cuh and csrc/ocmg_wavefront.cuh
P1_TABLE_DOUBLES = 49 * 28 * 2 + 49 * 2 * 2
WF_TABLE_DOUBLES = 49 * 38


class SingularMatrixError(RuntimeError):
    """Raised when a dense factorization meets an exactly singular pivot
    (sparse.py:18-19)."""


class CycleConfigC(ctypes.Structure):
    _fields_ = [("cycle_w", ctypes.c_int), ("nu_pre", ctypes.c_int),
                ("nu_post", ctypes.c_int), ("smoother", ctypes.c_int),
                ("gs_mode", ctypes.c_int), ("tau", ctypes.c_double)]


_LIB = None

# (name, restype, argtypes) for every exported symbol; tests check that the
# library exports exactly what include/ocmg_b200.h declares
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_PP = ctypes.POINTER(ctypes.c_void_p)
SIGNATURES = {
    "ocmg_last_error": (ctypes.c_char_p, []),
    "ocmg_abi_version": (_I, []),
    "ocmg_device_sm_count": (_I, [ctypes.POINTER(_I)]),
    "ocmg_launch_count": (_I, [ctypes.POINTER(_I64)]),
    "ocmg_level_create_csr": (_I, [_I, _I64, _P, _P, _P, _P, _I, _P,
                                   ctypes.c_uint32, _I, _PP]),
    "ocmg_level_create_p1": (_I, [_I, _D, _P, _I64, _PP]),
    "ocmg_level_destroy": (_I, [_P]),
    "ocmg_level_n": (_I64, [_P]),
    "ocmg_level_nnz": (_I64, [_P]),
    "ocmg_residual": (_I, [_P, _P, _P, _P, _P]),
    "ocmg_ne_jacobi_sweep": (_I, [_P, _D, _P, _P, _P, _P,
                                  ctypes.POINTER(_I64)]),
    "ocmg_ne_gs_sweep": (_I, [_P, _I, _I, _P, _P, _P, ctypes.POINTER(_I64)]),
    "ocmg_ne_gs_sweep_into": (_I, [_P, _I, _I, _P, _P, _P, _P,
                                   ctypes.POINTER(_I64)]),
    "ocmg_ne_gs_sweep_strip": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P,
                                    ctypes.POINTER(_I64)]),
    "ocmg_residual_rows": (_I, [_P, _P, _P, _P, _I, _I, _P]),
    "ocmg_cgs_sweep": (_I, [_P, _I, _P, _P, _P, _P, ctypes.POINTER(_I64)]),
    "ocmg_level_set_alpha": (_I, [_P, _D]),
    "ocmg_level_set_vanka": (_I, [_P, _I64, _I, _P, _P, _P]),
    "ocmg_vanka_sweep": (_I, [_P, _D, _I, _P, _P, _P, ctypes.POINTER(_I64)]),
    "ocmg_restrict_rows": (_I, [_P, _P, _P, _I, _I, _P]),
    "ocmg_ne_jacobi_p_rows": (_I, [_P, _D, _P, _P, _I, _I, _P]),
    "ocmg_ne_jacobi_apply_rows": (_I, [_P, _P, _P, _P, _I, _I, _P]),
    "ocmg_prolong_add_rows": (_I, [_P, _P, _P, _I, _I, _P]),
    "ocmg_mean_project": (_I, [_P, _P, _P]),
    "ocmg_norm2": (_I, [_P, _P, _I, _P, _P]),
    "ocmg_transfer_create_csr": (_I, [_I64, _I64, _P, _P, _P, _PP]),
    "ocmg_transfer_create_p1": (_I, [_I, _I, _PP]),
    "ocmg_transfer_destroy": (_I, [_P]),
    "ocmg_restrict": (_I, [_P, _P, _P, _P]),
    "ocmg_prolong_add": (_I, [_P, _P, _P, _P]),
    "ocmg_coarse_create": (_I, [_I, _I64, _P, _P, _I64, _I64, _I64, _PP]),
    "ocmg_coarse_destroy": (_I, [_P]),
    "ocmg_coarse_solve": (_I, [_P, _P, _P, _P]),
    "ocmg_hierarchy_create": (_I, [_I, _P, _P, _P,
                                   ctypes.POINTER(CycleConfigC), _PP]),
    "ocmg_hierarchy_destroy": (_I, [_P]),
    "ocmg_cycle": (_I, [_P, _P, _P, _P]),
    "ocmg_coarse_correction": (_I, [_P, _I, _P, _P, _P]),
    "ocmg_hierarchy_collapsed_level": (_I, [_P, _P]),
    "ocmg_solve": (_I, [_P, _P, _P, _D, _I, _I, _P, ctypes.POINTER(_I),
                        _P]),
    "ocmg_solve_ex": (_I, [_P, _P, _P, _D, _I, _I, _D, _P,
                           ctypes.POINTER(_I), ctypes.POINTER(_I), _P]),
}


def build(force=False, verbose=False):
    """Compile libocmg_b200.so in-tree (nvcc, sm_100a)."""
    cmd = ["make", "-C", CSRC]
    if force:
        cmd.insert(1, "-B")
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libocmg_b200.so failed:\n" + out.stdout
                           + out.stderr)
    if verbose:
        print(out.stdout)
    return LIB_PATH


def load():
    """Load the library (once).  Raises if it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA path has no fallback; run "
                "paper_1502_03917_b200._lib.build() (or __graft_entry__."
                "build()) first")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def check(status):
    """Map a C status to the reference's exception types."""
    if status == OCMG_OK:
        return
    msg = load().ocmg_last_error().decode(errors="replace")
    if status == OCMG_E_ARG:
        raise ValueError(msg)
    if status == OCMG_E_SINGULAR:
        raise SingularMatrixError(msg)
    raise RuntimeError(f"ocmg_b200 error {status}: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def new_handle():
    return ctypes.c_void_p()


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("ocmg_b200 needs a CUDA device (B200); no CPU "
                           "fallback exists")
    load()


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dptr(t):
    """Device pointer of a contiguous fp64 CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not (t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def launch_count():
    """Kernels launched by the library so far (ocmg_launch_count)."""
    out = ctypes.c_int64()
    check(load().ocmg_launch_count(ctypes.byref(out)))
    return out.value


def hptr(a):
    """Host pointer of a contiguous numpy array."""
    return a.ctypes.data_as(ctypes.c_void_p)
