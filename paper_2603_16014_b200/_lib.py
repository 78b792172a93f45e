"""ctypes binding of the CUDA library libfmtgp_b200.so (include/fastmtgp_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device is
usable, every call raises.  Status codes map onto the reference's exception types
(common.hpp:16-22): SchurBreakdown (retryable) and FastMtgpError (fatal).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FMTGP_LIB: a developer override for A/B runs of two builds of the same library (tools/r03_ab.sh)
LIB_PATH = os.environ.get("FMTGP_LIB") or os.path.join(HERE, "libfmtgp_b200.so")
SHARD_REC_LEN = 4 + 16 + 8 * 8 + 1 + 2 * 8  # FMTGP_SHARD_REC_LEN
MAX_D = 16
MAX_T = 8

OK, ERR_INVALID, ERR_SCHUR, ERR_NONREAL, ERR_CUDA, ERR_OOM, ERR_UNSUPPORTED = range(7)


class FastMtgpError(RuntimeError):
    """common.hpp:21 FastMtgpError."""


class SchurBreakdown(FastMtgpError):
    """common.hpp:16 SchurBreakdown (non-positive Schur pivot; escalate the nugget)."""


class CudaError(FastMtgpError):
    pass


class Unsupported(FastMtgpError):
    pass


_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class CDesign(C.Structure):
    _fields_ = [("kind", C.c_int), ("d", C.c_int), ("L", C.c_int), ("m", _ip), ("g", _u64p),
                ("n_max", C.c_uint64), ("columns", _u64p), ("m_cols", C.c_int), ("shift_bits", _u64p)]


class CHyper(C.Structure):
    _fields_ = [("gamma", C.c_double), ("eta", _dp), ("si_alpha", C.c_int), ("b", C.c_double * 4),
                ("B", _dp), ("s", C.c_int), ("t", _dp), ("xi", _dp)]


class CResult(C.Structure):
    _fields_ = [("nll", C.c_double), ("logdet", C.c_double), ("quad", C.c_double), ("dgamma", C.c_double),
                ("deta", C.c_double * MAX_D), ("dR", C.c_double * (MAX_T * MAX_T)),
                ("dB", C.c_double * (MAX_T * MAX_T)), ("dt", C.c_double * MAX_T), ("tau", C.c_double * MAX_T),
                ("xi_scale", C.c_double), ("escalations", C.c_int), ("status", C.c_int)]


class CFitReport(C.Structure):
    _fields_ = [("steps", C.c_int), ("n_params", C.c_int), ("escalations", C.c_int),
                ("final_loss", C.c_double), ("tau", C.c_double * MAX_T)]


_lib = None

_SIGS = {
    "fmtgp_last_error": (C.c_char_p, []),
    "fmtgp_abi_version": (C.c_int, []),
    "fmtgp_model_create": (C.c_int, [C.POINTER(CDesign), C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "fmtgp_model_destroy": (C.c_int, [C.c_void_p]),
    "fmtgp_model_set_y": (C.c_int, [C.c_void_p, _dp]),
    "fmtgp_model_set_y_device": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fmtgp_model_problem_y": (C.c_int, [C.c_void_p, C.c_char_p, _ip, C.c_double, C.c_uint64, _dp]),
    "fmtgp_problem_eval": (C.c_int, [C.c_char_p, C.c_int, _dp, C.c_uint64, _dp, C.c_int]),
    "fmtgp_model_stream": (C.c_void_p, [C.c_void_p]),
    "fmtgp_build_spectrum": (C.c_int, [C.c_void_p, C.POINTER(CHyper)]),
    "fmtgp_spectrum_read": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp, _dp]),
    "fmtgp_invert_and_logdet": (C.c_int, [C.c_void_p, _dp]),
    "fmtgp_solve": (C.c_int, [C.c_void_p, _dp, _dp]),
    "fmtgp_gram_matvec": (C.c_int, [C.c_void_p, _dp, _dp]),
    "fmtgp_extract_pi": (C.c_int, [C.c_void_p, _dp]),
    "fmtgp_trace_inverse": (C.c_int, [C.c_void_p, _dp]),
    "fmtgp_nll": (C.c_int, [C.c_void_p, C.POINTER(CHyper), C.c_int, C.POINTER(CResult)]),
    "fmtgp_nll_batch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(CHyper), C.c_int, C.POINTER(CResult)]),
    "fmtgp_coefficients": (C.c_int, [C.c_void_p, _dp]),
    "fmtgp_fit_param_count": (C.c_int, [C.c_void_p, C.c_int, _ip]),
    "fmtgp_fit": (C.c_int, [C.c_void_p, C.POINTER(CHyper), C.c_int, _dp, _dp, _dp, C.POINTER(CFitReport)]),
    "fmtgp_posterior_mean": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_int64, _dp]),
    "fmtgp_posterior_var": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_int64, _dp]),
    "fmtgp_posterior_cov": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_int, _dp, C.c_int64, _dp]),
    "fmtgp_extract_h": (C.c_int, [C.c_void_p, _dp, _dp]),
    "fmtgp_spectrum_read_range": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, _dp, _dp]),
    "fmtgp_cubature": (C.c_int, [C.c_void_p, _dp, _dp]),
    "fmtgp_gcv": (C.c_int, [C.c_void_p, C.POINTER(CHyper), _dp, _dp, _dp]),
    "fmtgp_shard_setup": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    "fmtgp_shard_begin": (C.c_int, [C.c_void_p, C.POINTER(CHyper), C.c_int, C.c_double, C.c_void_p]),
    "fmtgp_shard_mid": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fmtgp_shard_chunks": (C.c_int, [C.c_void_p, C.c_int]),
    "fmtgp_shard_begin_chunk": (C.c_int, [C.c_void_p, C.POINTER(CHyper), C.c_int, C.c_double, C.c_void_p, C.c_int]),
    "fmtgp_shard_mid_chunk": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "fmtgp_shard_end": (C.c_int, [C.c_void_p, C.c_void_p, _dp]),
    "fmtgp_shard_finish": (C.c_int, [C.c_void_p, C.POINTER(CHyper), _dp, C.c_int, C.c_double, C.c_int,
                                     C.POINTER(CResult)]),
    "fmtgp_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "fmtgp_bench_nll": (C.c_int, [C.c_void_p, C.POINTER(CHyper), C.c_int, C.c_int, C.c_size_t, _dp, _dp]),
    "fmtgp_profile_read": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_int, _dp, _ip]),
}

EXPORTED = sorted(_SIGS)


def load(path: str = LIB_PATH):
    """Load the CUDA library (no GPU needed to load; calls need one)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise FastMtgpError(f"CUDA library not built: {path} (run __graft_entry__.build())")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def check(rc: int):
    if rc == OK:
        return
    msg = load().fmtgp_last_error().decode(errors="replace")
    if rc == ERR_SCHUR:
        raise SchurBreakdown(msg)
    if rc == ERR_CUDA or rc == ERR_OOM:
        raise CudaError(msg)
    if rc == ERR_UNSUPPORTED:
        raise Unsupported(msg)
    raise FastMtgpError(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)
