"""ctypes mirrors of the design / hyperparameter structs shared by oracle/_ref
(ref_capi.cpp RefDesign/RefHyper) and oracle/fmtgp_oracle.h (OrcDesign/OrcHyper).
TEST INFRASTRUCTURE."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2603_16014_b200.designs import LATTICE, Design, Hyper

_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class CDesign(C.Structure):
    _fields_ = [("kind", C.c_int), ("d", C.c_int), ("L", C.c_int), ("m", _ip), ("g", _u64p),
                ("n_max", C.c_uint64), ("columns", _u64p), ("m_cols", C.c_int), ("shift_bits", _u64p)]


class CHyper(C.Structure):
    _fields_ = [("gamma", C.c_double), ("eta", _dp), ("si_alpha", C.c_int), ("b", C.c_double * 4),
                ("B", _dp), ("s", C.c_int), ("t", _dp), ("xi", _dp)]


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def make_cdesign(dz: Design):
    keep = []
    m = np.ascontiguousarray(dz.m, dtype=np.int32)
    sb = np.ascontiguousarray(dz.shift_bits, dtype=np.uint64)
    keep += [m, sb]
    cd = CDesign(kind=dz.kind, d=dz.d, L=dz.L, m=m.ctypes.data_as(_ip), shift_bits=sb.ctypes.data_as(_u64p))
    if dz.kind == LATTICE:
        g = np.ascontiguousarray(dz.g, dtype=np.uint64)
        keep.append(g)
        cd.g = g.ctypes.data_as(_u64p)
        cd.n_max = dz.n_max
    else:
        cols = np.ascontiguousarray(dz.columns, dtype=np.uint64)
        keep.append(cols)
        cd.columns = cols.ctypes.data_as(_u64p)
        cd.m_cols = cols.shape[1]
    return cd, keep


def make_chyper(hp: Hyper):
    eta = np.ascontiguousarray(hp.eta, dtype=np.float64)
    B = np.ascontiguousarray(hp.B, dtype=np.float64)
    t = np.ascontiguousarray(hp.t, dtype=np.float64)
    xi = np.ascontiguousarray(hp.xi, dtype=np.float64)
    ch = CHyper(gamma=hp.gamma, eta=dptr(eta), si_alpha=hp.si_alpha, b=(C.c_double * 4)(*hp.b), B=dptr(B),
                s=B.shape[1], t=dptr(t), xi=dptr(xi))
    return ch, [eta, B, t, xi]
