"""ctypes access to our C restatement of the reference path (oracle/fmtgp_oracle.c).

TEST INFRASTRUCTURE: checker and fallback CPU baseline.  Built by ``make -C oracle port``
(gcc only, no reference sources needed, so it also builds on the GPU box)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2603_16014_b200.designs import Design, Hyper

from ._cstructs import CDesign, CHyper, dptr, make_cdesign, make_chyper

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libfmtgp_oracle.so")


class PortError(RuntimeError):
    pass


class PortSchurBreakdown(PortError):
    pass


class COrcFit(C.Structure):
    _fields_ = [("nll", C.c_double), ("logdet", C.c_double), ("quad", C.c_double), ("tau", C.c_double * 8)]


_lib = None


def ensure_built():
    src = os.path.join(HERE, "fmtgp_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return lib()


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PortError(f"oracle port not built: {LIB_PATH}")
        L = C.CDLL(LIB_PATH)
        P, D = C.POINTER(CDesign), C.POINTER(CHyper)
        dp = C.POINTER(C.c_double)
        L.orc_last_error.restype = C.c_char_p
        L.orc_rand_u64.restype = C.c_uint64
        L.orc_rand_u64.argtypes = [C.c_uint64] * 3
        L.orc_normal.restype = C.c_double
        L.orc_normal.argtypes = [C.c_uint64] * 3
        L.orc_bit_reverse.restype = C.c_uint64
        L.orc_bit_reverse.argtypes = [C.c_uint64, C.c_int]
        L.orc_fwht.argtypes = [dp, C.c_size_t]
        L.orc_fft_bitrev.argtypes = [dp, C.c_size_t]
        L.orc_fft_bitrev_inv.argtypes = [dp, C.c_size_t]
        L.orc_si_bernoulli_1d.restype = C.c_double
        L.orc_si_bernoulli_1d.argtypes = [C.c_double, C.c_double, C.c_int]
        L.orc_dsi_order_1d.restype = C.c_double
        L.orc_dsi_order_1d.argtypes = [C.c_int, C.c_double, C.c_double]
        L.orc_design_points.argtypes = [P, dp]
        L.orc_build_spectrum.argtypes = [P, D, dp, dp]
        L.orc_invert_solve.argtypes = [P, D, dp, dp, dp, dp, dp, dp]
        L.orc_fit.argtypes = [P, D, dp, C.POINTER(COrcFit), dp]
        L.orc_posterior_mean.argtypes = [P, D, dp, C.c_int, dp, C.c_size_t, dp]
        L.orc_posterior_var.argtypes = [P, D, dp, C.c_int, dp, C.c_size_t, dp]
        L.orc_cubature.argtypes = [P, D, dp, dp, dp]
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 2:
        raise PortSchurBreakdown(msg)
    raise PortError(msg)


def fwht(a):
    a = np.array(a, dtype=np.float64)
    _check(lib().orc_fwht(dptr(a), a.size))
    return a


def fft_bitrev(a, inverse=False):
    z = np.array(a, dtype=np.complex128)
    f = lib().orc_fft_bitrev_inv if inverse else lib().orc_fft_bitrev
    _check(f(dptr(z.view(np.float64)), z.size))
    return z


def si_bernoulli_1d(x, xp, alpha):
    return lib().orc_si_bernoulli_1d(x, xp, alpha)


def dsi_order_1d(alpha, x, xp):
    return lib().orc_dsi_order_1d(alpha, x, xp)


def design_points(dz: Design):
    cd, k = make_cdesign(dz)
    out = np.empty((dz.N, dz.d))
    _check(lib().orc_design_points(C.byref(cd), dptr(out)))
    return out


def build_spectrum(dz: Design, hp: Hyper):
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    lens = [dz.n[l] for l in range(dz.L) for lp in range(l, dz.L)]
    re, im = np.empty(sum(lens)), np.empty(sum(lens))
    _check(lib().orc_build_spectrum(C.byref(cd), C.byref(ch), dptr(re), dptr(im)))
    out, o = [], 0
    for n in lens:
        out.append(re[o:o + n] + 1j * im[o:o + n])
        o += n
    return out


def invert_solve(dz: Design, hp: Hyper, b):
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x, kb = np.empty(dz.N), np.empty(dz.N)
    ld, tr = C.c_double(), C.c_double()
    Pi = np.empty((dz.L, dz.L))
    _check(lib().orc_invert_solve(C.byref(cd), C.byref(ch), dptr(b), dptr(x), dptr(kb), C.byref(ld), C.byref(tr),
                                  dptr(Pi)))
    return x, kb, ld.value, tr.value, Pi


def fit(dz: Design, hp: Hyper, y):
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    y = np.ascontiguousarray(y, dtype=np.float64)
    f = COrcFit()
    c = np.empty(dz.N)
    _check(lib().orc_fit(C.byref(cd), C.byref(ch), dptr(y), C.byref(f), dptr(c)))
    return dict(nll=f.nll, logdet=f.logdet, quad=f.quad, tau=np.array(f.tau[:dz.L]), c=c)


def posterior_mean(dz, hp, y, task, X):
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    y = np.ascontiguousarray(y, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty(X.shape[0])
    _check(lib().orc_posterior_mean(C.byref(cd), C.byref(ch), dptr(y), task, dptr(X), X.shape[0], dptr(out)))
    return out


def posterior_var(dz, hp, y, task, X):
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    y = np.ascontiguousarray(y, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty(X.shape[0])
    _check(lib().orc_posterior_var(C.byref(cd), C.byref(ch), dptr(y), task, dptr(X), X.shape[0], dptr(out)))
    return out


def cubature(dz, hp, y):
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    y = np.ascontiguousarray(y, dtype=np.float64)
    mu, S = np.empty(dz.L), np.empty((dz.L, dz.L))
    _check(lib().orc_cubature(C.byref(cd), C.byref(ch), dptr(y), dptr(mu), dptr(S)))
    return mu, S
