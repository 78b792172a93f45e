"""ctypes access to the reference library itself (oracle/_ref/libfmtgp_ref.so).

TEST INFRASTRUCTURE: the parity checker and the CPU baseline.  Built from the
unmodified reference sources by ``make -C oracle ref`` (needs /root/reference,
i.e. this container; the built .so travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from paper_2603_16014_b200.designs import Design, Hyper

from ._cstructs import CDesign, CHyper, dptr, make_cdesign, make_chyper

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libfmtgp_ref.so")
# The same extern "C" shim and the reference's own gp_core / cubature, but with fast_gram.cpp
# replaced by the B200 drop-in (paper_2603_16014_b200/seam/fast_gram_b200.cpp): `make -C oracle seam`.
SEAM_PATH = os.path.join(HERE, "_ref", "libfmtgp_seam.so")


class RefError(RuntimeError):
    pass


class RefSchurBreakdown(RefError):
    pass


_lib = None
_libs = {}


def available() -> bool:
    return os.path.exists(LIB_PATH)


def seam_available() -> bool:
    return os.path.exists(SEAM_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference oracle not built: {LIB_PATH} (run make -C oracle ref)")
        _lib = _load(LIB_PATH)
    return _lib


def seam_lib():
    """The reference's gp_core / cubature over the B200 fast_gram drop-in."""
    if not seam_available():
        raise RefError(f"seam library not built: {SEAM_PATH} (run make -C oracle seam)")
    return _load(SEAM_PATH)


def _load(path):
    if path not in _libs:
        L = C.CDLL(path)
        P, D = C.POINTER(CDesign), C.POINTER(CHyper)
        dp = C.POINTER(C.c_double)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rand_u64.restype = C.c_uint64
        L.ref_rand_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_normal.restype = C.c_double
        L.ref_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_bit_reverse.restype = C.c_uint64
        L.ref_bit_reverse.argtypes = [C.c_uint64, C.c_int]
        L.ref_fwht.argtypes = [dp, C.c_size_t]
        L.ref_fft_bitrev.argtypes = [dp, C.c_size_t]
        L.ref_fft_bitrev_inv.argtypes = [dp, C.c_size_t]
        L.ref_si_bernoulli_1d.restype = C.c_double
        L.ref_si_bernoulli_1d.argtypes = [C.c_double, C.c_double, C.c_int]
        L.ref_dsi_order_1d.restype = C.c_double
        L.ref_dsi_order_1d.argtypes = [C.c_int, C.c_double, C.c_double]
        L.ref_design_points.argtypes = [P, dp]
        L.ref_build_spectrum.argtypes = [P, D, dp, dp]
        L.ref_invert_solve.argtypes = [P, D, dp, dp, dp, dp, dp, dp]
        L.ref_pi_h.argtypes = [P, D, dp, dp, dp]
        L.ref_problem_y.argtypes = [P, C.c_char_p, C.POINTER(C.c_int), C.c_double, C.c_uint64, dp]
        L.ref_problem_eval.argtypes = [C.c_char_p, C.c_int, C.c_int, dp, C.c_size_t, dp]
        L.ref_model_create.restype = C.c_void_p
        L.ref_model_create.argtypes = [P, D, dp]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_set_hyper.argtypes = [C.c_void_p, P, D]
        L.ref_model_loss.argtypes = [C.c_void_p, C.c_int, dp]
        L.ref_model_state.argtypes = [C.c_void_p, dp, dp, dp, C.POINTER(C.c_int)]
        L.ref_model_posterior_mean.argtypes = [C.c_void_p, C.c_int, dp, C.c_size_t, dp]
        L.ref_model_posterior_cov.argtypes = [C.c_void_p, C.c_int, dp, C.c_int, dp, dp]
        L.ref_model_cubature.argtypes = [C.c_void_p, dp, dp]
        L.ref_model_single_cubature.argtypes = [C.c_void_p, dp, dp]
        L.ref_model_fit.argtypes = [C.c_void_p, C.c_int, dp, dp]
        L.ref_model_fit_timed.argtypes = [C.c_void_p, C.c_int, dp, dp, dp, C.POINTER(C.c_int)]
        _libs[path] = L
    return _libs[path]


def _check(rc: int, L=None):
    if rc == 0:
        return
    msg = (L or lib()).ref_last_error().decode()
    if rc == 2:
        raise RefSchurBreakdown(msg)
    raise RefError(msg)


def fwht(a: np.ndarray) -> np.ndarray:
    a = np.array(a, dtype=np.float64)
    _check(lib().ref_fwht(dptr(a), a.size))
    return a


def fft_bitrev(a: np.ndarray, inverse: bool = False) -> np.ndarray:
    z = np.array(a, dtype=np.complex128)
    buf = z.view(np.float64)
    f = lib().ref_fft_bitrev_inv if inverse else lib().ref_fft_bitrev
    _check(f(dptr(buf), z.size))
    return z


def si_bernoulli_1d(x: float, xp: float, alpha: int) -> float:
    return lib().ref_si_bernoulli_1d(x, xp, alpha)


def dsi_order_1d(alpha: int, x: float, xp: float) -> float:
    return lib().ref_dsi_order_1d(alpha, x, xp)


def design_points(dz: Design) -> np.ndarray:
    cd, keep = make_cdesign(dz)
    out = np.empty((dz.N, dz.d))
    _check(lib().ref_design_points(C.byref(cd), dptr(out)))
    return out


def build_spectrum(dz: Design, hp: Hyper, seam: bool = False):
    """List of complex vectors, pairs (l<=lp) row by row (fast_gram.cpp:35-40)."""
    L = seam_lib() if seam else lib()
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    lens = [dz.n[l] for l in range(dz.L) for lp in range(l, dz.L)]
    re, im = np.empty(sum(lens)), np.empty(sum(lens))
    _check(L.ref_build_spectrum(C.byref(cd), C.byref(ch), dptr(re), dptr(im)), L)
    out, o = [], 0
    for n in lens:
        out.append(re[o:o + n] + 1j * im[o:o + n])
        o += n
    return out


def problem_y(dz: Design, name: str, users, noise: float, seed: int) -> np.ndarray:
    """Benchmark observations as the reference's bench makes them (bench.cpp:84-101)."""
    cd, k1 = make_cdesign(dz)
    u = (C.c_int * dz.L)(*[int(v) for v in users])
    y = np.empty(dz.N)
    _check(lib().ref_problem_y(C.byref(cd), name.encode(), u, float(noise), int(seed), dptr(y)))
    return y


def problem_eval(name: str, level: int, X: np.ndarray) -> np.ndarray:
    """The reference's problem functions at the rows of X (problems.cpp)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty(X.shape[0])
    _check(lib().ref_problem_eval(name.encode(), int(level), X.shape[1], dptr(X), X.shape[0], dptr(out)))
    return out


def pi_h(dz: Design, hp: Hyper, seam: bool = False):
    """(Pi [L, L], H [L, r] complex) of extract_pi_h (fast_gram.cpp:311-335)."""
    L = seam_lib() if seam else lib()
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    r = dz.N // dz.n[dz.L - 1]
    Pi, hr, hi = np.empty((dz.L, dz.L)), np.empty((dz.L, r)), np.empty((dz.L, r))
    _check(L.ref_pi_h(C.byref(cd), C.byref(ch), dptr(Pi), dptr(hr), dptr(hi)), L)
    return Pi, hr + 1j * hi


def invert_solve(dz: Design, hp: Hyper, b: np.ndarray, seam: bool = False, trace: bool = True):
    """(x = K^-1 b, K b, logdet, trace(K^-1) or None, Pi) through the reference seam."""
    L = seam_lib() if seam else lib()
    cd, k1 = make_cdesign(dz)
    ch, k2 = make_chyper(hp)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x, kb = np.empty(dz.N), np.empty(dz.N)
    logdet, tr = C.c_double(), C.c_double()
    Pi = np.empty((dz.L, dz.L))
    _check(L.ref_invert_solve(C.byref(cd), C.byref(ch), dptr(b), dptr(x), dptr(kb), C.byref(logdet),
                              C.byref(tr) if trace else None, dptr(Pi)), L)
    return x, kb, logdet.value, (tr.value if trace else None), Pi


class Model:
    """GpModel (gp_core.hpp:32-56) on the reference library."""

    def __init__(self, dz: Design, hp: Hyper, y: np.ndarray, seam: bool = False):
        self.dz = dz
        self.L = seam_lib() if seam else lib()
        self._cd, self._k1 = make_cdesign(dz)
        ch, k2 = make_chyper(hp)
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        self.h = self.L.ref_model_create(C.byref(self._cd), C.byref(ch), dptr(self.y))
        if not self.h:
            raise RefError(self.L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and getattr(self, "L", None) is not None:
            self.L.ref_model_free(self.h)
            self.h = None

    def set_hyper(self, hp: Hyper):
        ch, k2 = make_chyper(hp)
        _check(self.L.ref_model_set_hyper(self.h, C.byref(self._cd), C.byref(ch)), self.L)

    def loss(self, kind: int = 0) -> float:
        v = C.c_double()
        _check(self.L.ref_model_loss(self.h, kind, C.byref(v)), self.L)
        return v.value

    def state(self):
        L, N = self.dz.L, self.dz.N
        logdet = C.c_double()
        tau, c = np.empty(L), np.empty(N)
        esc = C.c_int()
        _check(self.L.ref_model_state(self.h, C.byref(logdet), dptr(tau), dptr(c), C.byref(esc)), self.L)
        return dict(logdet=logdet.value, tau=tau, c=c, escalations=esc.value)

    def posterior_mean(self, task: int, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float64)
        out = np.empty(X.shape[0])
        _check(self.L.ref_model_posterior_mean(self.h, task, dptr(X), X.shape[0], dptr(out)), self.L)
        return out

    def posterior_cov(self, task: int, x: np.ndarray, task2: int, xp: np.ndarray) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        xp = np.ascontiguousarray(xp, dtype=np.float64)
        v = C.c_double()
        _check(self.L.ref_model_posterior_cov(self.h, task, dptr(x), task2, dptr(xp), C.byref(v)), self.L)
        return v.value

    def cubature(self):
        L = self.dz.L
        mu, S = np.empty(L), np.empty((L, L))
        _check(self.L.ref_model_cubature(self.h, dptr(mu), dptr(S)), self.L)
        return mu, S

    def fit(self, steps: int):
        trace = np.empty(max(steps, 1))
        fl = C.c_double()
        _check(self.L.ref_model_fit(self.h, steps, C.byref(fl), dptr(trace)), self.L)
        return fl.value, trace[:steps]


def fit_timed(model: "Model", steps: int):
    """The reference's own fit (gp_core.cpp:317-382) with its own per-step timer
    (FitReport::step_seconds): returns (step_seconds[steps], n_params, loss_trace)."""
    trace, secs = np.empty(max(steps, 1)), np.empty(max(steps, 1))
    fl, npar = C.c_double(), C.c_int()
    _check(model.L.ref_model_fit_timed(model.h, steps, C.byref(fl), dptr(trace), dptr(secs), C.byref(npar)), model.L)
    return secs[:steps].copy(), npar.value, trace[:steps].copy()


def nll_fd_grad(dz: Design, hp: Hyper, y: np.ndarray, h_rel: float = 1e-5, richardson: bool = True):
    """Central-FD gradient of the reference NMLL w.r.t. (eta, B, t, gamma) — the
    reference's only gradient (gp_core.cpp:341-351), here on the natural (not log)
    parameters and optionally Richardson-extrapolated for a tighter check."""
    model = Model(dz, hp, y)

    def f(h):
        model.set_hyper(h)
        return model.loss(0)

    base = f(hp)

    def d_along(get, put):
        x0 = get(hp)
        step = h_rel * max(1.0, abs(x0))

        def cd(s):
            return (f(put(hp, x0 + s)) - f(put(hp, x0 - s))) / (2 * s)

        g1 = cd(step)
        if not richardson:
            return g1
        g2 = cd(step / 2)
        return (4 * g2 - g1) / 3

    def setter(field, idx):
        def get(h):
            return float(getattr(h, field)[idx])

        def put(h, v):
            arr = np.array(getattr(h, field), dtype=np.float64, copy=True)
            arr[idx] = v
            return h.replace(**{field: arr})

        return get, put

    g_eta = np.array([d_along(*setter("eta", j)) for j in range(dz.d)])
    g_B = np.array([[d_along(*setter("B", (l, k))) for k in range(hp.B.shape[1])] for l in range(dz.L)])
    g_t = np.array([d_along(*setter("t", l)) for l in range(dz.L)])
    g_gamma = d_along(lambda h: h.gamma, lambda h, v: h.replace(gamma=v))
    return dict(nll=base, eta=g_eta, B=g_B, t=g_t, gamma=g_gamma)
