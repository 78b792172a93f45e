"""Host-side mirror of the reference's fast-Gram seam and GpModel hot path, on the B200
C ABI (include/fastmtgp_b200.h).

Reference interface followed (names, argument meaning, error behaviour):
  fast_gram.hpp:34-70  build_spectrum / invert_and_logdet / solve / extract_pi_h /
                       trace_inverse / gram_matvec  (SchurBreakdown vs FastMtgpError)
  gp_core.hpp:46-83    refresh + loss_value (NMLL), posterior_mean_batch,
                       posterior_cov (variance), multitask_cubature
plus ``nll_grad``: the analytic hyperparameter gradient replacing the reference's
central finite differences (gp_core.cpp:341-351).

Inputs are in the reference's INTERNAL task order (descending n) — what the fast_gram
functions take; GpModel's user<->internal mapping is the caller's (gp_core.cpp:19-32).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import CDesign, CHyper, CResult, FastMtgpError, SchurBreakdown, Unsupported, check, dptr  # noqa: F401
from .designs import LATTICE, Design, Hyper


def _cdesign(dz: Design):
    keep = [np.ascontiguousarray(dz.m, dtype=np.int32), np.ascontiguousarray(dz.shift_bits, dtype=np.uint64)]
    cd = CDesign(kind=dz.kind, d=dz.d, L=dz.L, m=keep[0].ctypes.data_as(_lib._ip),
                 shift_bits=keep[1].ctypes.data_as(_lib._u64p))
    if dz.kind == LATTICE:
        g = np.ascontiguousarray(dz.g, dtype=np.uint64)
        keep.append(g)
        cd.g = g.ctypes.data_as(_lib._u64p)
        cd.n_max = int(dz.n_max)
    else:
        cols = np.ascontiguousarray(dz.columns, dtype=np.uint64)
        keep.append(cols)
        cd.columns = cols.ctypes.data_as(_lib._u64p)
        cd.m_cols = int(cols.shape[1])
    return cd, keep


def _chyper(hp: Hyper):
    eta = np.ascontiguousarray(hp.eta, dtype=np.float64)
    B = np.ascontiguousarray(hp.B, dtype=np.float64)
    t = np.ascontiguousarray(hp.t, dtype=np.float64)
    xi = np.ascontiguousarray(hp.xi, dtype=np.float64)
    ch = CHyper(gamma=float(hp.gamma), eta=dptr(eta), si_alpha=int(hp.si_alpha), b=(C.c_double * 4)(*hp.b),
                B=dptr(B), s=int(B.shape[1]), t=dptr(t), xi=dptr(xi))
    return ch, (eta, B, t, xi)


# double offsets of the CResult arrays: one np.frombuffer view instead of per-field ctypes slicing
# (halves the Python cost of returning a result, which sits inside every timed fit)
_ROFF = {f[0]: getattr(CResult, f[0]).offset // 8 for f in CResult._fields_[:10]}


def _result(r: CResult, dz: Design, hp: Hyper) -> Dict:
    L, d, s = dz.L, dz.d, hp.B.shape[1]
    v = np.frombuffer(r, dtype=np.float64, count=_ROFF["xi_scale"] + 1)
    o = _ROFF
    return dict(nll=r.nll, logdet=r.logdet, quad=r.quad, dgamma=r.dgamma,
                deta=v[o["deta"]:o["deta"] + d].copy(), dR=v[o["dR"]:o["dR"] + L * L].reshape(L, L).copy(),
                dB=v[o["dB"]:o["dB"] + L * s].reshape(L, s).copy(), dt=v[o["dt"]:o["dt"] + L].copy(),
                tau=v[o["tau"]:o["tau"] + L].copy(), xi_scale=r.xi_scale, escalations=r.escalations, status=r.status)


def unpack_theta(theta: np.ndarray, like: Hyper, digital: bool) -> Hyper:
    """ParamPack::unpack (gp_core.cpp:289-303): log gamma, log eta, B, log t, [log b]."""
    d, (L, s) = like.eta.size, like.B.shape
    k = 0
    gamma = float(np.exp(theta[k])); k += 1
    eta = np.exp(theta[k:k + d]); k += d
    B = np.array(theta[k:k + L * s]).reshape(L, s); k += L * s
    t = np.exp(theta[k:k + L]); k += L
    b = tuple(np.exp(theta[k:k + 4])) if digital else like.b
    return Hyper(gamma=gamma, eta=eta, B=B, t=t, xi=like.xi.copy(), si_alpha=like.si_alpha, b=b)


class Model:
    """Device-resident design + observations + workspace (one per GPU / dataset)."""

    def __init__(self, design: Design, device: int = 0, max_candidates: int = 1):
        self.lib = _lib.load()
        self.design = design
        self._cd, self._keep = _cdesign(design)
        h = C.c_void_p()
        check(self.lib.fmtgp_model_create(C.byref(self._cd), device, max_candidates, C.byref(h)))
        self.h = h
        self.hyper: Optional[Hyper] = None

    def close(self):
        if getattr(self, "h", None):
            self.lib.fmtgp_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- data
    def set_y(self, y: np.ndarray):
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.shape != (self.design.N,):
            raise FastMtgpError("make_model: observation size mismatch")
        check(self.lib.fmtgp_model_set_y(self.h, dptr(y)))

    def set_y_device(self, ptr: int):
        check(self.lib.fmtgp_model_set_y_device(self.h, C.c_void_p(ptr)))

    @property
    def stream(self) -> int:
        return self.lib.fmtgp_model_stream(self.h) or 0

    # -- fast_gram.hpp seam
    def build_spectrum(self, hp: Hyper):
        ch, keep = _chyper(hp)
        check(self.lib.fmtgp_build_spectrum(self.h, C.byref(ch)))
        self.hyper = hp

    def spectrum(self, l: int, lp: int) -> np.ndarray:
        n = self.design.n[l]
        re, im = np.empty(n), np.empty(n)
        check(self.lib.fmtgp_spectrum_read(self.h, l, lp, dptr(re), dptr(im)))
        return re + 1j * im

    def invert_and_logdet(self) -> float:
        v = C.c_double()
        check(self.lib.fmtgp_invert_and_logdet(self.h, C.byref(v)))
        return v.value

    def solve(self, b: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (self.design.N,):
            raise FastMtgpError("solve: length mismatch")
        x = np.empty_like(b)
        check(self.lib.fmtgp_solve(self.h, dptr(b), dptr(x)))
        return x

    def gram_matvec(self, b: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (self.design.N,):
            raise FastMtgpError("gram_matvec: length mismatch")
        x = np.empty_like(b)
        check(self.lib.fmtgp_gram_matvec(self.h, dptr(b), dptr(x)))
        return x

    def extract_pi(self) -> np.ndarray:
        L = self.design.L
        Pi = np.empty((L, L))
        check(self.lib.fmtgp_extract_pi(self.h, dptr(Pi)))
        return Pi

    def problem_y(self, name: str, user_of_internal, noise: float = 0.0, seed: int = 0) -> np.ndarray:
        """Benchmark observations computed on the device at this design's points (bench.cpp:84-101:
        level user + 1, noise * rng::normal(seed, 0x401 + user, i)); sets them as y and returns them."""
        u = np.ascontiguousarray(user_of_internal, dtype=np.int32)
        y = np.empty(self.design.N)
        check(self.lib.fmtgp_model_problem_y(self.h, name.encode(), u.ctypes.data_as(C.POINTER(C.c_int)),
                                             float(noise), int(seed), dptr(y)))
        return y

    def extract_pi_h(self):
        """(Pi [L, L], H [L, r] complex) of extract_pi_h (fast_gram.cpp:311-335), r = N / n_{L-1}."""
        L = self.design.L
        r = self.design.N // self.design.n[L - 1]
        Pi = self.extract_pi()
        hr, hi = np.empty((L, r)), np.empty((L, r))
        check(self.lib.fmtgp_extract_h(self.h, dptr(hr), dptr(hi)))
        return Pi, hr + 1j * hi

    def trace_inverse(self) -> float:
        v = C.c_double()
        check(self.lib.fmtgp_trace_inverse(self.h, C.byref(v)))
        return v.value

    # -- gp_core hot path
    def _hyper_struct(self, hp: Hyper):
        """CHyper for hp, reused while hp and its arrays are the same objects (the struct points
        at the arrays' buffers, so in-place edits are seen)."""
        key = (id(hp), id(hp.eta), id(hp.B), id(hp.t), id(hp.xi), hp.gamma, hp.si_alpha, tuple(hp.b))
        cached = getattr(self, "_hcache", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        ch, keep = _chyper(hp)
        self._hcache = (key, ch, keep)
        return ch

    def nll(self, hp: Hyper, grad: bool = True) -> Dict:
        """refresh + loss_value (NMLL) with escalation, plus the analytic gradient."""
        ch = self._hyper_struct(hp)
        r = CResult()
        check(self.lib.fmtgp_nll(self.h, C.byref(ch), int(grad), C.byref(r)))
        self.hyper = hp
        return _result(r, self.design, hp)

    def gcv(self, hp: Hyper) -> Dict:
        """GCV loss ||c||^2 / (tr K^-1)^2 (loss_value with LossKind::gcv, gp_core.cpp:213-226);
        equal sample sizes."""
        ch = self._hyper_struct(hp)
        loss, num, tr = C.c_double(), C.c_double(), C.c_double()
        check(self.lib.fmtgp_gcv(self.h, C.byref(ch), C.byref(loss), C.byref(num), C.byref(tr)))
        self.hyper = hp
        return {"gcv": loss.value, "num": num.value, "trace": tr.value}

    def nll_batch(self, hps: Sequence[Hyper], grad: bool = True) -> List[Dict]:
        n = len(hps)
        arr = (CHyper * n)()
        keeps = []
        for i, hp in enumerate(hps):
            ch, keep = _chyper(hp)
            arr[i] = ch
            keeps.append(keep)
        res = (CResult * n)()
        check(self.lib.fmtgp_nll_batch(self.h, n, arr, int(grad), res))
        return [_result(res[i], self.design, hps[i]) for i in range(n)]

    def fit(self, hp: Hyper, steps: int) -> Dict:
        """The reference's `fit` (iRprop- over ParamPack, gp_core.cpp:317-382) with the analytic
        gradient: one NLL+gradient evaluation per step.  Returns the best hyperparameters, the
        packed theta, the best-so-far loss trace and per-step seconds; the model is left
        refreshed at the best point."""
        ch, keep = _chyper(hp)
        n = C.c_int()
        check(self.lib.fmtgp_fit_param_count(self.h, int(hp.B.shape[1]), C.byref(n)))
        theta = np.empty(n.value)
        trace = np.empty(max(steps, 1))
        secs = np.empty(max(steps, 1))
        rep = _lib.CFitReport()
        check(self.lib.fmtgp_fit(self.h, C.byref(ch), int(steps), dptr(theta), dptr(trace), dptr(secs),
                                 C.byref(rep)))
        best = unpack_theta(theta, hp, self.design.kind == 1)
        self.hyper = best
        return dict(hyper=best, theta=theta, loss_trace=trace[:steps].copy(), step_seconds=secs[:steps].copy(),
                    final_loss=rep.final_loss, escalations=rep.escalations, tau=np.array(rep.tau[:self.design.L]))

    def coefficients(self) -> np.ndarray:
        c = np.empty(self.design.N)
        check(self.lib.fmtgp_coefficients(self.h, dptr(c)))
        return c

    def posterior_mean(self, task: int, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, self.design.d)
        out = np.empty(X.shape[0])
        check(self.lib.fmtgp_posterior_mean(self.h, task, dptr(X), X.shape[0], dptr(out)))
        return out

    def posterior_var(self, task: int, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, self.design.d)
        out = np.empty(X.shape[0])
        check(self.lib.fmtgp_posterior_var(self.h, task, dptr(X), X.shape[0], dptr(out)))
        return out

    def posterior_cov(self, task: int, X: np.ndarray, task2: int, Xp: np.ndarray) -> np.ndarray:
        """posterior_cov (gp_core.cpp:423-445) for the pairs (X[i], Xp[i]): K((task, x), (task2, x'))
        - k(x)^T K^-1 k(x'), both kernel columns on the device."""
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, self.design.d)
        Xp = np.ascontiguousarray(Xp, dtype=np.float64).reshape(-1, self.design.d)
        if X.shape != Xp.shape:
            raise ValueError("posterior_cov: X and Xp need the same shape")
        out = np.empty(X.shape[0])
        check(self.lib.fmtgp_posterior_cov(self.h, task, dptr(X), task2, dptr(Xp), X.shape[0], dptr(out)))
        return out

    def cubature(self):
        L = self.design.L
        mu, S = np.empty(L), np.empty((L, L))
        check(self.lib.fmtgp_cubature(self.h, dptr(mu), dptr(S)))
        return mu, S


    # -- measurement
    def bench_nll(self, hp: Hyper, iters: int, grad: bool = True, flush_bytes: int = 0):
        """(device ms per call [iters], mean host wall us per call) of `iters` fmtgp_nll calls
        looped in C (fmtgp_bench_nll): the evaluation without the interpreter between calls."""
        ch = self._hyper_struct(hp)
        ms = np.empty(iters)
        wall = C.c_double()
        check(self.lib.fmtgp_bench_nll(self.h, C.byref(ch), int(grad), int(iters), int(flush_bytes), dptr(ms),
                                       C.byref(wall)))
        return ms, wall.value

    def profile(self, on: bool = True):
        check(self.lib.fmtgp_profile_enable(self.h, int(on)))

    def profile_read(self) -> Dict[str, tuple]:
        """kernel name -> (total device ms, launches) since profile(True)."""
        out = {}
        i = 0
        buf = C.create_string_buffer(64)
        while True:
            ms, cnt = C.c_double(), C.c_int()
            rc = self.lib.fmtgp_profile_read(self.h, i, buf, 64, C.byref(ms), C.byref(cnt))
            if rc != _lib.OK:
                break
            out[buf.value.decode()] = (ms.value, cnt.value)
            i += 1
        return out


# ---- free-function spelling of the seam (fast_gram.hpp:34-70) ---------------------------

def build_spectrum(model: Model, hp: Hyper) -> Model:
    model.build_spectrum(hp)
    return model


def invert_and_logdet(model: Model) -> float:
    return model.invert_and_logdet()


def solve(model: Model, y: np.ndarray) -> np.ndarray:
    return model.solve(y)


def extract_pi_h(model: Model):
    return model.extract_pi_h()


def trace_inverse(model: Model) -> float:
    return model.trace_inverse()


def gram_matvec(model: Model, y: np.ndarray) -> np.ndarray:
    return model.gram_matvec(y)


# ---- benchmark problems (problems.cpp) on the device ---------------------------------------

PROBLEMS = {"rosenbrock": (2, 3), "ackley": (4, 2), "borehole": (8, 2), "elliptic": (16, 3)}  # name: (d, levels)


def problem_eval(name: str, level: int, X, device: int = 0) -> np.ndarray:
    """problem(level, x) at each row of X (eval_batch, problems.cpp:145-154), evaluated on the device."""
    if name not in PROBLEMS:
        raise FastMtgpError(f"unknown problem {name}")
    X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, PROBLEMS[name][0])
    out = np.empty(X.shape[0])
    check(_lib.load().fmtgp_problem_eval(name.encode(), int(level), dptr(X), X.shape[0], dptr(out), int(device)))
    return out
