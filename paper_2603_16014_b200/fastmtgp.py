"""Python front-end with the surface of the reference's pybind module ``fastmtgp``
(/root/reference/proj/python/bindings.cpp:129-213) on the B200 C ABI, plus the model document
I/O of gp_core.cpp:447-508 (``to_json`` / ``from_json``).

    m = Model("si-lattice", d=4, n=[2**18, 2**16], seed=7, y=[y0, y1], loss="nmll", task_rank=1)
    m = Model.from_problem("ackley", "si-lattice", n=[2**18, 2**16], seed=7, noise=0.01)  # bench.cpp fit_trial
    rep = m.fit(10)              # iRprop- (gp_core.cpp:317-382) with the analytic gradient
    m.loss(); m.tau()            # loss_value / optimal_tau
    m.posterior_mean(0, x); m.posterior_mean_batch(1, X); m.posterior_cov(0, x, 1, xp)
    mu, Sigma = m.cubature()     # multitask_cubature (single-task formula when L = 1)
    m.l2_relative_error(u, X)    # held-out error against the problem (bench.cpp:159-170)
    doc = m.to_json(); m2 = Model.from_json(doc)

Task indices are USER indices (the reference's make_design sorts tasks by descending size and
keeps user <-> internal maps, ld_sequences.cpp:160-209; gp_core.cpp:19-32); this module maps
them onto the C ABI's internal order.  Deliberate differences, all raised loudly:
* designs: the reference's ``make_design(kind, d, m, seed)`` draws from its shipped generator
  tables (``default_lattice`` / ``default_digital``), which are not part of this repository.
  This module uses the seeded generators of ``designs.py`` (the BASELINE recipe: seeded odd
  lattice vectors / scrambled Sobol'-type nets) with the reference's task order and one shift
  stream per USER task.  Documents therefore carry the generator itself (key ``"generator"``) and
  round-trip exactly; a reference-written document (no generator) raises ``Unsupported``.
* ``"se-dense"`` (the reference's dense squared-exponential path) is not on the B200 fast path
  (out of scope): ``Unsupported``.
* ``fit`` with ``loss="gcv"``: ``Unsupported`` (the GPU fit loop optimises the NMLL; the GCV loss
  itself, equal or unequal n, is ``loss()``).
"""
from __future__ import annotations

import json
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import designs as dz_mod
from ._lib import Unsupported
from .designs import DIGITAL, LATTICE, Design, Hyper
from .fast_gram import PROBLEMS, problem_eval
from .fast_gram import Model as _GpuModel

KERNELS = {"si-lattice": LATTICE, "dsi-digital": DIGITAL}
_INIT_STREAM = 0xB011  # init_hyperparams' B stream (gp_core.cpp:169-185)
_TEST_STREAM = 0x7E57  # the benchmark's held-out set (bench.cpp:22, 155-157)


def _log2_exact(n: int) -> int:
    n = int(n)
    if n < 1 or n & (n - 1):
        raise ValueError("length must be a power of two")
    return n.bit_length() - 1


def _order(m_user: Sequence[int]) -> List[int]:
    """internal -> user: stable sort by descending size (ld_sequences.cpp:175-176)."""
    return sorted(range(len(m_user)), key=lambda u: -m_user[u])


def make_design(kind: int, d: int, m_user: Sequence[int], seed: int, m_cols: int = 32) -> (Design, List[int]):
    """(Design in internal order, internal_to_user) with the seeded generators of designs.py and
    one shift substream per user task (make_design's `stream = user task`, ld_sequences.cpp:192-199)."""
    i2u = _order(m_user)
    m = [int(m_user[u]) for u in i2u]
    if kind == LATTICE:
        stream = 0x5A1
        shifts = np.stack([dz_mod.bits53(seed, stream + u, np.arange(d)) for u in i2u])
        n_max = 1 << m[0]
        return Design(LATTICE, d, m, shifts, g=dz_mod.lattice_generator(d, n_max, seed), n_max=n_max), i2u
    cols = dz_mod.lms_scramble(dz_mod.sobol_type_columns(d, max(m_cols, m[0]), seed), seed)
    shifts = np.stack([dz_mod.bits53(seed, 0xD15 + u, np.arange(d)) for u in i2u])
    return Design(DIGITAL, d, m, shifts, columns=cols), i2u


def design_points(kind: str, d: int, n: Sequence[int], seed: int = 0) -> List[np.ndarray]:
    """Per-task point sets in USER order, each an n_u x d array (bindings.cpp design_points)."""
    k = {"lattice": LATTICE, "digital": DIGITAL}.get(kind)
    if k is None:
        raise ValueError("kind must be 'lattice' or 'digital'")
    design, i2u = make_design(k, d, [_log2_exact(v) for v in n], seed)
    out: List[Optional[np.ndarray]] = [None] * design.L
    for l, u in enumerate(i2u):
        out[u] = design.points(l)
    return out  # type: ignore[return-value]


def test_points(kernel: str, d: int, count: int, seed: int) -> np.ndarray:
    """The benchmark's held-out set (bench.cpp:155-157: shifted_points(kind, d, 0, count, seed,
    0x7E57)): the first `count` points of this module's generator for `seed` (count a power of two,
    at most the lattice's n_max) under the test-stream shift; count x d."""
    kind = KERNELS[kernel]
    m = _log2_exact(count)
    design, _ = make_design(kind, d, [m], seed)
    shifts = dz_mod.bits53(seed, _TEST_STREAM, np.arange(d)).reshape(1, d)
    if kind == LATTICE:
        t = Design(LATTICE, d, [m], shifts, g=design.g, n_max=design.n_max)
    else:
        t = Design(DIGITAL, d, [m], shifts, columns=design.columns)
    return t.points(0)


def optimal_weights(mu, Sigma, chi):
    """Task combination weights minimising the posterior MSE and that MSE (cubature.cpp:76-85)."""
    mu, Sigma, chi = (np.asarray(a, dtype=np.float64) for a in (mu, Sigma, chi))
    Minv_mu = np.linalg.solve(Sigma + np.outer(mu, mu), mu)
    target = float(chi @ mu)
    return target * Minv_mu, target * target * (1.0 - float(mu @ Minv_mu))


class Model:
    """GpModel behind the reference's pybind ``Model`` (bindings.cpp:35-123, 197-212)."""

    def __init__(self, kernel: str, d: int, n: Sequence[int], seed: int, y: Sequence[Sequence[float]],
                 loss: str = "nmll", task_rank: int = 1, jitter: float = 1e-8, device: int = 0,
                 _state: Optional[Dict] = None):
        if kernel == "se-dense":
            raise Unsupported("se-dense: the dense squared-exponential path is not on the B200 fast path")
        if kernel not in KERNELS:
            raise ValueError("kernel must be 'si-lattice', 'dsi-digital' or 'se-dense'")
        if loss not in ("nmll", "gcv"):
            raise ValueError("loss must be 'nmll' or 'gcv'")
        self.kernel, self.loss_kind, self.seed, self.d = kernel, loss, int(seed), int(d)
        m_user = [_log2_exact(v) for v in n]
        if len(y) != len(m_user):
            raise ValueError("make_model: observation task count mismatch")
        if _state is not None:
            self.design, self.i2u = _state["design"], _state["i2u"]
        else:
            self.design, self.i2u = make_design(KERNELS[kernel], d, m_user, seed)
        L = self.design.L
        self.y_user = [np.ascontiguousarray(v, dtype=np.float64) for v in y]
        for u in range(L):
            if self.y_user[u].size != (1 << m_user[u]):
                raise ValueError("make_model: observation size mismatch")
        if _state is not None and "hyper" in _state:
            self.hyper = _state["hyper"]
        else:  # init_hyperparams (gp_core.cpp:169-185), user order
            y_all = np.concatenate(self.y_user)
            s = int(task_rank)
            B = np.array([[0.1 * float(dz_mod.normal(self.seed, _INIT_STREAM, np.array([u * s + k]))[0])
                           for k in range(s)] for u in range(L)]).reshape(L, s)
            self.hyper = Hyper(gamma=max(float(np.var(y_all)), 1e-12), eta=np.ones(d), B=B, t=np.full(L, 0.1),
                               xi=np.full(L, float(jitter)), si_alpha=1, b=(1.0, 1.0, 1.0, 1.0))
        if _state is not None and "gpu" in _state:
            self.gpu = _state["gpu"]  # observations already on the device (from_problem)
        else:
            self.gpu = _GpuModel(self.design, device=device)
            self.gpu.set_y(np.concatenate([self.y_user[u] for u in self.i2u]))
        self._fresh = None

    @staticmethod
    def from_problem(problem: str, kernel: str, n: Sequence[int], seed: int = 0, noise: float = 0.0,
                     loss: str = "nmll", task_rank: int = 1, jitter: float = 1e-8, device: int = 0) -> "Model":
        """fit_trial's model (bench.cpp:84-107): the design for `seed`, observations of the problem's
        fidelity u + 1 for user task u plus noise * N(0, 1) (stream 0x401 + u) computed ON THE
        DEVICE at the design points (fmtgp_model_problem_y), init_hyperparams from them."""
        if problem not in PROBLEMS:
            raise ValueError(f"unknown problem {problem}")
        if kernel not in KERNELS:
            raise Unsupported(f"{kernel}: not on the B200 fast path") if kernel == "se-dense" else ValueError(kernel)
        d, levels = PROBLEMS[problem]
        m_user = [_log2_exact(v) for v in n]
        if len(m_user) > levels:
            raise ValueError("more tasks requested than the problem has fidelities")
        design, i2u = make_design(KERNELS[kernel], d, m_user, seed)
        gpu = _GpuModel(design, device=device)
        y_int = gpu.problem_y(problem, i2u, noise, seed)
        y_user: List[Optional[np.ndarray]] = [None] * design.L
        for l, u in enumerate(i2u):
            y_user[u] = y_int[design.offset[l]:design.offset[l + 1]]
        m = Model(kernel, d, n, seed, y_user, loss=loss, task_rank=task_rank, jitter=jitter, device=device,
                  _state={"design": design, "i2u": i2u, "gpu": gpu})
        m.problem = problem
        return m

    def l2_relative_error(self, task: int, X) -> float:
        """||mean - truth|| / ||truth|| over the rows of X, truth = the problem's fidelity task + 1
        on the device (l2_relative_error, bench.cpp:159-170)."""
        name = getattr(self, "problem", None)
        if name is None:
            raise ValueError("l2_relative_error: the model was not made from a problem")
        X = np.asarray(X, dtype=np.float64).reshape(-1, self.d)
        truth = problem_eval(name, task + 1, X)
        pred = np.asarray(self.posterior_mean_batch(task, X))
        return float(np.sqrt(np.sum((pred - truth) ** 2) / np.sum(truth * truth)))

    # -- user <-> internal
    def _internal(self, h: Hyper) -> Hyper:
        i = self.i2u
        return h.replace(B=h.B[i], t=h.t[i], xi=h.xi[i])

    def _user(self, h: Hyper) -> Hyper:
        inv = np.argsort(self.i2u)
        return h.replace(B=h.B[inv], t=h.t[inv], xi=h.xi[inv])

    def _uvec(self, v) -> np.ndarray:
        out = np.empty(self.design.L)
        out[self.i2u] = np.asarray(v)[: self.design.L]
        return out

    def _umat(self, A) -> np.ndarray:
        A = np.asarray(A)
        out = np.empty_like(A)
        out[np.ix_(self.i2u, self.i2u)] = A
        return out

    def _refresh(self):
        if self._fresh is None:
            self._fresh = self.gpu.nll(self._internal(self.hyper), grad=False)
        return self._fresh

    # -- the pybind methods
    def fit(self, steps: int) -> Dict:
        if self.loss_kind != "nmll":
            raise Unsupported("fit: the GPU fit loop optimises the NMLL (fmtgp_fit)")
        r = self.gpu.fit(self._internal(self.hyper), int(steps))
        self.hyper = self._user(r["hyper"])
        self._fresh = None
        res = self._refresh()
        return {"steps": int(steps), "final_loss": r["final_loss"], "loss_trace": list(r["loss_trace"]),
                "step_seconds": list(r["step_seconds"]), "jitter_escalations": res["escalations"],
                "tau": list(self._uvec(res["tau"]))}

    def loss(self) -> float:
        if self.loss_kind == "gcv":
            return float(self.gpu.gcv(self._internal(self.hyper))["gcv"])
        return float(self._refresh()["nll"])

    def tau(self) -> List[float]:
        if self.loss_kind == "gcv":
            raise Unsupported("tau: the GCV prior means are not exposed by the library (equal-n fmtgp_gcv)")
        return list(self._uvec(self._refresh()["tau"]))

    def posterior_mean(self, task: int, x) -> float:
        return float(self.posterior_mean_batch(task, [x])[0])

    def posterior_mean_batch(self, task: int, X) -> List[float]:
        self._refresh()
        X = np.asarray(X, dtype=np.float64).reshape(-1, self.d)
        return list(self.gpu.posterior_mean(self._task(task), X))

    def posterior_cov(self, task: int, x, task2: int, xp) -> float:
        self._refresh()
        x = np.asarray(x, dtype=np.float64).reshape(1, self.d)
        xp = np.asarray(xp, dtype=np.float64).reshape(1, self.d)
        return float(self.gpu.posterior_cov(self._task(task), x, self._task(task2), xp)[0])

    def cubature(self):
        self._refresh()
        mu, S = self.gpu.cubature()
        return self._uvec(mu), self._umat(S)

    def _task(self, u: int) -> int:
        if not 0 <= u < self.design.L:
            raise IndexError("task out of range")
        return self.i2u.index(u)

    # -- model document (gp_core.cpp:447-508), plus the generator (see module doc)
    def to_json(self) -> str:
        h, dz = self.hyper, self.design
        m_user = [0] * dz.L
        for l, u in enumerate(self.i2u):
            m_user[u] = dz.m[l]
        gen = {"kind": "lattice" if dz.kind == LATTICE else "digital", "internal_to_user": list(self.i2u),
               "shift_bits": [[int(v) for v in row] for row in dz.shift_bits]}
        if dz.kind == LATTICE:
            gen.update(g=[int(v) for v in dz.g], n_max=int(dz.n_max))
        else:
            gen.update(columns=[[int(v) for v in row] for row in dz.columns])
        doc = {"kind": "lattice" if dz.kind == LATTICE else "digital", "family": self.kernel,
               "loss": self.loss_kind, "d": self.d, "seed": self.seed, "m": m_user,
               "hyper": {"gamma": h.gamma, "eta": list(map(float, h.eta)), "si_alpha": int(h.si_alpha),
                         "b": list(map(float, h.b)), "t": list(map(float, h.t)), "xi": list(map(float, h.xi)),
                         "tau": [0.0] * dz.L, "lengthscales": [0.25] * self.d,
                         "B": [list(map(float, row)) for row in h.B]},
               "y": [list(map(float, v)) for v in self.y_user], "generator": gen}
        return json.dumps(doc, indent=1)

    @staticmethod
    def from_json(text: str, device: int = 0) -> "Model":
        doc = json.loads(text)
        gen = doc.get("generator")
        if gen is None:
            raise Unsupported("from_json: the document has no 'generator' (written by the reference, whose "
                              "make_design tables are not vendored here); its design cannot be rebuilt exactly")
        hj = doc["hyper"]
        L = len(doc["m"])
        i2u = [int(v) for v in gen["internal_to_user"]]
        m = [int(doc["m"][u]) for u in i2u]
        if gen["kind"] == "lattice":
            design = Design(LATTICE, int(doc["d"]), m, np.array(gen["shift_bits"], dtype=np.uint64),
                            g=np.array(gen["g"], dtype=np.uint64), n_max=int(gen["n_max"]))
        else:
            design = Design(DIGITAL, int(doc["d"]), m, np.array(gen["shift_bits"], dtype=np.uint64),
                            columns=np.array(gen["columns"], dtype=np.uint64))
        B = np.array(hj["B"], dtype=np.float64).reshape(L, -1)
        hyper = Hyper(gamma=float(hj["gamma"]), eta=np.array(hj["eta"]), B=B, t=np.array(hj["t"]),
                      xi=np.array(hj["xi"]), si_alpha=int(hj["si_alpha"]), b=tuple(float(v) for v in hj["b"]))
        return Model(doc["family"], int(doc["d"]), [1 << v for v in doc["m"]], int(doc["seed"]), doc["y"],
                     loss=doc["loss"], device=device, _state={"design": design, "i2u": i2u, "hyper": hyper})


__all__ = ["Model", "design_points", "optimal_weights", "make_design", "test_points", "problem_eval", "KERNELS",
           "PROBLEMS"]
