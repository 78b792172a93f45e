"""Quick GPU-vs-reference diagnostics (prints, never asserts) — development aid."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.designs import DIGITAL, LATTICE, Hyper, digital_design, lattice_design, normal  # noqa
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def case(name, dz, hp, y):
    print(f"== {name}: kind={dz.kind} m={dz.m} d={dz.d}", flush=True)
    try:
        M = Model(dz)
        M.set_y(y)
        M.build_spectrum(hp)
        lam_ref = ref.build_spectrum(dz, hp)
        p = 0
        errs = []
        for l in range(dz.L):
            for lp in range(l, dz.L):
                errs.append(rel(M.spectrum(l, lp), lam_ref[p]))
                p += 1
        print("  spectrum rel err per pair:", ["%.1e" % e for e in errs])
        ld = M.invert_and_logdet()
        b = normal(7, 3, np.arange(dz.N))
        x_ref, kb_ref, ld_ref, tr_ref, Pi_ref = ref.invert_solve(dz, hp, b)
        print("  logdet gpu %.12g ref %.12g diff %.2e" % (ld, ld_ref, ld - ld_ref))
        x = M.solve(b)
        print("  solve rel %.2e" % rel(x, x_ref))
        kb = M.gram_matvec(b)
        print("  matvec rel %.2e" % rel(kb, kb_ref))
        try:
            print("  trace gpu %.10g ref %.10g" % (M.trace_inverse(), tr_ref))
            print("  Pi rel %.2e" % rel(M.extract_pi(), Pi_ref))
        except Exception as e:
            print("  trace/pi:", e)
        rm = ref.Model(dz, hp, y)
        nll_ref = rm.loss(0)
        st = rm.state()
        r = M.nll(hp, grad=True)
        print("  nll gpu %.12g ref %.12g diff %.2e (1e-8 N = %.1e)" % (r["nll"], nll_ref, r["nll"] - nll_ref,
                                                                       1e-8 * dz.N))
        print("  tau rel %.2e" % rel(r["tau"], st["tau"]))
        c = M.coefficients()
        print("  c rel %.2e" % rel(c, st["c"]))
        if dz.N <= 4096:
            fd = ref.nll_fd_grad(dz, hp, y)
            print("  deta gpu", r["deta"], "\n       fd ", fd["eta"], " rel %.2e" % rel(r["deta"], fd["eta"]))
            print("  dB rel %.2e  dt rel %.2e  dgamma %.8g vs %.8g" % (rel(r["dB"], fd["B"]), rel(r["dt"], fd["t"]),
                                                                     r["dgamma"], fd["gamma"]))
        if dz.N <= 8192:
            X = np.random.default_rng(0).random((64, dz.d))
            for t in range(dz.L):
                pm = M.posterior_mean(t, X)
                print("  post mean task %d rel %.2e" % (t, rel(pm, rm.posterior_mean(t, X))))
            mu, S = M.cubature()
            mu_r, S_r = rm.cubature()
            print("  cubature mu rel %.2e  Sigma rel %.2e" % (rel(mu, mu_r), rel(S, S_r)))
        M.close()
    except Exception:
        traceback.print_exc()


def main():
    for kind, dfn in ((LATTICE, lattice_design), (DIGITAL, digital_design)):
        for m in ([0], [1], [2, 2], [3, 3, 3], [5, 5], [8, 8], [12, 12], [14, 14], [15, 15], [16, 16, 16]):
            d = 3
            dz = dfn(d, m, seed=11)
            L = len(m)
            hp = Hyper(gamma=1.3, eta=np.array([0.9, 0.5, 0.3]), B=normal(3, 4, np.arange(L)).reshape(L, 1),
                       t=np.full(L, 0.3), xi=np.full(L, 1e-4), si_alpha=1 + (m[0] % 2), b=(0.5, 0.2, 0.1, 1.0))
            y = normal(5, 6, np.arange(dz.N))
            case(f"{'lat' if kind == LATTICE else 'dig'} {m}", dz, hp, y)
    for cfg, mm in ((1, None), (2, [12, 12, 12]), (2, None)):
        inst = configs.make(cfg, m=mm)
        t = time.time()
        case(f"config{cfg} {mm}", inst.design, inst.hyper, inst.y)
        print("  (%.1f s)" % (time.time() - t))


if __name__ == "__main__":
    main()
