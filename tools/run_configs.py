#!/usr/bin/env python3
"""Run every BASELINE config at full size on one GPU: timing (CUDA events), per-kernel
profile, and the checks that are feasible at that size (reference parity where the
reference finishes, self-consistency otherwise).  Development / evidence tool:
    python tools/run_configs.py [--configs 1,2,3,4,5] [--ref-check]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402


def timed(fn, reps=3, warm=1):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return out, min(ts), float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--ref-check", action="store_true")
    ap.add_argument("--cand", type=int, default=256)
    ap.add_argument("--queries", type=int, default=1 << 14)
    args = ap.parse_args()
    res = {}
    for cfg in [int(c) for c in args.configs.split(",")]:
        t0 = time.perf_counter()
        kw = {}
        if cfg == 5:
            kw["n_cand"] = args.cand
        if cfg == 3:
            kw["n_test"] = args.queries
        inst = configs.make(cfg, **kw)
        gen_s = time.perf_counter() - t0
        dz = inst.design
        out = {"N": dz.N, "input_gen_s": gen_s}
        if cfg == 5:
            M = Model(dz, max_candidates=64)
        else:
            M = Model(dz)
        M.set_y(inst.y)
        M.profile(True)
        if cfg in (1, 2, 4):
            r, best, med = timed(lambda: M.nll(inst.hyper, grad=True))
            out.update(nll=r["nll"], logdet=r["logdet"], deta=list(r["deta"]), fit_s_best=best, fit_s_med=med)
        if cfg in (1, 2, 4):  # the iRprop- fit loop, seconds per optimisation step
            M.profile(False)
            steps = 20 if cfg != 4 else 5
            f = M.fit(inst.hyper, steps)
            out.update(fit_steps=steps, fit_step_s_med=float(np.median(f["step_seconds"])),
                       fit_final_loss=f["final_loss"], fit_loss_first=float(f["loss_trace"][0]))
            M.profile(True)
        if cfg == 1:
            c = M.coefficients()
            pm, b2, m2 = timed(lambda: np.stack([M.posterior_mean(t, inst.X_test) for t in range(dz.L)]))
            out.update(post_mean_s=b2, c_norm=float(np.linalg.norm(c)))
        if cfg == 3:
            r, best, med = timed(lambda: M.nll(inst.hyper, grad=False), reps=2)
            out.update(nll=r["nll"], logdet=r["logdet"], fit_s_best=best)
            mu, S = M.cubature()
            out.update(cub_mu=list(mu), cub_Sigma=S.tolist())
            X = inst.X_test
            pv, b3, _ = timed(lambda: M.posterior_var(0, X), reps=1, warm=0)
            out.update(post_var_s=b3, post_var_min=float(pv.min()), post_var_max=float(pv.max()),
                       queries=int(X.shape[0]))
        if cfg == 5:
            rs, best, med = timed(lambda: M.nll_batch(inst.candidates, grad=True), reps=2)
            out.update(sweep_s_best=best, n_cand=len(rs), nll_first=rs[0]["nll"],
                       status=sorted({r["status"] for r in rs}), escalations=sum(r["escalations"] for r in rs))
        out["kernels"] = {k: {"ms": v[0], "n": v[1]} for k, v in M.profile_read().items()}
        if args.ref_check and cfg in (1, 2, 3):
            from oracle import ref
            rm = ref.Model(dz, inst.hyper, inst.y)
            t1 = time.perf_counter()
            nl = rm.loss(0)
            out["ref_loss_s"] = time.perf_counter() - t1
            out["ref_nll"] = nl
            out["nll_abs_diff"] = abs(nl - out["nll"])
            out["tol_1e-8N"] = 1e-8 * dz.N
        res[f"config{cfg}"] = out
        print(json.dumps({f"config{cfg}": out}), flush=True)
        M.close()


if __name__ == "__main__":
    main()
