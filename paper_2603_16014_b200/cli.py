"""Command-line front-end with the subcommands of the reference CLI (tools/fastmtgp_cli.cpp:41-88,
bench.cpp:197-372) on the B200 path:

    python -m paper_2603_16014_b200.cli points   --kernel si-lattice --n 1024,256 --d 3 --seed 7
    python -m paper_2603_16014_b200.cli fit      --problem ackley --kernel si-lattice --n 4096,1024 --steps 20
    python -m paper_2603_16014_b200.cli fit      --model model.json --steps 20 [--model-out fitted.json]
    python -m paper_2603_16014_b200.cli cubature --problem borehole --n 1024,256 [--steps 20]
    python -m paper_2603_16014_b200.cli bench    --problem rosenbrock --n 256,64,16 --trials 3
    python -m paper_2603_16014_b200.cli scaling  --kernel dsi-digital --n 4096,1024 --trials 3

`points` writes the per-task designs as CSV (task 1-based, index, x_1..x_d; user task order).
`fit` / `cubature` / `bench` run the reference's fit_trial (bench.cpp:84-107) on a benchmark problem
(--problem: observations of fidelity u + 1 for user task u plus --noise, computed on the device at
the design points) or on a model document (--model: gp_core.cpp:447-508 plus the generator) and
print the reference's JSON / CSV reports; `fit`'s l2_rel_error is over the held-out set of
--test-points points (bench.cpp:155-170) with the problem evaluated on the device.  `scaling` times
build + invert (cmd_scaling).  Deviations: the reference's frozen integral table (problems.cpp
refs(); data/) is not vendored, so `cubature` / `bench` report mu without abs_error_vs_reference;
designs come from this package's seeded generators (fastmtgp module doc).
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import fastmtgp


def _sizes(text: str):
    return [int(v) for v in text.split(",") if v]


def _n_label(n) -> str:
    return "x".join(str(v) for v in n)


def _problem_n(a):
    """--n, or 2^6 per fidelity of the problem (default_m, bench.cpp:45-48)."""
    return _sizes(a.n) if a.n else [64] * fastmtgp.PROBLEMS[a.problem][1]


def cmd_points(a, out) -> int:
    kind = "lattice" if a.kernel == "si-lattice" else "digital"
    d = a.d if a.d > 0 else fastmtgp.PROBLEMS[a.problem][0]
    pts = fastmtgp.design_points(kind, d, _sizes(a.n) if a.n else [8], a.seed)
    out.write("task,index," + ",".join(f"x{j + 1}" for j in range(d)) + "\n")
    for u, P in enumerate(pts):
        for i, row in enumerate(P):
            out.write(f"{u + 1},{i}," + ",".join(repr(float(v)) for v in row) + "\n")
    return 0


def _trial(a, trial: int = 0) -> fastmtgp.Model:
    """fit_trial (bench.cpp:84-107): the model for seed + trial, fitted --steps."""
    m = fastmtgp.Model.from_problem(a.problem, a.kernel, _problem_n(a), seed=a.seed + trial, noise=a.noise,
                                    loss=a.loss, task_rank=a.task_rank, jitter=a.jitter)
    m.report = m.fit(a.steps) if a.steps > 0 else {"steps": 0, "final_loss": m.loss(), "loss_trace": [],
                                                   "step_seconds": [], "jitter_escalations": 0, "tau": m.tau()}
    return m


def _hyper_json(m: fastmtgp.Model):
    h = m.hyper
    return {"gamma": h.gamma, "eta": list(map(float, h.eta)), "si_alpha": int(h.si_alpha), "b": list(map(float, h.b)),
            "B": [list(map(float, r)) for r in h.B], "t": list(map(float, h.t)), "xi": list(map(float, h.xi))}


def _load(path: str) -> fastmtgp.Model:
    with open(path) as f:
        return fastmtgp.Model.from_json(f.read())


def cmd_fit(a, out) -> int:
    if not a.model:  # cmd_fit (bench.cpp:217-241)
        m = _trial(a)
        n = _problem_n(a)
        X = fastmtgp.test_points(a.kernel, m.d, a.test_points, a.seed)
        doc = {"problem": a.problem, "kernel": a.kernel, "loss": a.loss, "n": _n_label(n), "seed": a.seed,
               "hyperparameters": _hyper_json(m), "report": m.report,
               "l2_rel_error": [m.l2_relative_error(u, X) for u in range(len(n))]}
        if a.model_out:
            with open(a.model_out, "w") as f:
                f.write(m.to_json())
            doc["model_out"] = a.model_out
        json.dump(doc, out, indent=1)
        out.write("\n")
        return 0
    m = _load(a.model)
    rep = m.fit(a.steps) if a.steps > 0 else {"steps": 0, "final_loss": m.loss()}
    rep["loss"] = m.loss()
    if a.model_out:
        with open(a.model_out, "w") as f:
            f.write(m.to_json())
    json.dump(rep, out, indent=1)
    out.write("\n")
    return 0


def cmd_cubature(a, out) -> int:
    if a.model:
        m = _load(a.model)
        if a.steps > 0:
            m.fit(a.steps)
    else:
        m = _trial(a)
    mu, S = m.cubature()
    chi = np.ones(len(mu))
    w, mse = fastmtgp.optimal_weights(mu, S, chi)
    doc = {"mu": list(map(float, mu)), "Sigma": [list(map(float, r)) for r in S],
           "Sigma_diag": list(map(float, np.diag(S))), "chi": list(map(float, chi)), "chi_mu": float(chi @ mu),
           "chi_Sigma_chi": float(chi @ S @ chi), "weights": list(map(float, w)), "weights_mse_min": float(mse),
           "loss": m.loss()}
    if not a.model:  # cmd_cubature (bench.cpp:243-283) keys
        doc = {"problem": a.problem, "kernel": a.kernel, "n": _n_label(_problem_n(a)), "seed": a.seed, **doc}
    json.dump(doc, out, indent=1)
    out.write("\n")
    return 0


def cmd_bench(a, out) -> int:
    """cmd_bench (bench.cpp:285-332): per trial the median step time, the top task's l2 error and the
    final loss (trials run one after another on the device); a failed trial is reported and makes
    the exit code 1."""
    n = _problem_n(a)
    out.write("problem,method,n,trial,time_per_step,l2_rel_error,final_loss\n")
    rows, bad = [], 0
    X = fastmtgp.test_points(a.kernel, fastmtgp.PROBLEMS[a.problem][0], a.test_points, a.seed)
    for t in range(a.trials):
        try:
            m = _trial(a, t)
            st = m.report["step_seconds"]
            rows.append((float(np.median(st)) if st else 0.0, m.l2_relative_error(len(n) - 1, X),
                         float(m.report["final_loss"])))
            out.write(f"{a.problem},{a.kernel},{_n_label(n)},{t}," + ",".join(repr(v) for v in rows[-1]) + "\n")
        except Exception as e:  # noqa: BLE001
            print(f"bench: trial {t} failed: {e}", file=sys.stderr)
            bad += 1
    if rows:
        med = np.median(np.array(rows), axis=0)
        out.write(f"{a.problem},{a.kernel},{_n_label(n)},median," + ",".join(repr(float(v)) for v in med) + "\n")
    return 0 if bad == 0 else 1


def cmd_scaling(a, out) -> int:
    from .designs import Hyper
    from .fast_gram import Model as GpuModel
    kind = fastmtgp.KERNELS[a.kernel]
    d = a.d if a.d > 0 else 4  # time_build_invert's d = 4 (bench.cpp:334-336)
    grid = [_sizes(a.n)] if a.n else [[1 << m] for m in range(10, 17)] + [[4096, 4096], [16384, 16]]
    out.write("kind,n,seconds\n")
    for n in grid:
        design, _ = fastmtgp.make_design(kind, d, [int(np.log2(v)) for v in n], a.seed)
        L = design.L
        hp = Hyper(gamma=1.0, eta=np.ones(d), B=np.full((L, 1), 0.5), t=np.full(L, 0.5), xi=np.full(L, a.jitter),
                   b=(1.0, 1.0, 1.0, 1.0))
        g = GpuModel(design)
        secs = []
        for _ in range(max(1, a.trials)):
            t0 = time.perf_counter()
            g.build_spectrum(hp)
            if not np.isfinite(g.invert_and_logdet()):
                raise RuntimeError("time_build_invert: bad logdet")
            secs.append(time.perf_counter() - t0)
        g.close()
        out.write(f"{a.kernel},{_n_label(n)},{float(np.median(secs)):.6g}\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2603_16014_b200.cli",
                                 description="fast multitask GP regression and Bayesian cubature on a B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("points", "fit", "cubature", "bench", "scaling"):
        p = sub.add_parser(name)
        p.add_argument("--problem", default="ackley", choices=sorted(fastmtgp.PROBLEMS))
        p.add_argument("--kernel", default="dsi-digital", choices=sorted(fastmtgp.KERNELS))
        p.add_argument("--loss", default="nmll", choices=["nmll", "gcv"])
        p.add_argument("--n", default="", help="samples per task, powers of two (user task order)")
        p.add_argument("--d", type=int, default=0, help="dimension override (points, scaling)")
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--steps", type=int, default=100 if name in ("fit", "cubature", "bench") else 0)
        p.add_argument("--trials", type=int, default=1)
        p.add_argument("--noise", type=float, default=0.0)
        p.add_argument("--jitter", type=float, default=1e-8)
        p.add_argument("--task-rank", type=int, default=1)
        p.add_argument("--test-points", type=int, default=2048)
        p.add_argument("--model", default="", help="model document (JSON) for fit / cubature instead of --problem")
        p.add_argument("--model-out", default="")
        p.add_argument("--out", default="", help="output path (default stdout)")
    a = ap.parse_args(argv)
    out = open(a.out, "w") if a.out else sys.stdout
    try:
        return {"points": cmd_points, "fit": cmd_fit, "cubature": cmd_cubature, "bench": cmd_bench,
                "scaling": cmd_scaling}[a.cmd](a, out)
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 1
    finally:
        if a.out:
            out.close()


if __name__ == "__main__":
    sys.exit(main())
