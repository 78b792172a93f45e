"""Command-line front-end with the subcommands of the reference CLI (tools/fastmtgp_cli.cpp:41-88)
on the B200 path:

    python -m paper_2603_16014_b200.cli points   --kernel si-lattice --n 1024,256 --d 3 --seed 7
    python -m paper_2603_16014_b200.cli fit      --model model.json --steps 20 [--model-out fitted.json]
    python -m paper_2603_16014_b200.cli cubature --model model.json [--steps 20]
    python -m paper_2603_16014_b200.cli scaling  --kernel dsi-digital --n 4096,1024 --d 4 --trials 3

`points` writes the per-task designs as CSV (task, index, x_1..x_d; user task order); `fit` and
`cubature` read a model document (gp_core.cpp:447-508 plus the generator, paper_2603_16014_b200.
fastmtgp) and print a JSON report; `scaling` times build + invert (the reference's cmd_scaling) on
the device.  The reference's `--problem` benchmark functions (problems.cpp) are not part of the B200
path: observations come from the model document.
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


def cmd_points(a, out) -> int:
    kind = "lattice" if a.kernel == "si-lattice" else "digital"
    pts = fastmtgp.design_points(kind, a.d, _sizes(a.n), a.seed)
    out.write("task,index," + ",".join(f"x{j + 1}" for j in range(a.d)) + "\n")
    for u, P in enumerate(pts):
        for i, row in enumerate(P):
            out.write(f"{u},{i}," + ",".join(repr(float(v)) for v in row) + "\n")
    return 0


def _load(path: str) -> fastmtgp.Model:
    with open(path) as f:
        return fastmtgp.Model.from_json(f.read())


def cmd_fit(a, out) -> int:
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
    m = _load(a.model)
    if a.steps > 0:
        m.fit(a.steps)
    mu, S = m.cubature()
    json.dump({"mu": list(map(float, mu)), "Sigma": [list(map(float, r)) for r in S], "loss": m.loss()}, out, indent=1)
    out.write("\n")
    return 0


def cmd_scaling(a, out) -> int:
    from .designs import Hyper
    from .fast_gram import Model as GpuModel
    kind = fastmtgp.KERNELS[a.kernel]
    n = _sizes(a.n)
    design, _ = fastmtgp.make_design(kind, a.d, [int(np.log2(v)) for v in n], a.seed)
    L = design.L
    hp = Hyper(gamma=1.0, eta=np.ones(a.d), B=np.full((L, 1), 0.5), t=np.full(L, 0.1), xi=np.full(L, a.jitter),
               b=(0.0, 0.0, 0.0, 1.0))
    g = GpuModel(design)
    out.write("N,L,trial,build_invert_ms\n")
    for k in range(a.trials):
        t0 = time.perf_counter()
        g.build_spectrum(hp)
        g.invert_and_logdet()
        out.write(f"{design.N},{L},{k},{1e3 * (time.perf_counter() - t0):.4f}\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2603_16014_b200.cli",
                                 description="fast multitask GP regression and Bayesian cubature on a B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("points", "fit", "cubature", "scaling"):
        p = sub.add_parser(name)
        p.add_argument("--kernel", default="si-lattice", choices=sorted(fastmtgp.KERNELS))
        p.add_argument("--n", default="1024", help="samples per task, powers of two (user task order)")
        p.add_argument("--d", type=int, default=2)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--steps", type=int, default=0)
        p.add_argument("--trials", type=int, default=1)
        p.add_argument("--jitter", type=float, default=1e-8)
        p.add_argument("--model", help="model document (JSON) for fit / cubature")
        p.add_argument("--model-out", default="")
        p.add_argument("--out", default="", help="output path (default stdout)")
    a = ap.parse_args(argv)
    out = open(a.out, "w") if a.out else sys.stdout
    try:
        if a.cmd in ("fit", "cubature") and not a.model:
            ap.error(f"{a.cmd} needs --model")
        return {"points": cmd_points, "fit": cmd_fit, "cubature": cmd_cubature, "scaling": cmd_scaling}[a.cmd](a, out)
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 1
    finally:
        if a.out:
            out.close()


if __name__ == "__main__":
    sys.exit(main())
