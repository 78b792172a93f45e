"""Validate the N log2 N extrapolation of bench.py's CPU reference arm (config 4) with real
reference runs, including ONE full-size loss_value (2 x 2^26 points; minutes, ~35 GB RSS).

  python tools/ref_scaling.py [--max-m 26] > gpurun_out/ref_scaling.json

Times the reference's loss_value (build_spectrum + invert_and_logdet + tau + solve,
gp_core.cpp:197-227) on the config-4 generator / kernel / hyperparameters at 2^m per task, and
the reference fit step (FD gradient, 2 P + 1 losses) at the bench's sample size; reports the
N log2 N prediction from the sample next to each measurement.  TEST INFRASTRUCTURE (oracle)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-m", type=int, default=26)
    ap.add_argument("--sample-m", type=int, default=18)
    args = ap.parse_args()
    os.environ["FASTMTGP_THREADS"] = str(os.cpu_count() or 1)
    from oracle import ref
    from paper_2603_16014_b200 import configs

    def loss_time(m):
        inst = configs.make(4, m=[m, m])
        rm = ref.Model(inst.design, inst.hyper, inst.y)
        t0 = time.perf_counter()
        v = rm.loss(0)
        return time.perf_counter() - t0, v, inst.design.N

    out = {"cores": os.cpu_count(), "config": "config4 shape (T=2, d=4, B2, eta=0.8)", "loss_value": []}
    t_s, _, N_s = loss_time(args.sample_m)
    inst = configs.make(4, m=[args.sample_m] * 2)
    secs, npar, _ = ref.fit_timed(ref.Model(inst.design, inst.hyper, inst.y), 3)
    out["sample"] = {"m": args.sample_m, "N": N_s, "loss_s": t_s, "fit_step_s": secs[1:].tolist(), "n_params": npar,
                     "fit_step_over_loss": float(np.mean(secs[1:]) / t_s)}
    for m in range(args.sample_m, args.max_m + 1, 2):
        t, v, N = loss_time(m)
        pred = t_s * (N * np.log2(N)) / (N_s * np.log2(N_s))
        out["loss_value"].append({"m": m, "N": N, "seconds": t, "predicted_nlogn_s": pred, "measured_over_predicted": t / pred,
                                  "nll": v})
        print(json.dumps(out["loss_value"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
