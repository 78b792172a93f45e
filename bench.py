#!/usr/bin/env python3
"""Benchmark of the fast-MTGP fit hot path (BASELINE.json metric) on B200.

Default workload: BASELINE configs[1] ("config 2"): T=3 tasks, d=5, n=2^16 points per
task on scrambled digital nets, order-4 Walsh DSI kernel; one step = one fit evaluation
= NLL + logdet + analytic gradient w.r.t. (eta, w, v, gamma), inputs resident in HBM.

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the library's
stream; L2 is flushed (512 MiB write) before every timed step, outside the events; the
step times are summed, barrier + synchronize on both sides, max over ranks.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 2]

N > 1 (torchrun, NCCL): the fit does not shard (configs 1-2 are
"replicas only"), so every rank runs an independent replica and value = N x fits/s.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "MTGP fits/s (solve+logdet+NLL grad) at N=T·n; HBM GB/s vs B200 peak"


def load_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- roofline
def offset_classes(dz) -> int:
    """Distinct pair shift offsets (Delta_a ^ Delta_b digital, Delta_a - Delta_b lattice): the
    transforms run once per class, not per pair (diagonal pairs all share offset 0)."""
    sb = np.asarray(dz.shift_bits, dtype=np.uint64)
    mask = np.uint64((1 << 53) - 1)
    seen = set()
    for a in range(dz.L):
        for b in range(a, dz.L):
            o = (sb[a] ^ sb[b]) if dz.kind == 1 else ((sb[a] - sb[b]) & mask)
            seen.add(tuple(int(x) for x in o))
    return len(seen)


def algorithmic_bytes(kernel: str, inst, P: int, T: int, nc: int = 1) -> float:
    """Minimal HBM bytes one launch of `kernel` must move for this workload (8-byte words;
    SURVEY.md §8d per-kernel split).  Real (digital) slots are 8 B, lattice
    half-spectrum slots 16 B for n/2 of them: either way 8n bytes per vector.  Transforms run
    per pair-offset class (V of them, V <= P); the fused digital kernels also stream the
    design-time kappa table (d values per element per class)."""
    dz = inst.design
    n = dz.n[0]
    vec = 8.0 * n
    V = offset_classes(dz)
    # nc candidates per launch (config 5: 64): the kappa table and yhat are read once per launch
    table = {
        "dig_col_fwd": V * (nc + dz.d) * vec,  # kappa table in, intermediate out
        "dig_mid": (2 * V * nc + T) * vec,  # intermediate + yhat in; Z (class adjoints) out
        "dig_col_inv": V * (nc + dz.d) * vec,  # intermediate + kappa table in
        "fwd_col_dig": P * vec, "fwd_col_lat": P * vec,  # generator on the fly -> write intermediate
        "fwd_row_dig": 2 * P * vec, "fwd_row_lat": 2 * P * vec,  # read intermediate, write spectra
        "fwd_small_dig": P * vec, "fwd_small_lat": P * vec,  # write spectra
        "solve_equal": (2 * P + T) * vec,  # read P spectra + T yhat, write P adjoints M
        "inv_row_dig": 2 * P * vec, "inv_row_lat": 2 * P * vec,  # read M, write intermediate
        "inv_col_dig": P * vec, "inv_col_lat": P * vec,  # read intermediate, dot in registers
        "inv_small_dig": P * vec, "inv_small_lat": P * vec,
        "finalize": 0.0, "dig_finalize": 0.0,
        # fused lattice path (lattice.cuh): n/2 complex slots of 16 B = 8n bytes per vector
        "lat_col_fwd": V * vec,  # generator on the fly -> intermediate out
        "lat_mid": (2 * V + T) * vec,  # intermediate + yhat in; inverse-row intermediate out
        "lat_col_inv": V * vec,  # intermediate in, gradient dot in registers
    }
    return table.get(kernel, 0.0)


def ncu_traffic(kernel: str):
    """dram__bytes_read+write per launch from the committed ncu --set full capture."""
    path = os.path.join(HERE, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm
def cpu_reference(inst, steps: int, warmup: int, grad_params: int):
    """Time the reference C++ library itself (oracle/_ref) on host cores: one step = one
    loss_value (build_spectrum + invert_and_logdet + tau + solve) of the full workload;
    a fit with the reference's own central-FD gradient costs (1 + 2 P_theta) of them
    (gp_core.cpp:341-351), so fits/s = 1 / ((1 + 2 P_theta) * t_loss)."""
    threads = os.cpu_count() or 1
    os.environ["FASTMTGP_THREADS"] = str(threads)
    from oracle import ref  # test-infrastructure checker / CPU baseline only
    kind = "reference"
    if not ref.available():
        raise RuntimeError("oracle/_ref not built")
    model = ref.Model(inst.design, inst.hyper, inst.y)
    for _ in range(warmup):
        model.set_hyper(inst.hyper)
        model.loss(0)
    ts = []
    for _ in range(steps):
        model.set_hyper(inst.hyper)  # invalidate caches: full refresh every step
        t0 = time.perf_counter()
        model.loss(0)
        ts.append(time.perf_counter() - t0)
    t_loss = statistics.median(ts)
    evals = 1 + 2 * grad_params
    return {"value": 1.0 / (evals * t_loss), "unit": "fits/s", "cores": threads, "kind": kind,
            "sample": f"{len(ts)} x reference loss_value at N = {inst.design.N} (median {t_loss * 1e3:.1f} ms); "
                      f"fit = {evals} loss evaluations (central-FD gradient over {grad_params} parameters)",
            "t_loss_s": t_loss}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics only: skip the L2 flush")
    args = ap.parse_args()
    warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2603_16014_b200 import configs

    inst = configs.make(args.config)
    dz, hp = inst.design, inst.hyper
    P, T = dz.L * (dz.L + 1) // 2, dz.L
    grad_params = dz.d + hp.B.size + T + 1  # eta, w, v, gamma
    workload = {1: "config1", 2: "config2: T=3 d=5 n=2^16 scrambled digital net, order-4 Walsh DSI kernel",
                3: "config3", 4: "config4: T=2 d=4 n=2^26 lattice B2",
                5: "config5: T=4 d=10 n=2^18 digital order-4 Walsh, 256-candidate sweep per step"}[args.config]
    config = {"workload": workload, "N": dz.N, "T": T, "d": dz.d, "n": dz.n[0],
              "outputs": "NLL, logdet, dNLL/d(eta, w, v, gamma)", "l2": "flushed before every step (512 MiB write)",
              "parallelism": {4: "frequency-sharded (2 NCCL all-to-alls per fit)",
                              5: "candidate-sharded (gather of the records)"}.get(args.config, "replicas")
              if args.gpus > 1 else "single"}

    if args.impl == "reference":
        if rank != 0:
            return
        if args.config == 4:  # as the cpu_baseline below: 2^20 per task, scaled by N log2 N
            small = configs.make(4, m=[20, 20])
            cb = cpu_reference(small, args.steps, warmup, grad_params)
            f = (dz.N * np.log2(dz.N)) / (small.design.N * np.log2(small.design.N))
            cb["value"] /= f
            cb["sample"] += f"; measured at 2 x 2^20 points and scaled by N log2 N (x{f:.1f}) to 2 x 2^26"
        else:
            cb = cpu_reference(inst, args.steps, warmup, grad_params)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "fits/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": warmup, "ms_per_step": 1e3 / cb["value"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": "fits/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_2603_16014_b200.fast_gram import Model

    model = Model(dz, device=local_rank, max_candidates=64 if args.config == 5 else 1)
    model.set_y(inst.y)
    stream = torch.cuda.ExternalStream(model.stream, device=torch.device("cuda", local_rank))
    sharded = (args.config == 4 and world > 1) or args.config == 5  # one job-wide unit per step
    if args.config == 4 and world > 1:
        # config 4 at N > 1: the frequency-sharded fit — one fit per step over all
        # ranks (strong scaling): column pass -> NCCL all-to-all -> row pass + solve -> all-to-all ->
        # inverse column pass + gradient dot -> gather of the 101-double records
        from paper_2603_16014_b200 import sharding
        shard = sharding.ShardedLatticeFit(dz, rank, world, device=local_rank, model=model)
        ex, ga = sharding.dist_exchange(shard), sharding.dist_gather(shard)

        class _Sharded:
            def nll(self, h, grad=True):
                return sharding.sharded_nll([shard], h, grad=grad, exchange=ex, gather=ga)

            def set_y(self, y):
                model.set_y(y)

            def profile(self, on=True):
                model.profile(on)

            def profile_read(self):
                return model.profile_read()
        fitter = _Sharded()
    elif args.config == 5:
        # config 5: one step = the 256-candidate sweep (NLL + full gradient each), candidates
        # sharded over the ranks (strong scaling, no data-path collective)
        from paper_2603_16014_b200 import sharding

        class _Sweep:
            def nll(self, h, grad=True):
                res = sharding.sweep(lambda cs: model.nll_batch(cs, grad=grad), inst.candidates, world, rank)
                return res[0]

            def set_y(self, y):
                model.set_y(y)

            def profile(self, on=True):
                model.profile(on)

            def profile_read(self):
                return model.profile_read()
        fitter = _Sweep()
    else:
        fitter = model
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local_rank}")

    for _ in range(warmup):
        fitter.nll(hp, grad=True)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def timed_pass(profile: bool):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        fitter.profile(profile)
        barrier()
        for k in range(args.steps):
            if not args.no_flush:
                with torch.cuda.stream(stream):
                    flush.fill_(float(k))
            ev[k][0].record(stream)
            r = fitter.nll(hp, grad=True)
            ev[k][1].record(stream)
        barrier()
        prof = fitter.profile_read() if profile else {}
        fitter.profile(False)
        return r, sum(a.elapsed_time(b) for a, b in ev), prof

    # ---- device-resident timed region.  Per-kernel CUDA events (event-record nodes inside the
    # fit's graph) cost ~35 us of graph overhead per step, so `value` comes from an
    # un-instrumented pass and the per-kernel durations from a second, instrumented pass of the
    # same K steps (roofline["timing"]).
    with ClockSampler(local_rank) as clk:
        res, total_ms, _ = timed_pass(False)
        _, prof_total_ms, prof = timed_pass(True)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    per_step = len(inst.candidates) if args.config == 5 else 1  # fits per step (config 5: the sweep)
    value = per_step * (1 if sharded else world) * 1e3 / ms_per_step  # sharded: one unit over all ranks

    # ---- end to end through the public API: pinned host y -> device, fit, result -> host
    y_pinned = torch.empty(dz.N, dtype=torch.float64).pin_memory().numpy()
    y_pinned[:] = inst.y
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))
        e2e_ev[k][0].record(stream)
        fitter.set_y(y_pinned)  # H2D + yhat transform + tau
        res = fitter.nll(hp, grad=True)  # fit; result (NLL + gradient) copied back to host
        e2e_ev[k][1].record(stream)
    barrier()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
    if dist:
        t = torch.tensor([e2e_ms], device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = per_step * (1 if sharded else world) * 1e3 * args.steps / e2e_ms
    hyper_bytes = 8 * (dz.d + 1 + P + 2 * P)
    h2d = 8 * dz.N + hyper_bytes
    d2h = 8 * ((4 + 16 + 64) + 1 + 2 * 8 + 8)  # result block: record, bad flag, non-real maxima, tau (model.cu res_len)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel
    peak, peak_src = load_peaks()
    launches = sum(c for _, c in prof.values())
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_cnt) = dom
    avg_ms = dom_ms / max(dom_cnt, 1)
    ncl = 64 if args.config == 5 else 1  # candidates per launch
    alg = algorithmic_bytes(dom_name, inst, P, T, ncl)
    achieved = alg / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else 0.0
    kernels = {k: {"avg_us": 1e3 * v[0] / max(v[1], 1), "launches": v[1],
                   "share": v[0] / max(sum(x[0] for x in prof.values()), 1e-12),
                   "alg_GBps": (algorithmic_bytes(k, inst, P, T, ncl) / (1e-3 * v[0] / max(v[1], 1)) / 1e9)
                   if v[0] > 0 else None} for k, v in prof.items()}
    roofline = {"bound": "hbm", "kernel": dom_name,
                "timing": "per-kernel CUDA events on the fit stream, second pass of the same K steps "
                          f"({1e3 * prof_total_ms / args.steps:.1f} us/step instrumented)", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(dom_name) if args.config in (2, 4) else None,  # captured configs "alg_bytes_per_launch": alg,
                "peak_source": peak_src, "kernels": kernels}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            if args.config == 4:
                # one reference loss at n = 2^26 per task takes minutes: time it at 2^20 per task
                # and scale by N log2 N (FFT-dominated) — stated in `sample`
                small = configs.make(4, m=[20, 20])
                cb = cpu_reference(small, 2, 1, grad_params)
                n_s, n_f = small.design.N, dz.N
                f = (n_f * np.log2(n_f)) / (n_s * np.log2(n_s))
                cb["value"] /= f
                cb["sample"] += f"; measured at 2 x 2^20 points and scaled by N log2 N (x{f:.1f}) to 2 x 2^26"
            else:
                cb = cpu_reference(inst, 3, 1, grad_params)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "fits/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    line = {"metric": METRIC, "value": value, "unit": "fits/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config; no dataset)",
            "config": config, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "fits/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "clocks": clk.summary(), "gpu_launches": launches,
            "result": {"nll": res["nll"], "logdet": res["logdet"]}}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
