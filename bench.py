#!/usr/bin/env python3
"""Benchmark of the fast-MTGP fit hot path (BASELINE.json metric) on B200.

Default workload: BASELINE config 4 -- the largest single-GPU configuration, on which the
north-star's HBM-roofline target is stated: T=2 tasks, d=4, n=2^26 points per task on a rank-1
lattice (N = 2^27), B2 kernel; one step = one fit evaluation = NLL + logdet + analytic gradient
w.r.t. (eta, w, v, gamma), inputs resident in HBM.  `--config 2|5` runs the other configs.

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the library's
stream; L2 is flushed (512 MiB write) before every timed step, outside the events; the
step times are summed, barrier + synchronize on both sides, max over ranks.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 4]

N > 1 (one process per GPU; `--gpus N` self-launches torchrun when WORLD_SIZE is unset):
config 4 runs the frequency-sharded fit (SURVEY.md §8e, strong scaling), config 5 shards the
candidates, configs 1-2 run independent replicas (value = N x fits/s).

Reference arm (`--impl reference`): the reference's own `fit` (oracle/_ref, built from the
unmodified reference sources) on the host cores, its own per-step timer; see cpu_reference.
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


def ncu_traffic(cfg: int, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    `ncu --set full` capture of this config (profiles/ncu_traffic.json, written by
    tools/ncu_summary.py from the capture named there); (None, None) if not captured."""
    path = os.path.join(HERE, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        ent = d.get(f"config{cfg}", {})
        if kernel in ent:
            return ent[kernel], ent.get("_source", "profiles/ncu_traffic.json")
    except Exception:
        pass
    return None, None


# ----------------------------------------------------------------------------- reference arm
# Bounded samples for the CPU reference (one reference fit step at the full config 4 / 5 size takes
# ~40 min / ~75 s on the host): the same generator, kernel and hyperparameters at 2^m per task,
# scaled to the full size by N log2 N (the reference's cost is transform-dominated at these
# shapes; checked against one full-size reference loss_value, tools/ref_scaling.py
# -> profiles/r02_ref_scaling.json).  Configs 1-2 run at full size.
REF_SAMPLE_M = {4: 18, 5: 14}
# config 3: the reference's own solve throws at full size ("abnormal imaginary residue",
# fast_gram.cpp:289-296, SURVEY.md §8c caveat 1), so its cost is sampled at n = 2^16..2^10
# (same generator, kernel, hyperparameters) and scaled by N log2 N: one loss_value (the fit's
# build + invert + solves) plus REF_C3_QUERIES posterior_cov calls (one solve each,
# gp_core.cpp:423-445) scaled to the 2^14 test points.
REF_C3_M = [16, 14, 12, 10]
REF_C3_QUERIES = 8


def nlogn(N: int) -> float:
    return N * np.log2(N)


def cpu_reference(cfg: int, inst, steps: int, warmup: int):
    """The reference's own fit (gp_core.cpp:317-382) on host cores, timed by the reference's own
    per-step timer (FitReport::step_seconds): one step = central-FD gradient (2 P_theta calls of
    loss_value) + iRprop- update + loss at the new theta = the reference's NLL + gradient, our
    unit of work.  Returns the per-step seconds actually measured and the metric value
    (fits/s of the full workload; config 5: candidate fits/s)."""
    threads = os.cpu_count() or 1
    os.environ["FASTMTGP_THREADS"] = str(threads)
    from oracle import ref  # test-infrastructure checker / CPU baseline only
    if not ref.available():
        raise RuntimeError("oracle/_ref not built")
    from paper_2603_16014_b200 import configs
    dz = inst.design
    if cfg == 3:
        import time as _t
        sample = configs.make(3, m=REF_C3_M, n_test=REF_C3_QUERIES)
        model = ref.Model(sample.design, sample.hyper, sample.y)
        model.loss(0)  # warm-up
        t0 = _t.perf_counter()
        model.loss(0)
        t_fit = _t.perf_counter() - t0
        t0 = _t.perf_counter()
        for x in sample.X_test:
            model.posterior_cov(0, x, 0, x)
        t_q = (_t.perf_counter() - t0) / len(sample.X_test)
        scale = nlogn(dz.N) / nlogn(sample.design.N)
        nq = len(inst.X_test)
        t_step = (t_fit + nq * t_q) * scale
        what = (f"reference loss_value ({t_fit:.3f} s) + {len(sample.X_test)} posterior_cov calls ({t_q:.4f} s each) "
                f"at n = 2^{REF_C3_M[0]}..2^{REF_C3_M[-1]} (N = {sample.design.N}; the reference's solve throws at "
                f"full size, fast_gram.cpp:289-296), {nq} queries, scaled by N log2 N (x{scale:.1f}) to N = {dz.N}")
        return {"value": 1.0 / t_step, "unit": "fits/s", "cores": threads, "kind": "reference", "sample": what,
                "t_step_s": (t_fit + len(sample.X_test) * t_q), "scale": scale, "n_params": 0}
    m_s = REF_SAMPLE_M.get(cfg)
    if m_s is not None and m_s < dz.m[0]:
        sample = configs.make(cfg, m=[m_s] * dz.L, **({"n_cand": 1} if cfg == 5 else {}))
        scale = nlogn(dz.N) / nlogn(sample.design.N)
    else:
        sample, scale = inst, 1.0
    model = ref.Model(sample.design, sample.hyper, sample.y)
    secs, n_params, _ = ref.fit_timed(model, warmup + steps)
    timed = secs[warmup:]
    t_step = float(np.mean(timed))
    what = (f"reference fit (gp_core.cpp:317-382), {len(timed)} timed iRprop- steps after {warmup} warm-up, each "
            f"= central-FD gradient over {n_params} parameters ({2 * n_params} loss_value calls) + update + "
            f"loss at the new theta; mean {t_step:.3f} s/step at N = {sample.design.N}")
    if scale != 1.0:
        what += (f"; sample 2^{m_s} per task, scaled by N log2 N (x{scale:.1f}) to N = {dz.N} "
                 f"(validation: profiles/r02_ref_scaling.json)")
    if cfg == 5:
        what += "; one candidate per step (value = candidate fits/s)"
    return {"value": 1.0 / (t_step * scale), "unit": "fits/s", "cores": threads, "kind": "reference",
            "sample": what, "t_step_s": t_step, "scale": scale, "n_params": n_params}


# ----------------------------------------------------------------------------- main
WORKLOADS = {1: "config1: T=2 d=2 n=2^10 lattice B2",
             2: "config2: T=3 d=5 n=2^16 scrambled digital net, order-4 Walsh DSI kernel",
             3: "config3: T=4 d=8 n=2^20/2^18/2^16/2^14 lattice B4",
             4: "config4: T=2 d=4 n=2^26 lattice B2 (N = 2^27)",
             5: "config5: T=4 d=10 n=2^18 digital order-4 Walsh, 256-candidate sweep per step"}


def self_launch(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks on this node (NCCL over NVLink),
    one process per GPU, rendezvous on 127.0.0.1; rank 0's JSON line is this process's output."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config; default 4 = the largest single-GPU config (headline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics only: skip the L2 flush")
    ap.add_argument("--chunks", type=int, default=2,
                    help="config 4 at N > 1: all-to-all pipeline depth (fmtgp_shard_chunks; 1 = unpipelined)")
    args = ap.parse_args()
    warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    from paper_2603_16014_b200 import configs

    inst = configs.make(args.config)
    dz, hp = inst.design, inst.hyper
    P, T = dz.L * (dz.L + 1) // 2, dz.L
    parallelism = "single"
    if args.gpus > 1:
        parallelism = {4: f"frequency-sharded over {world} GPUs (2 NCCL all-to-alls per fit, each in "
                          f"{args.chunks} chunk(s) under the L1 / L2 kernels)",
                       5: f"candidate-sharded over {world} GPUs (gather of the records)"}.get(args.config,
                                                                                      f"{world} replicas")
    config = {"workload": WORKLOADS[args.config], "N": dz.N, "T": T, "d": dz.d, "n": dz.n[0],
              "outputs": ("c, logdet, NLL, posterior variance at 2^14 test points, cubature mu and Sigma "
                          "(one 'fit' = all of them)") if args.config == 3 else "NLL, logdet, dNLL/d(eta, w, v, gamma)",
              "l2": "flushed before every step (512 MiB write)" if not args.no_flush else "not flushed",
              "parallelism": parallelism}

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference(args.config, inst, args.steps, warmup)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "fits/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": warmup, "ms_per_step": 1e3 * cb["t_step_s"],
                "ms_per_step_note": "what the reference actually ran per step (the bounded sample); value is "
                                    "scaled to the full workload as cpu_baseline.sample states",
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config,
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
    sharded = (args.config == 4 and world > 1) or args.config in (3, 5)  # one job-wide unit per step
    if args.config == 4 and world > 1:
        # config 4 at N > 1: the frequency-sharded fit — one fit per step over all
        # ranks (strong scaling): column pass -> NCCL all-to-all -> row pass + solve -> all-to-all ->
        # inverse column pass + gradient dot -> gather of the 101-double records
        from paper_2603_16014_b200 import sharding
        shard = sharding.ShardedLatticeFit(dz, rank, world, device=local_rank, model=model, chunks=args.chunks)
        ex, ga = sharding.dist_exchange(shard), sharding.dist_gather(shard)
        # guard (untimed): the pipelined exchange must reproduce the unpipelined one bit for bit
        if args.chunks > 1:
            ref_shard = sharding.ShardedLatticeFit(dz, rank, world, device=local_rank, model=model)
            a = sharding.sharded_nll([ref_shard], hp, grad=True, exchange=sharding.dist_exchange(ref_shard),
                                     gather=sharding.dist_gather(ref_shard))
            from paper_2603_16014_b200._lib import check
            check(model.lib.fmtgp_shard_chunks(model.h, args.chunks))  # ref_shard's setup reset it
            b = sharding.sharded_nll([shard], hp, grad=True, exchange=ex, gather=ga)
            if not (a["nll"] == b["nll"] and np.array_equal(a["deta"], b["deta"])):
                raise RuntimeError(f"pipelined exchange differs: {a['nll']} vs {b['nll']}")
            del ref_shard

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
    elif args.config == 3:
        # config 3: one step = fit (solve + logdet + NLL, unequal n) + posterior variance at the
        # 2^14 test points + multitask cubature (BASELINE configs[2] outputs); with N > 1 ranks the
        # test points are sharded (sharding.sharded_posterior_var)
        from paper_2603_16014_b200 import sharding

        class _Config3:
            def nll(self, h, grad=True):
                r = model.nll(h, grad=False)
                sharding.sharded_posterior_var(lambda Xb: model.posterior_var(0, Xb), inst.X_test, world, rank)
                model.cubature()
                return r

            def set_y(self, y):
                model.set_y(y)

            def profile(self, on=True):
                model.profile(on)

            def profile_read(self):
                return model.profile_read()
        fitter = _Config3()
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

    # ---- the same evaluation looped in C through the C ABI (fmtgp_bench_nll): no interpreter
    # between calls, so the Python call's cost is reported separately (configs with one model)
    c_loop = None
    if fitter is model and world == 1:
        cms, wall_us = model.bench_nll(hp, args.steps, grad=True, flush_bytes=0 if args.no_flush else 512 << 20)
        c_ms = float(np.mean(cms))
        c_loop = {"ms_per_step": c_ms, "value": per_step * 1e3 / c_ms, "host_wall_us_per_call": wall_us,
                  "python_api_us_per_step": 1e3 * (ms_per_step - c_ms),
                  "note": "fmtgp_nll looped in C (fmtgp_bench_nll), CUDA events per call on the model stream, "
                          "same L2 flush; `value` above is measured through the Python Model.nll"}

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
    traffic, traffic_src = ncu_traffic(args.config, dom_name)
    # whole fit against SURVEY.md §8d's algorithmic bytes 8n(6P + T) (the north-star's 60 % target)
    b_fit = 8.0 * dz.n[0] * (6 * P + T) * (len(inst.candidates) if args.config == 5 else 1)
    b_def = "SURVEY.md 8(d) B_alg = 8n(6P+T) per fit"
    if args.config == 3:  # fit 8(2S + 4N) + variance 16 N Q
        S_ = sum((T - l) * dz.n[l] for l in range(T))
        b_fit = 8.0 * (2 * S_ + 4 * dz.N) + 16.0 * dz.N * len(inst.X_test)
        b_def = "SURVEY.md 8(d) B_alg = 8(2S+4N) (fit) + 16 N Q (posterior variance), S = sum (T-l) n_l"
    fit_level = {"alg_bytes": b_fit, "definition": b_def,
                 "achieved": b_fit / (ms_per_step * 1e-3) / 1e9 * (1 if sharded else world),
                 "frac": b_fit / (ms_per_step * 1e-3) / 1e9 * (1 if sharded else world) / peak}
    # fp64 compute roof (SURVEY.md 8(d) approximate fp64 flops per step; peak = the DFMA
    # microbenchmark tools/micro/fp64_peak.cu on this pool's B200, profiles/r02_fp64_peak.log)
    fp64_flops = {2: 0.13e9, 3: 0.8e9 + 2.9e12, 4: 39e9, 5: 50e9}.get(args.config)
    fp64 = None
    if fp64_flops:
        fp64_peak = 34.13
        tf = fp64_flops / (ms_per_step * 1e-3) / 1e12 * (1 if sharded else world)
        fp64 = {"flops_per_step": fp64_flops, "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": tf / fp64_peak, "source": "SURVEY.md 8(d) flop estimate; peak measured "
                                                  "(profiles/r02_fp64_peak.log, DFMA, 2 flops per FMA)"}
    roofline = {"bound": "hbm", "kernel": dom_name,
                "timing": "per-kernel CUDA events on the fit stream, second pass of the same K steps "
                          f"({1e3 * prof_total_ms / args.steps:.1f} us/step instrumented)",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "alg_bytes_per_launch": alg, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": peak_src, "kernels": kernels, "fit": fit_level, "fp64": fp64}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:  # bounded: 1 warm-up + 2 timed reference fit steps (10-30 s of host work)
            cb = cpu_reference(args.config, inst, 2, 1)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "fits/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    line = {"metric": METRIC, "value": value, "unit": "fits/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config; no dataset)",
            "config": config, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "fits/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "clocks": clk.summary(), "gpu_launches": launches, "c_loop": c_loop,
            "result": {"nll": res["nll"], "logdet": res["logdet"]}}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
