"""Per-rank kernel cost of the pipelined exchange at the config-4 size (measurement aid).

G virtual ranks on one device run one correct sharded fit (local block copies); then rank 0's
phases are re-timed with CUDA events on its stream for chunks K = 1, 2, 4: L1 (all column chunks),
L2 (all row chunks), L3.  No all-to-all is timed (one GPU): the numbers say what chunking costs
the kernels (smaller launches, wave tails) — the exchange it hides is NVLink time.
python tools/shard_chunk_cost.py [G] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs, sharding  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
inst = configs.make(4)
dz, hp, y = inst.design, inst.hyper, inst.y
base = Model(dz)
base.set_y(y)
want = base.nll(hp, grad=True)
out = {"G": G, "elems_per_rank": None, "unsharded_nll": want["nll"]}
for K in (1, 2, 4):
    ranks = []
    if G <= 2:  # every rank: one correct fit first (the receive buffers hold real exchange blocks)
        for g in range(G):
            m = Model(dz)
            m.set_y(y)
            ranks.append(sharding.ShardedLatticeFit(dz, g, G, model=m, chunks=K))
        got = sharding.sharded_nll(ranks, hp, grad=True, exchange=sharding.local_exchange(G), gather=lambda r: r)
        assert abs(got["nll"] - want["nll"]) <= 1e-11 * abs(want["nll"]), (got["nll"], want["nll"])
    else:  # rank 0 only (G full models do not fit): zero receive buffers, same kernel work
        ranks.append(sharding.ShardedLatticeFit(dz, 0, G, model=base, chunks=K))
        for b in ranks[0].bufs:
            b.zero_()
    r0 = ranks[0]
    out["elems_per_rank"] = r0.elems
    st = r0.stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = {"L1": [], "L2": [], "L3": []}
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record(st)
        for k in range(K):
            r0.begin_chunk(hp, True, 1.0, k) if K > 1 else r0.begin(hp, True, 1.0)
        ev[1].record(st)
        for k in range(K):
            r0.mid_chunk(k) if K > 1 else r0.mid()
        ev[2].record(st)
        r0.end()  # synchronizes
        ev[3].record(st)
        torch.cuda.synchronize()
        for i, key in enumerate(("L1", "L2", "L3")):
            t[key].append(ev[i].elapsed_time(ev[i + 1]))
    out[f"K{K}_ms"] = {k: float(np.median(v)) for k, v in t.items()}
    del ranks
    torch.cuda.empty_cache()
print(out)
