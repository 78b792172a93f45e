"""The frequency-sharded fused lattice fit with REAL ranks: two processes, each
running its own fmtgp_shard_{begin,mid,end} phases (its column blocks and row clusters) on the
device, exchanging the exchange blocks with torch.distributed all_to_all_single and the records
with all_gather (gloo, staged through host memory — the pool gives one GPU per job, so both
processes share cuda:0; no kernel of one rank waits on the other, the exchanges are host-side
between phases).  Every rank's result must equal the unsharded one-process fit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2603_16014_b200 import configs
    inst = configs.make(4, m=[18, 18])
    return inst.design, inst.hyper, inst.y


def _worker(rank, world, chunks, port, q):
    import torch.distributed as dist

    from paper_2603_16014_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dz, hp, y = _case()
        shard = sharding.ShardedLatticeFit(dz, rank, world, device=0, chunks=chunks)
        shard.set_y(y)
        res = sharding.sharded_nll([shard], hp, grad=True, exchange=sharding.host_exchange(shard),
                                   gather=sharding.host_gather(shard))
        q.put((rank, {k: np.asarray(res[k]) for k in ("nll", "logdet", "deta", "dB", "dt", "dgamma")}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks", [(2, 1), (4, 1), (2, 4)])
def test_sharded_fit_real_ranks(world, chunks):
    from paper_2603_16014_b200.fast_gram import Model
    dz, hp, y = _case()
    M = Model(dz)
    M.set_y(y)
    want = M.nll(hp, grad=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, chunks, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        g = got[r]
        assert abs(float(g["nll"]) - want["nll"]) <= 1e-11 * abs(want["nll"])
        assert abs(float(g["logdet"]) - want["logdet"]) <= 1e-11 * abs(want["logdet"])
        for k in ("deta", "dB", "dt"):
            assert np.linalg.norm(g[k] - np.asarray(want[k])) <= 1e-9 * max(1.0, np.linalg.norm(want[k])), k
