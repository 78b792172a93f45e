"""Multi-process host logic on CPU (gloo, world_size 2): candidate sharding of the config-5
sweep returns, on every rank, exactly the single-process results in candidate order."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_16014_b200 import configs, sharding


def test_shard_range_partitions():
    for n in (0, 1, 5, 256, 257):
        for world in (1, 2, 3, 8):
            spans = [sharding.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        sharding.shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_eval(inst):
    from oracle import port

    def ev(cands):
        return [{"nll": port.fit(inst.design, h, inst.y)["nll"]} for h in cands]
    return ev


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = configs.make(5, m=[3] * 4, n_cand=7)
        res = sharding.sweep(_oracle_eval(inst), inst.candidates, world=world, rank=rank)
        q.put((rank, [r["nll"] for r in res]))
    finally:
        dist.destroy_process_group()


def test_candidate_sweep_gloo_world2(port):
    inst = configs.make(5, m=[3] * 4, n_cand=7)
    want = [r["nll"] for r in sharding.sweep(_oracle_eval(inst), inst.candidates)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for r in range(2):
        assert np.array_equal(np.array(got[r]), np.array(want))
