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


def _var_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = np.random.default_rng(3).random((37, 8))
        res = sharding.sharded_posterior_var(_fake_var, X, world=world, rank=rank)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _fake_var(Xb):
    # stands in for Model.posterior_var: a per-point function (the GPU numerics are checked
    # against the reference in tests/test_gpu_parity.py and test_gpu_seam_dropin.py)
    return np.cos(Xb).prod(axis=1) - 0.5 * Xb[:, 0]


def test_posterior_var_sharding_gloo_world2():
    """Config-3 test-point sharding: every rank gets all variances in point order,
    identical to one process."""
    X = np.random.default_rng(3).random((37, 8))
    want = sharding.sharded_posterior_var(_fake_var, X)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_var_worker, args=(r, 2, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for r in range(2):
        assert np.array_equal(got[r], want)


# ----------------------------------------------------------------------------- frequency sharding
# The orchestration of sharding.sharded_nll (two all-to-alls of exchange blocks + a rank-order
# record combine + the escalation loop) over real gloo all_to_all_single, world size 2.  The CUDA
# phases are replaced by a fake rank that stamps every exchange element with (source rank,
# destination rank, class, local row, local column) and checks the stamps it receives: the
# numerics of the phases are checked against the unsharded fit on the GPU (virtual ranks,
# tests/test_gpu_lattice_fused.py).
class _FakeRank:
    V, R, WC = 2, 3, 4  # classes, rows per rank, columns per rank

    def __init__(self, rank, world):
        import torch
        self.rank, self.world = rank, world
        self.elems = self.V * self.R * self.WC * world
        self.bufs = [torch.zeros(2 * self.elems, dtype=torch.float64) for _ in range(2)]
        self.calls = 0

    def _stamp(self, src, dst, o, i, jl, phase):
        return float(((((phase * 8 + src) * 8 + dst) * 4 + o) * 8 + i) * 8 + jl)

    def _fill(self, buf, phase, row_owner_is_dest):
        v = buf.view(self.world, self.V, self.R, self.WC, 2)
        for h in range(self.world):
            for o in range(self.V):
                for i in range(self.R):
                    for jl in range(self.WC):
                        v[h, o, i, jl, 0] = self._stamp(self.rank, h, o, i, jl, phase)
                        v[h, o, i, jl, 1] = -1.0

    def _check(self, buf, phase):
        v = buf.view(self.world, self.V, self.R, self.WC, 2)
        for s in range(self.world):
            for o in range(self.V):
                for i in range(self.R):
                    for jl in range(self.WC):
                        assert v[s, o, i, jl, 0].item() == self._stamp(s, self.rank, o, i, jl, phase)

    def begin(self, hp, grad, xi_scale):
        self.scale = xi_scale
        self._fill(self.bufs[0], 1, True)
        return self.bufs[0]

    def mid(self):
        self._check(self.bufs[1], 1)  # block s came from rank s, addressed to me
        self._fill(self.bufs[1], 2, False)
        return self.bufs[1]

    def end(self):
        self._check(self.bufs[0], 2)
        return self._rec()

    def _rec(self):
        rec = np.zeros(sharding.NOUT + 1 + 16)
        rec[: sharding.NOUT] = np.arange(sharding.NOUT) * (self.rank + 1)
        rec[sharding.NOUT] = 0x7f7f7f7f if self.scale >= 100.0 else 5 + self.rank  # Schur until xi x 100
        rec[sharding.NOUT + 1:] = self.rank
        return rec

    def finish(self, hp, rec, grad, xi_scale, escalations):
        from paper_2603_16014_b200._lib import ERR_SCHUR, OK
        self.calls += 1
        return {"status": ERR_SCHUR if rec[sharding.NOUT] != 0x7f7f7f7f else OK, "rec": rec,
                "xi_scale": xi_scale, "escalations": escalations}


class _FakeChunkedRank(_FakeRank):
    """The pipelined exchange (chunks = 2): forward blocks column-chunked [kc][h][o][i][jl'],
    return blocks row-chunked [kr][h][o][i'][jl], three buffers (fmtgp_shard_chunks layouts)."""
    V, R, WC = 2, 4, 4
    chunks = 2

    def __init__(self, rank, world):
        import torch
        super().__init__(rank, world)
        self.bufs.append(torch.zeros(2 * self.elems, dtype=torch.float64))
        self.log = []

    def region(self, b, k):
        return self.bufs[b].view(self.chunks, -1)[k]

    def begin_chunk(self, hp, grad, xi_scale, k):
        self.scale = xi_scale
        self.log.append(("begin", k))
        wk = self.WC // self.chunks
        v = self.region(0, k).view(self.world, self.V, self.R, wk, 2)
        for h in range(self.world):
            for o in range(self.V):
                for i in range(self.R):
                    for j in range(wk):
                        v[h, o, i, j, 0] = self._stamp(self.rank, h, o, i, k * wk + j, 1)
        return self.region(0, k)

    def mid_chunk(self, k):
        self.log.append(("mid", k))
        wk, rk = self.WC // self.chunks, self.R // self.chunks
        if k == 0:  # every forward chunk has arrived before the first row chunk
            for kc in range(self.chunks):
                v = self.region(1, kc).view(self.world, self.V, self.R, wk, 2)
                for s in range(self.world):
                    for o in range(self.V):
                        for i in range(self.R):
                            for j in range(wk):
                                assert v[s, o, i, j, 0].item() == self._stamp(s, self.rank, o, i, kc * wk + j, 1)
        v = self.region(0, k).view(self.world, self.V, rk, self.WC, 2)
        for h in range(self.world):
            for o in range(self.V):
                for i in range(rk):
                    for jl in range(self.WC):
                        v[h, o, i, jl, 0] = self._stamp(self.rank, h, o, k * rk + i, jl, 2)
        return self.region(0, k)

    def end(self):
        rk = self.R // self.chunks
        for kr in range(self.chunks):
            v = self.region(2, kr).view(self.world, self.V, rk, self.WC, 2)
            for s in range(self.world):
                for o in range(self.V):
                    for i in range(rk):
                        for jl in range(self.WC):
                            assert v[s, o, i, jl, 0].item() == self._stamp(s, self.rank, o, kr * rk + i, jl, 2)
        assert self.log[-2 * self.chunks:] == [("begin", 0), ("begin", 1), ("mid", 0), ("mid", 1)]
        return self._rec()


def _shard_worker(rank, world, port, q, chunked=False):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fr = (_FakeChunkedRank if chunked else _FakeRank)(rank, world)

        def ex(sends, recvs):
            dist.all_to_all_single(recvs[0], sends[0])

        def ga(recs):
            t = torch.from_numpy(recs[0])
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return [o.numpy() for o in out]

        res = sharding.sharded_nll([fr], None, grad=True, exchange=ex, gather=ga)
        q.put((rank, res["rec"].tolist(), res["xi_scale"], res["escalations"]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunked", [False, True], ids=["whole", "chunked"])
def test_sharded_nll_orchestration_gloo_world2(chunked):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, p, q, chunked)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    nout = sharding.NOUT
    for rank, rec, scale, esc in out:
        assert not isinstance(rec, str), rec
        rec = np.asarray(rec)
        assert np.array_equal(rec[:nout], np.arange(nout) * 3.0)  # rank-order sum of 1x and 2x
        assert rec[nout] == 0x7f7f7f7f and np.all(rec[nout + 1:] == 1.0)  # min of flags, max of maxima
        assert scale == 100.0 and esc == 2  # two escalations (xi x 10 each), as gp_core.cpp:98-127


def test_combine_records_rank_order():
    a = np.zeros(sharding.NOUT + 17)
    b = a.copy()
    a[:3], b[:3] = [1.0, 2.0, 3.0], [0.5, 0.25, 0.125]
    a[sharding.NOUT], b[sharding.NOUT] = 9.0, 4.0
    a[sharding.NOUT + 1], b[sharding.NOUT + 1] = 1e-9, 2e-9
    c = sharding.combine_records([a, b])
    assert list(c[:3]) == [1.5, 2.25, 3.125] and c[sharding.NOUT] == 4.0 and c[sharding.NOUT + 1] == 2e-9
