"""Multi-GPU host logic: one process per GPU, torch.distributed for the plumbing.

* Candidate sharding (BASELINE config 5): hyperparameter candidates are
  independent — contiguous blocks per rank, no data-path collective, one gather of the small
  per-candidate result records at the end.  Results are bit-identical to a single-GPU sweep
  (each candidate's evaluation does not depend on its batch neighbours; tested).
* Frequency sharding of the fused lattice fit (config 4, `sharded_nll`): rank r owns a block of
  column tiles of the four-step column passes and a block of row clusters (Hermitian partner row
  pairs) of the row pass.  Per evaluation: column pass -> all-to-all -> row FFT + per-frequency
  solve + inverse row FFT -> all-to-all -> inverse column pass + gradient dot -> one gather of
  the 101-double records, summed in rank order (deterministic).  The three phases are the
  library's fmtgp_shard_{begin,mid,end} (include/fastmtgp_b200.h); the exchanges are
  torch.distributed all_to_all_single (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Sequence, Tuple

import numpy as np

from ._lib import ERR_NONREAL, ERR_SCHUR, SHARD_REC_LEN, CResult, FastMtgpError, SchurBreakdown, check
from .fast_gram import _result


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [start, stop) of n items for `rank` (first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def freq_slab(nrows: int, world: int, rank: int) -> Tuple[int, int]:
    """Rows of the four-step row pass owned by `rank` (row pairs k1, N1-k1 stay together)."""
    npairs = nrows // 2  # cluster index q owns rows {q, N1-q} (q = 0 owns {0, N1/2})
    a, b = shard_range(npairs, world, rank)
    return a, b


def sweep(evaluate: Callable[[Sequence], List[dict]], candidates: Sequence, world: int = 1, rank: int = 0,
          group=None) -> List[dict]:
    """Evaluate `candidates` sharded over `world` ranks; every rank returns all results in
    candidate order.  `evaluate` is e.g. ``Model.nll_batch`` (GPU) or an oracle (tests)."""
    start, stop = shard_range(len(candidates), world, rank)
    local = list(evaluate(candidates[start:stop])) if stop > start else []
    if world == 1:
        return local
    import torch.distributed as dist
    gathered: List[List[dict]] = [None] * world  # type: ignore[list-item]
    dist.all_gather_object(gathered, local, group=group)
    out: List[dict] = []
    for part in gathered:
        out.extend(part)
    return out


def sharded_posterior_var(evaluate: Callable[[np.ndarray], np.ndarray], X, world: int = 1, rank: int = 0,
                          group=None) -> np.ndarray:
    """Posterior variance at the rows of X sharded over `world` ranks (BASELINE config 3, SURVEY.md
    §8e): the test points are independent — contiguous blocks per rank, `evaluate(X_block)` (e.g.
    ``lambda Xb: model.posterior_var(task, Xb)``, each rank's model holding the same fit), one
    all-gather of the variances.  Every rank returns all values in point order, bit-identical to
    one process (each query's fold is independent of its batch neighbours)."""
    X = np.asarray(X, dtype=np.float64)
    start, stop = shard_range(len(X), world, rank)
    local = np.asarray(evaluate(X[start:stop]), dtype=np.float64) if stop > start else np.empty(0)
    if world == 1:
        return local
    import torch.distributed as dist
    gathered: List[np.ndarray] = [None] * world  # type: ignore[list-item]
    dist.all_gather_object(gathered, local, group=group)
    return np.concatenate(gathered)


# ----------------------------------------------------------------------------- frequency sharding
NOUT = 4 + 16 + 8 * 8  # result record (csrc/kernels.cuh OUT_*)


def combine_records(recs) -> "np.ndarray":
    """Rank-order sum of the NOUT sums, min of the first failing slot, max of the per-stage
    non-real maxima (fmtgp_shard_end's record layout)."""
    recs = [np.asarray(r, dtype=np.float64) for r in recs]
    out = recs[0].copy()
    for r in recs[1:]:
        out[:NOUT] += r[:NOUT]
        out[NOUT] = min(out[NOUT], r[NOUT])
        out[NOUT + 1:] = np.maximum(out[NOUT + 1:], r[NOUT + 1:])
    return out


class ShardedLatticeFit:
    """One rank of the frequency-sharded fused lattice fit (equal n, n >= 2^17, T <= 4).

    `exchange(send, recv)` is an all-to-all of `world` equal chunks (default: torch.distributed
    all_to_all_single on the model's stream) and `gather(rec)` returns every rank's record in
    rank order (default: torch.distributed.all_gather).  Both are injectable so the same
    orchestration runs with virtual ranks on one device (tests).

    `chunks` > 1 pipelines each all-to-all (fmtgp_shard_chunks): L1 runs per column chunk and L2
    per row chunk, and chunk k's all-to-all runs on a separate communication stream under chunk
    k+1's kernel (buffers: 0 = L1 out / L2 out, 1 = forward receive, 2 = return receive)."""

    def __init__(self, design, rank: int, world: int, device: int = 0, model=None, chunks: int = 1):
        import torch

        from .fast_gram import Model

        self.rank, self.world = rank, world
        self.model = model if model is not None else Model(design, device=device)
        n = C.c_int64()
        check(self.model.lib.fmtgp_shard_setup(self.model.h, rank, world, C.byref(n)))
        self.elems = int(n.value)  # complex values per exchange buffer
        self.chunks = int(chunks)
        if self.chunks > 1:
            check(self.model.lib.fmtgp_shard_chunks(self.model.h, self.chunks))
        dev = torch.device("cuda", device)
        self.bufs = [torch.empty(2 * self.elems, dtype=torch.float64, device=dev)
                     for _ in range(2 if self.chunks == 1 else 3)]
        self.stream = torch.cuda.ExternalStream(self.model.stream, device=dev)
        self.comm = torch.cuda.Stream(device=dev) if self.chunks > 1 else self.stream

    def region(self, b: int, k: int):
        """Chunk k of buffer b (a contiguous view: `world` equal blocks of exchange_elems / chunks)."""
        return self.bufs[b].view(self.chunks, -1)[k]

    def set_y(self, y):
        self.model.set_y(y)

    # -- the three phases (asynchronous on the model's stream except `end`)
    def begin(self, hp, grad: bool, xi_scale: float):
        ch = self.model._hyper_struct(hp)
        check(self.model.lib.fmtgp_shard_begin(self.model.h, C.byref(ch), int(grad), float(xi_scale),
                                               C.c_void_p(self.bufs[0].data_ptr())))
        return self.bufs[0]

    def mid(self):
        check(self.model.lib.fmtgp_shard_mid(self.model.h, C.c_void_p(self.bufs[1].data_ptr())))
        return self.bufs[1]

    def begin_chunk(self, hp, grad: bool, xi_scale: float, k: int):
        ch = self.model._hyper_struct(hp)
        check(self.model.lib.fmtgp_shard_begin_chunk(self.model.h, C.byref(ch), int(grad), float(xi_scale),
                                                     C.c_void_p(self.bufs[0].data_ptr()), int(k)))
        return self.region(0, k)

    def mid_chunk(self, k: int):
        check(self.model.lib.fmtgp_shard_mid_chunk(self.model.h, C.c_void_p(self.bufs[1].data_ptr()),
                                                   C.c_void_p(self.bufs[0].data_ptr()), int(k)))
        return self.region(0, k)

    def end(self):
        rec = np.zeros(SHARD_REC_LEN)
        back = self.bufs[0 if self.chunks == 1 else 2]
        check(self.model.lib.fmtgp_shard_end(self.model.h, C.c_void_p(back.data_ptr()),
                                             rec.ctypes.data_as(C.POINTER(C.c_double))))
        return rec

    def finish(self, hp, rec, grad: bool, xi_scale: float, escalations: int):
        ch = self.model._hyper_struct(hp)
        r = CResult()
        rec = np.ascontiguousarray(rec, dtype=np.float64)
        check(self.model.lib.fmtgp_shard_finish(self.model.h, C.byref(ch), rec.ctypes.data_as(C.POINTER(C.c_double)),
                                                int(grad), float(xi_scale), int(escalations), C.byref(r)))
        return _result(r, self.model.design, hp)

    def default_exchange(self, send, recv, group=None):
        """NCCL all-to-all ordered after the work queued so far on the model's stream; with chunks
        it runs on the communication stream (so the next chunk's kernel overlaps it) until join()."""
        import torch
        import torch.distributed as dist
        if self.comm is not self.stream:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            dist.all_to_all_single(recv, send, group=group)

    def join(self):
        """The model's stream waits for every exchange issued so far."""
        if self.comm is not self.stream:
            import torch
            ev = torch.cuda.Event()
            ev.record(self.comm)
            self.stream.wait_event(ev)

    def default_gather(self, rec, group=None):
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(np.asarray(rec, dtype=np.float64)).to(self.bufs[0].device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=group)
        return [o.cpu().numpy() for o in out]


def sharded_nll(ranks, hp, grad: bool = True, exchange=None, gather=None, max_retries: int = 6):
    """Frequency-sharded NLL (+ gradient) with the reference's escalation schedule
    (xi x 10 per SchurBreakdown, at most 6 retries, gp_core.cpp:98-127).

    `ranks` is this process's ShardedLatticeFit (one element, multi-process) or all of them
    (virtual ranks on one device, in which case `exchange` / `gather` act on the list)."""
    local = list(ranks)
    K = getattr(local[0], "chunks", 1)
    join = getattr(exchange, "join", None) or (lambda: None)
    scale, attempt = 1.0, 0
    while True:
        if K == 1:
            sends = [r.begin(hp, grad, scale) for r in local]
            exchange(sends, [r.bufs[1] for r in local])  # column blocks -> row owners
            mids = [r.mid() for r in local]
            exchange(mids, [r.bufs[0] for r in local])  # row blocks -> column owners
        else:  # pipelined: chunk k's all-to-all under chunk k+1's kernel
            for k in range(K):
                sends = [r.begin_chunk(hp, grad, scale, k) for r in local]
                exchange(sends, [r.region(1, k) for r in local])
            join()  # L2 needs every forward chunk
            for k in range(K):
                outs = [r.mid_chunk(k) for r in local]
                exchange(outs, [r.region(2, k) for r in local])
        join()
        recs = [r.end() for r in local]
        allrec = gather(recs)
        rec = combine_records(allrec)
        res = local[0].finish(hp, rec, grad, scale, attempt)
        if res["status"] == ERR_SCHUR and attempt < max_retries:
            scale *= 10.0
            attempt += 1
            continue
        if res["status"] == ERR_SCHUR:  # as fmtgp_nll: schedule exhausted
            raise SchurBreakdown("noise escalation schedule exhausted")
        if res["status"] == ERR_NONREAL:
            raise FastMtgpError("invert_and_logdet: non-real Schur complement")
        return res


def local_exchange(world: int):
    """All-to-all among virtual ranks on one device: block h of rank g's send buffer -> block g
    of rank h's receive buffer (each rank's buffer = `world` equal chunks)."""
    def ex(sends, recvs):
        import torch
        torch.cuda.synchronize()
        chunks = [s.view(world, -1) for s in sends]
        for h in range(world):
            rv = recvs[h].view(world, -1)
            for g in range(world):
                rv[g].copy_(chunks[g][h])
        torch.cuda.synchronize()
    return ex


def dist_exchange(rank_obj, group=None):
    """Multi-process all-to-all (torch.distributed; NCCL on GPUs), ordered after the model's
    stream; `ex.join()` orders the model's stream after it (chunked exchanges)."""
    def ex(sends, recvs):
        rank_obj.default_exchange(sends[0], recvs[0], group)
    ex.join = rank_obj.join
    return ex


def host_exchange(rank_obj, group=None):
    """All-to-all staged through host memory (gloo's CPU all_to_all_single): for process groups
    without a device transport (the CPU-plumbing tests of the real shard phases)."""
    def ex(sends, recvs):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        s, r = sends[0].cpu(), torch.empty_like(sends[0], device="cpu")
        dist.all_to_all_single(r, s, group=group)
        recvs[0].copy_(r)
        torch.cuda.synchronize()
    return ex


def host_gather(rank_obj, group=None):
    def ga(recs):
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(np.asarray(recs[0], dtype=np.float64))
        out = [torch.empty_like(t) for _ in range(rank_obj.world)]
        dist.all_gather(out, t, group=group)
        return [o.numpy() for o in out]
    return ga


def dist_gather(rank_obj, group=None):
    def ga(recs):
        return rank_obj.default_gather(recs[0], group)
    return ga
