"""Multi-GPU host logic: one process per GPU, torch.distributed for the plumbing.

* Candidate sharding (BASELINE config 5): hyperparameter candidates are
  independent — contiguous blocks per rank, no data-path collective, one gather of the small
  per-candidate result records at the end.  Results are bit-identical to a single-GPU sweep
  (each candidate's evaluation does not depend on its batch neighbours; tested).
* Frequency sharding of the per-frequency solves (config 4) uses `freq_slab`: rank r owns the
  contiguous slot range of the four-step row pass, so after the column pass + all-to-all the
  solve and the adjoint are local and only {logdet, quad, dR, deta} are all-reduced.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


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
