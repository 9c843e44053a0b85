"""Table-wise sharding across GPUs (§6.7).

ScratchPipe manages its cache per embedding table ("N embedding tables will
have N instance of ScratchPipe's cache manager module"), and
table-wise model parallelism needs no reordering of lookups and has no
inter-GPU RAW hazards.  So each GPU owns a disjoint set of
tables with its own sp_ctx, and the only cross-GPU step is the all-to-all
that turns table-sharded pooled embeddings [T_g][N][D] into the batch-sharded
layout [T][N/G][D] a data-parallel dense model consumes (and back for the
gradients).  That exchange is pure data movement, so G-GPU results equal
1-GPU results bit for bit.
"""
from __future__ import annotations

from typing import List, Sequence

import torch


def lpt_assign(weights: Sequence[float], world: int) -> List[int]:
    """Greedy longest-processing-time assignment of tables to ranks.
    Deterministic: ties broken by table index, then by rank."""
    order = sorted(range(len(weights)), key=lambda t: (-float(weights[t]), t))
    load = [0.0] * world
    owner = [0] * len(weights)
    for t in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[t] = r
        load[r] += float(weights[t])
    return owner


def table_weights(rows: Sequence[int], slots: Sequence[int], lookups: int, dim: int) -> List[float]:
    """Per-table cost estimate: Train bytes (lookups) plus host-link bytes,
    which only tables that do not fit in their Storage generate."""
    return [lookups * (1.0 + (2.0 if R > S else 0.0)) * dim for R, S in zip(rows, slots)]


def tables_of(owner: Sequence[int], rank: int) -> List[int]:
    return [t for t, r in enumerate(owner) if r == rank]


def _all_to_all(recv, send, counts_in, counts_out, group):
    """all_to_all_single; over a backend without CUDA all-to-all (gloo, used by
    the tests to run several ranks on one GPU) the buffers go through host
    memory.  NCCL moves CUDA tensors directly over NVLink."""
    import torch.distributed as dist
    if send.is_cuda and dist.get_backend(group) != "nccl":
        r = recv.cpu()
        dist.all_to_all_single(r, send.cpu(), counts_in, counts_out, group=group)
        recv.copy_(r)
    else:
        dist.all_to_all_single(recv, send, counts_in, counts_out, group=group)


def _split_bags(N: int, world: int) -> List[int]:
    base, rem = divmod(N, world)
    return [base + (1 if r < rem else 0) for r in range(world)]


def exchange_forward(pooled_local: torch.Tensor, owner: Sequence[int], rank: int, world: int,
                     group=None) -> torch.Tensor:
    """[T_g][N][D] (this rank's tables, ascending table id) -> [T][N_r][D]
    (all tables, this rank's slice of the batch), via one all_to_all."""
    Tg, N, D = pooled_local.shape
    nb = _split_bags(N, world)
    send = torch.cat([pooled_local[:, sum(nb[:h]):sum(nb[:h + 1])].reshape(-1) for h in range(world)])
    counts_in = [len(tables_of(owner, h)) * nb[rank] * D for h in range(world)]
    counts_out = [Tg * nb[h] * D for h in range(world)]
    recv = send.new_empty(sum(counts_in))
    _all_to_all(recv, send, counts_in, counts_out, group)
    out = recv.new_empty((len(owner), nb[rank], D))
    off = 0
    for h in range(world):
        th = tables_of(owner, h)
        k = len(th) * nb[rank] * D
        if th:
            out[th] = recv[off:off + k].view(len(th), nb[rank], D)
        off += k
    return out


def exchange_backward(grad_batch: torch.Tensor, owner: Sequence[int], rank: int, world: int,
                      N: int, group=None) -> torch.Tensor:
    """Inverse of exchange_forward: [T][N_r][D] -> [T_g][N][D]."""
    T, Nr, D = grad_batch.shape
    nb = _split_bags(N, world)
    mine = tables_of(owner, rank)
    send = torch.cat([grad_batch[tables_of(owner, h)].reshape(-1) for h in range(world)])
    counts_out = [len(tables_of(owner, h)) * Nr * D for h in range(world)]
    counts_in = [len(mine) * nb[h] * D for h in range(world)]
    recv = send.new_empty(sum(counts_in))
    _all_to_all(recv, send, counts_in, counts_out, group)
    out = recv.new_empty((len(mine), N, D))
    off = 0
    for h in range(world):
        k = len(mine) * nb[h] * D
        out[:, sum(nb[:h]):sum(nb[:h + 1])] = recv[off:off + k].view(len(mine), nb[h], D)
        off += k
    return out
