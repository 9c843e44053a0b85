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


# ---------------------------------------------------------------- row split
# table-wise sharding of Terabyte caps the link-bound
# speedup near 6x at G = 8 because a few 40M-row tables carry most of the
# misses.  A table split by row range into k "virtual tables" (each its own
# cache manager over the rows [lo, hi)) balances them: the
# seeded Feistel permutation of the trace (reading R16) spreads hot rows
# evenly over the ID range, so each piece sees ~1/k of the table's lookups
# and misses.  A lookup of the table becomes a lookup of exactly one piece
# and -1 (no lookup, SP_FLAG_PADDING) in the others, so with one lookup per
# bag (L = 1, the Criteo shapes) the table's pooled row is the sum of its
# pieces' pooled rows with all but one of them zero -- exact -- and each
# piece's gradient is the table's gradient.

def zipf_miss_weight(rows: Sequence[int], slots: Sequence[int], lookups: int, dim: int,
                     alpha: float, link_only: bool = False) -> List[float]:
    """Per-table cost: Train bytes plus host-link bytes (link_only: the
    host-link bytes alone, the bound of the Criteo shapes), with the miss
    share estimated as 1 - (Zipf(alpha) mass of the S hottest of R rows)."""
    import math

    def H(k):  # generalised harmonic number sum_{r<=k} r^-alpha (integral approximation)
        if abs(alpha - 1.0) < 1e-9:
            return math.log(k + 1.0) + 0.5772
        return ((k + 1.0) ** (1.0 - alpha) - 1.0) / (1.0 - alpha) + 1.0
    out = []
    for R, S in zip(rows, slots):
        miss = 0.0 if S >= R else max(0.0, 1.0 - H(S) / H(R))
        out.append(lookups * dim * ((0.0 if link_only else 1.0) + 2.0 * miss))
    return out


def row_split(rows: Sequence[int], slots: Sequence[int], weights: Sequence[float], world: int,
              factor: float = 4.0):
    """Pieces [(table, row_lo, row_hi, slots, weight)]: a table heavier than
    total / (factor * world) is cut into k equal row ranges so no piece
    exceeds that; slots are split in proportion to rows (at least 1)."""
    total = float(sum(weights))
    cap = total / (factor * max(1, world)) if world > 1 else float("inf")
    pieces = []
    for t, (R, S, w) in enumerate(zip(rows, slots, weights)):
        k = max(1, min(int(R), int(-(-w // cap)) if cap != float("inf") else 1))
        for i in range(k):
            lo, hi = R * i // k, R * (i + 1) // k
            s = min(hi - lo, max(1, -(-S * (hi - lo) // R)))
            pieces.append((t, lo, hi, s, w / k))
    return pieces


def split_trace(trace: torch.Tensor, pieces) -> torch.Tensor:
    """[nb][T][N][L] -> [nb][V][N][L]: piece v = (t, lo, hi) sees id - lo for
    lo <= id < hi and -1 (no lookup) elsewhere.  Input preparation (done once
    per pre-generated trace, like the data loader's sharding)."""
    outs = []
    for t, lo, hi, _, _ in pieces:
        x = trace[:, t]
        inr = (x >= lo) & (x < hi)
        outs.append(torch.where(inr, x - lo, torch.full_like(x, -1)))
    return torch.stack(outs, dim=1).contiguous()


def combine_pooled(pooled_v: torch.Tensor, pieces, num_tables: int) -> torch.Tensor:
    """[V][N][D] pieces -> [T][N][D]: each table's pieces summed in piece
    order (exact for one lookup per bag: all but one addend are zero)."""
    out = torch.zeros((num_tables,) + tuple(pooled_v.shape[1:]), dtype=pooled_v.dtype, device=pooled_v.device)
    for v, (t, _, _, _, _) in enumerate(pieces):
        out[t] += pooled_v[v]
    return out


def expand_grad(grad: torch.Tensor, pieces) -> torch.Tensor:
    """[T][N][D] -> [V][N][D]: every piece receives its table's gradient."""
    return grad[[p[0] for p in pieces]].contiguous()
