"""Table-wise sharding (§6.7): host logic and the
all-to-all layout, on CPU with world_size-2 gloo process groups.

The exchange is pure data movement, so the batch-sharded pooled embeddings
(and the gradients sent back) must equal slices of the single-process result
bit for bit; the per-table values come from the oracle (Part A) here, since
this container has no GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_04702_b200.sharding import (exchange_backward, exchange_forward, lpt_assign,
                                            table_weights, tables_of)


def test_lpt_is_deterministic_and_balanced():
    w = [5, 3, 3, 2, 2, 2, 1]
    a = lpt_assign(w, 2)
    assert a == lpt_assign(w, 2)
    loads = [sum(x for x, r in zip(w, a) if r == k) for k in range(2)]
    assert max(loads) - min(loads) <= max(w)
    assert sorted(set(a)) == [0, 1]
    # a table that fits its Storage (R == S) weighs less than one that misses
    tw = table_weights([100, 100], [100, 10], 8, 4)
    assert tw[1] > tw[0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, N, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    owner = lpt_assign([7, 1, 4, 4, 2][:T], world)
    gen = torch.Generator().manual_seed(11)
    full = torch.randn(T, N, D, generator=gen)           # what one GPU would produce
    mine = tables_of(owner, rank)
    local = full[mine].contiguous()                      # this rank's tables, all bags
    out = exchange_forward(local, owner, rank, world)     # -> all tables, my bag slice
    nb = [N // world + (1 if r < N % world else 0) for r in range(world)]
    lo = sum(nb[:rank])
    ok_fwd = torch.equal(out, full[:, lo:lo + nb[rank]])
    g = out * 2 + 1                                       # "MLP" on the batch shard
    back = exchange_backward(g.contiguous(), owner, rank, world, N)
    ok_bwd = torch.equal(back, (full * 2 + 1)[mine])
    q.put((rank, bool(ok_fwd), bool(ok_bwd)))
    dist.destroy_process_group()


@pytest.mark.parametrize("T,N", [(5, 8), (3, 7), (2, 5)])
def test_gloo_world2_exchange_is_exact(T, N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, T, N, 4, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] and r[2] for r in res), res


def _oracle_worker(rank, world, port, q):
    """Each rank trains ITS tables with the oracle (standing in for its GPU
    context); the exchanged pooled values equal the single-process oracle's."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import UncachedTrainer
    from workload import sample_trace
    rows, D, N, L = [50, 80, 30], 4, 6, 2
    tr = sample_trace(rows, N, L, 1.0, 3, 4).numpy()
    owner = lpt_assign(table_weights(rows, rows, N * L, D), world)
    mine = tables_of(owner, rank)
    orc = UncachedTrainer([rows[t] for t in mine], D, N, L, 4702, table_ids=mine) if mine else None
    ok = True
    full_ref = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(3):
        want = full_ref.step(tr[b], 0.5, 0.01, 0.01, want_pooled=True)
        local = torch.from_numpy(orc.step(tr[b][mine], 0.5, 0.01, 0.01, want_pooled=True)) if mine \
            else torch.empty((0, N, D))
        out = exchange_forward(local, owner, rank, world)
        nb = [N // world + (1 if r < N % world else 0) for r in range(world)]
        lo = sum(nb[:rank])
        ok &= bool(np.array_equal(out.numpy(), want[:, lo:lo + nb[rank]]))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_gloo_world2_sharded_training_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_oracle_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
