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


# ---- the library's own sharded exchange (sp_shard_plan: the message lists
# sp_forward / sp_train post to NCCL), checked on the host


def _simulate(world, owner, T_all, N, D, seed):
    """Run every rank's message list through NCCL's pairing rule (the k-th
    send from i to j meets the k-th receive on j from i) on host arrays."""
    from paper_2205_04702_b200 import shard_plan
    rng = np.random.default_rng(seed)
    full = rng.standard_normal((T_all, N, D)).astype(np.float32)
    Ns = N // world
    plans = [shard_plan(world, r, owner) for r in range(world)]
    mine = [[t for t in range(T_all) if owner[t] == r] for r in range(world)]
    local = [full[m] for m in mine]                       # [T_r][N][D] on rank r
    out = [np.full((T_all, Ns, D), np.nan, np.float32) for _ in range(world)]
    queues = {}
    for r, (snd, _) in enumerate(plans):                  # posted sends, per (src, dst) in order
        for peer, tl, tg in snd:
            assert mine[r][tl] == tg
            queues.setdefault((r, peer), []).append(local[r][tl, peer * Ns:(peer + 1) * Ns])
    for r, (_, rcv) in enumerate(plans):
        for peer, tg in rcv:
            out[r][tg] = queues[(peer, r)].pop(0)
    assert all(len(v) == 0 for v in queues.values())
    for r in range(world):                                # forward: the batch shard of every table
        assert np.array_equal(out[r], full[:, r * Ns:(r + 1) * Ns])
    # backward: the mirror image (receives become sends) rebuilds [T_r][N][D]
    back = [np.full_like(local[r], np.nan) for r in range(world)]
    queues = {}
    for r, (_, rcv) in enumerate(plans):
        for peer, tg in rcv:
            queues.setdefault((r, peer), []).append(out[r][tg] * 2 + 1)
    for r, (snd, _) in enumerate(plans):
        for peer, tl, tg in snd:
            back[r][tl, peer * Ns:(peer + 1) * Ns] = queues[(peer, r)].pop(0)
    for r in range(world):
        assert np.array_equal(back[r], full[mine[r]] * 2 + 1)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_library_shard_plan_pairs_and_layout(world):
    T_all = 26
    for seed in range(3):
        owner = lpt_assign(list(np.random.default_rng(seed).integers(1, 100, T_all)), world)
        _simulate(world, owner, T_all, 8 * world, 4, seed)


def test_library_shard_plan_rejects_bad_maps():
    from paper_2205_04702_b200 import SpError, shard_plan
    with pytest.raises(SpError):
        shard_plan(2, 0, [0, 2])          # owner out of range
    with pytest.raises(SpError):
        shard_plan(2, 2, [0, 1])          # rank out of range


def _lib_plan_worker(rank, world, port, q):
    """Two processes post the library's message lists through gloo P2P in the
    listed order (as sp_forward / sp_train post them to NCCL)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2205_04702_b200 import shard_plan
    T_all, N, D = 7, 6, 3
    owner = lpt_assign([9, 1, 4, 4, 2, 8, 3], world)
    full = torch.arange(T_all * N * D, dtype=torch.float32).view(T_all, N, D)
    mine = [t for t in range(T_all) if owner[t] == rank]
    local = full[mine].contiguous()
    Ns = N // world
    snd, rcv = shard_plan(world, rank, owner)
    out = torch.empty(T_all, Ns, D)
    reqs = []
    for peer, tl, tg in snd:
        buf = local[tl, peer * Ns:(peer + 1) * Ns].contiguous()
        reqs.append(dist.isend(buf, peer) if peer != rank else None)
        if peer == rank:
            out[tg] = buf
    for peer, tg in rcv:
        if peer != rank:
            r = torch.empty(Ns, D)
            dist.recv(r, peer)
            out[tg] = r
    for r in reqs:
        if r is not None:
            r.wait()
    q.put((rank, bool(torch.equal(out, full[:, rank * Ns:(rank + 1) * Ns]))))
    dist.destroy_process_group()


def test_gloo_world2_library_message_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_lib_plan_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


# ---- row split of the heaviest tables
from paper_2205_04702_b200.sharding import (combine_pooled, expand_grad, row_split, split_trace,  # noqa: E402
                                            zipf_miss_weight)


def test_row_split_covers_rows_and_balances_terabyte():
    from workload import CONFIGS
    c = CONFIGS["terabyte"]
    w = zipf_miss_weight(c.rows, c.slots, c.batch * c.pooling, c.dim, c.alpha, link_only=True)
    for G in (2, 4, 8):
        pieces = row_split(c.rows, c.slots, w, G)
        for t, R in enumerate(c.rows):   # every row of every table in exactly one piece
            rng = sorted((lo, hi) for tt, lo, hi, _, _ in pieces if tt == t)
            assert rng[0][0] == 0 and rng[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
        assert sum(p[3] for p in pieces) >= sum(c.slots)
        whole = lpt_assign(w, G)
        split = lpt_assign([p[4] for p in pieces], G)
        lw = [sum(x for x, r in zip(w, whole) if r == k) for k in range(G)]
        ls = [sum(p[4] for p, r in zip(pieces, split) if r == k) for k in range(G)]
        # the speedup cap sum/max does not get worse, and is within 30% of the ideal G
        assert sum(ls) / max(ls) >= 0.98 * sum(lw) / max(lw)   # (LPT is greedy: not monotone)
        assert sum(ls) / max(ls) >= 0.7 * G, (G, sum(ls) / max(ls))


def test_split_trace_combine_is_exact_for_one_lookup_per_bag():
    rows, N, D = [1000, 7], 16, 4
    gen = torch.Generator().manual_seed(3)
    trace = torch.stack([torch.randint(0, 1000, (5, N, 1), generator=gen),
                         torch.randint(0, 7, (5, N, 1), generator=gen)], dim=1)
    pieces = [(0, 0, 300, 10, 1.0), (0, 300, 1000, 20, 1.0), (1, 0, 7, 7, 1.0)]
    vt = split_trace(trace, pieces)
    assert vt.shape == (5, 3, N, 1)
    # exactly one piece holds each lookup of table 0, shifted by its lo
    hit = (vt[:, :2] >= 0).sum(dim=1)
    assert torch.all(hit == 1)
    back = torch.where(vt[:, 0] >= 0, vt[:, 0], vt[:, 1] + 300)
    assert torch.equal(back, trace[:, 0])
    # pooled: a row table E, pooled_v = E[lo + id] or 0 -> combined == E[id]
    E = torch.randn(1000, D)
    pv = []
    for v, (_, lo, _, _, _) in enumerate(pieces[:2]):
        ids = vt[0, v, :, 0]
        pv.append(torch.where((ids >= 0).unsqueeze(1), E[(ids + lo).clamp(0, 999)], torch.zeros(N, D)))
    pv = torch.stack(pv)
    pv = torch.cat([pv, torch.zeros(1, N, D)])
    comb = combine_pooled(pv, pieces, 2)
    assert torch.equal(comb[0], E[trace[0, 0, :, 0]])
    g = torch.randn(2, N, D)
    ge = expand_grad(g, pieces)
    assert torch.equal(ge[0], g[0]) and torch.equal(ge[1], g[0]) and torch.equal(ge[2], g[1])
