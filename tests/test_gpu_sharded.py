"""Table-wise sharding on the GPU path (§6.7): two ranks,
each with its own ScratchPipe context over its tables, exchange pooled
embeddings and gradients with the all-to-all of bench.py's N>1 path.  The
exchange is pure data movement and the surrogate is element-wise, so every
rank's tables must match the single-process oracle.  Both ranks share cuda:0
here (gloo process group; the driver's GPU box has one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import UncachedTrainer
        from paper_2205_04702_b200 import ScratchPipe
        from paper_2205_04702_b200.sharding import (exchange_backward, exchange_forward, lpt_assign,
                                                    table_weights, tables_of)
        from tests.gpu_helpers import max_window_union, pinned_tables
        from workload import sample_trace
        rows, D, N, L, nb = [3000, 500, 1200, 40, 800], 32, 64, 3, 30
        tr = sample_trace(rows, N, L, 0.95, nb, 77)
        slots_all = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 6) for t, R in enumerate(rows)]
        owner = lpt_assign(table_weights(rows, slots_all, N * L, D), world)
        mine = tables_of(owner, rank)
        torch.cuda.set_device(0)
        tables_all = pinned_tables(rows, D, 4702)
        tables = [tables_all[t] for t in mine]
        sp = ScratchPipe([rows[t] for t in mine], tables, D, [slots_all[t] for t in mine], N, L,
                         index_dtype="int32", index_on_device=True)
        trace = tr[:, mine].to(torch.int32).cuda().contiguous()
        g, d, e = 0.5, 0.01, 0.05
        pooled = torch.empty((len(mine), N, D), device="cuda")
        ahead = sp.F + sp.P + 1
        for j in range(ahead):
            sp.plan_device(trace[j])
        for b in range(nb):
            if b + ahead < nb:
                sp.plan_device(trace[b + ahead])
            elif b + ahead == nb:
                sp.end_of_data()
            sp.forward(pooled)
            pb = exchange_forward(pooled, owner, rank, world)        # [T][N/2][D]
            gb = sp.surrogate(pb, g, d)
            gl = exchange_backward(gb, owner, rank, world, N)         # [T_mine][N][D]
            sp.train(gl.contiguous(), e)
        sp.flush()
        torch.cuda.synchronize()
        orc = UncachedTrainer(rows, D, N, L, 4702)
        for b in range(nb):
            orc.step(tr.numpy()[b], g, d, e)
        worst = 0.0
        for i, t in enumerate(mine):
            touched = orc.touched(t)
            got = tables[i][torch.from_numpy(touched)].numpy()
            want = orc.rows_of(t, touched)
            worst = max(worst, float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-4))))
        sp.close()
        q.put((rank, len(mine), worst, None))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, 0, 1.0, repr(ex)))


def test_two_ranks_tablewise_match_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    for rank, ntab, worst, err in res:
        assert err is None, err
        assert ntab >= 1
        assert worst <= 1e-5, (rank, worst)


@pytest.mark.gpu
def test_library_nccl_exchange_world1_matches_oracle():
    """The library's own sharded path (sp_desc.world / nccl_id: NCCL
    send/recv of every table's rows inside sp_forward / sp_train) at world
    size 1 -- the only size one GPU allows; every message is a self
    send/recv -- gives the oracle's pooled values and final tables."""
    from paper_2205_04702_b200 import nccl_unique_id
    from tests.gpu_helpers import max_window_union, run_parity
    from workload import sample_trace
    rows, D, N, L, nb = [700, 90, 2500], 16, 32, 2, 30
    tr = sample_trace(rows, N, L, 0.9, nb, 91)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 6) for t, R in enumerate(rows)]
    kw = dict(world=1, rank=0, nccl_id=nccl_unique_id(), table_owner=[0, 0, 0], table_ids=[0, 1, 2])
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02), policy_kw=None,
                     sp_kw=kw)
    assert rep["evictions"] > 50
    assert rep["tables"]["max_rel"] <= 1e-5 and rep["tables"]["mismatch"] == 0, rep["tables"]


@pytest.mark.gpu
def test_row_split_virtual_tables_match_unsplit_oracle():
    """SURVEY §8(f) f1 row split: the 20k-row table is cut into 3 row ranges,
    each its own context table (host rows = a sub-range view of the table,
    -1 padding where a lookup falls in another piece).  With one lookup per
    bag the pieces' pooled rows sum exactly to the table's, and the trained
    host table equals the unsplit oracle's, bit for bit."""
    from oracle import UncachedTrainer
    from paper_2205_04702_b200 import ScratchPipe
    from paper_2205_04702_b200.harness import run_loop
    from paper_2205_04702_b200.sharding import combine_pooled, split_trace
    from tests.gpu_helpers import max_window_union, pinned_tables
    from workload import sample_trace
    rows, D, N, L, nb = [20000, 300, 7], 16, 256, 1, 30
    g, d, e = float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 1.0
    tr = sample_trace(rows, N, L, 1.05, nb, 93)
    tables = pinned_tables(rows, D, 4702)
    pieces = [(0, 0, 7000, 0, 1.0), (0, 7000, 13000, 0, 1.0), (0, 13000, 20000, 0, 1.0),
              (1, 0, 300, 0, 1.0), (2, 0, 7, 0, 1.0)]
    vt = split_trace(tr, pieces)
    vrows = [hi - lo for _, lo, hi, _, _ in pieces]
    vslots = [min(R, max_window_union(vt.numpy(), v, 3, 2) + 4) for v, R in enumerate(vrows)]
    views = [tables[t][lo:hi] for t, lo, hi, _, _ in pieces]
    sp = ScratchPipe(vrows, views, D, vslots, N, L, padding=True)
    orc = UncachedTrainer(rows, D, N, L, 4702)
    bad = []

    def on_pooled(b, pooled):
        want = orc.step(tr.numpy()[b], g, d, e, want_pooled=True)
        got = combine_pooled(pooled, pieces, 3).cpu().numpy()
        if not np.array_equal(got, want):
            bad.append(b)
    run_loop(sp, vt, g, d, e, on_pooled=on_pooled)
    assert not bad, bad
    for t in range(3):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        assert np.array_equal(got, orc.rows_of(t, touched)), t
    sp.close()
