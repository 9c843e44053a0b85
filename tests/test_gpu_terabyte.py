"""GPU parity at the Criteo-Terabyte shape (BASELINE configs[2], the bench
headline) against the oracle.

The full 26 MLPerf Criteo-1TB cardinalities (largest 39,979,771 rows: 26-bit
keys, four 8-bit radix passes in the dedup CTA), D = 128, N = 4096, L = 1,
Zipf 1.05, 96 GB of host tables (sp_host_alloc: THP + registered), the GPU
pull transfer mode (the default above 32 MB of rows per batch).  Storage is
sized just above each table's window working set so evictions start within
the first checked batches (the bench's 5% would take thousands of batches).

* per-call API, 24 batches: every Plan record bit-exact (U, hit/miss, victim
  slots, evicted IDs) for every (b, t), every pooled output bit-exact, sampled
  final rows within 1e-5;
* graph mode (sp_run_steps, the launch configuration bench.py times), 2,000
  batches with a one-slot-per-slot LRU log (log_factor = 1: the ring wraps and
  is compacted in place thousands of times): the final per-slot state
  (resident ID, last_use) of every table bit-exact, the last 16 Plan records
  bit-exact, sampled final rows within 1e-5.
"""
import numpy as np
import pytest
import torch

from oracle import Policy, UncachedTrainer
from paper_2205_04702_b200 import HostTable, ScratchPipe
from tests.gpu_helpers import compare_tables, max_window_union, run_parity
from workload import CONFIGS, init_rows_np, init_table, sample_trace

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def tb_tables():
    c = CONFIGS["terabyte"]
    tabs = [HostTable(R, c.dim) for R in c.rows]
    yield tabs
    for h in tabs:
        h.free()


def _reinit(tabs, c):
    for t, h in enumerate(tabs):
        init_table(c.init_seed, t, c.rows[t], c.dim, device="cuda", out=h.tensor)
    torch.cuda.synchronize()


def _tight_slots(c, tr_np, margin):
    return [min(R, max_window_union(tr_np, t, 3, 2) + margin) for t, R in enumerate(c.rows)]


def test_terabyte_full_size_every_plan_and_pooled(tb_tables):
    c = CONFIGS["terabyte"]
    nb = 24
    tr = sample_trace(c.rows, c.batch, c.pooling, c.alpha, nb, c.trace_seed, device="cuda").cpu()
    assert max(c.rows) >= 1 << 25  # 26-bit keys: 4 radix passes
    slots = _tight_slots(c, tr.numpy(), 128)
    _reinit(tb_tables, c)
    g, d, e = c.surrogate()
    rep = run_parity(c.rows, slots, c.dim, c.batch, c.pooling, nb, 3, 2, trace=tr,
                     init_seed=c.init_seed, gde=(g, d, e), index_dtype="int32", index_on_device=True,
                     check_slots=True, sample_rows=3000, tables=tb_tables)
    assert rep["plans"] == nb and rep["pooled"] == nb
    assert rep["evictions"] > 10000, rep["evictions"]
    assert rep["stats"]["transfer_mode"] in ("hybrid", "gpu_pull")  # default above 32 MB of rows per batch
    assert rep["tables"]["max_rel"] <= TOL, rep["tables"]


def test_terabyte_graph_mode_2000_batches_log_wrap(tb_tables):
    c = CONFIGS["terabyte"]
    nb = 2000
    T, N, L, D = c.num_tables, c.batch, c.pooling, c.dim
    tr_dev = sample_trace(c.rows, N, L, c.alpha, nb, c.trace_seed + 1, device="cuda", dtype=torch.int32)
    tr_np = tr_dev.cpu().numpy().astype(np.int64)
    slots = [min(R, max_window_union(tr_np[:200], t, 3, 2) * 3 // 2 + 64) for t, R in enumerate(c.rows)]
    _reinit(tb_tables, c)
    g, d, e = c.surrogate()
    sp = ScratchPipe(c.rows, tb_tables, D, slots, N, L, window=3, index_dtype="int32",
                     index_on_device=True, log_factor=1)
    pooled = torch.empty((T, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    sp.run_steps(tr_dev, nb, pooled, grad, g, d, e)   # graph replay after the first 16 steps
    torch.cuda.synchronize()
    st = sp.stats()
    assert st["trained"] == nb and st["graph_steps"] > nb - 40, st["graph_steps"]
    # oracle: policy over every batch, uncached training over every batch
    pol = Policy(c.rows, slots, 3, 2)
    orc = UncachedTrainer(c.rows, D, N, L, c.init_seed)
    recs = None
    evictions = 0
    for b in range(nb):
        recs = pol.plan(tr_np, b)
        evictions += sum(r.evictions for r in recs)
        if b >= nb - 16:   # ring entries still live: the last 16 Plans bit-exact
            for t in range(T):
                gp = sp.debug_plan(b, t)
                r = recs[t]
                assert (gp["U"], gp["hits"], gp["misses"], gp["evictions"]) == \
                    (r.U, r.hits, r.misses, r.evictions), (b, t)
                assert np.array_equal(gp["slot"], r.slot) and np.array_equal(gp["evicted"], r.evicted), (b, t)
        orc.step(tr_np[b], g, d, e)
    assert evictions > 1_000_000, evictions
    for t in range(T):   # every slot of every table: resident ID and LRU stamp
        res, lu = sp.debug_slots(t)
        ores, olu = pol.slot_state(t)
        assert np.array_equal(res, ores), t
        assert np.array_equal(lu, olu), t
    sp.flush()
    worst = 0.0
    for t, R in enumerate(c.rows):
        touched = orc.touched(t)
        if len(touched) > 2000:
            touched = np.sort(np.random.default_rng(t).choice(touched, 2000, replace=False))
        want = orc.rows_of(t, touched)
        got = tb_tables[t].tensor[torch.from_numpy(touched)].numpy()
        cmp = compare_tables(got, want, init_rows_np(c.init_seed, t, touched, D))
        worst = max(worst, cmp["max_rel"])
    assert worst <= TOL, worst
    sp.close()


def test_terabyte_full_size_bf16_storage(tb_tables):
    """bf16 Storage (SP_FLAG_BF16, reading R28) at the full Terabyte shape
    against the oracle's bf16 mode: every Plan record and pooled output
    bit-exact, sampled final rows within one bf16 unit (2^-7 relative)."""
    c = CONFIGS["terabyte"]
    nb = 24
    tr = sample_trace(c.rows, c.batch, c.pooling, c.alpha, nb, c.trace_seed + 2, device="cuda").cpu()
    slots = _tight_slots(c, tr.numpy(), 128)
    _reinit(tb_tables, c)
    g, d, e = c.surrogate()
    rep = run_parity(c.rows, slots, c.dim, c.batch, c.pooling, nb, 3, 2, trace=tr,
                     init_seed=c.init_seed, gde=(g, d, e), index_dtype="int32", index_on_device=True,
                     check_slots=True, sample_rows=3000, tables=tb_tables, bf16=True)
    assert rep["plans"] == nb and rep["pooled"] == nb
    assert rep["evictions"] > 10000, rep["evictions"]
    assert rep["tables"]["max_rel"] <= 2.0 ** -7, rep["tables"]
