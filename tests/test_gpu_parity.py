"""GPU parity: the CUDA path through the C ABI vs the CPU oracle.

Bar (BASELINE.json north_star): unique / hit / miss / victim / evicted /
resident sets and slot stamps bit-exact; pooled outputs bit-exact (same fp32
left fold); final host tables within max relative error 1e-5 (bit-exact
expected: the coalesced gradient is an fp64 sum on both sides, rounded once).
"""
import numpy as np
import pytest
import torch

from oracle import Policy
from paper_2205_04702_b200 import SP_ERR_CAPACITY, SP_ERR_INDEX_RANGE, ScratchPipe, SpError
from paper_2205_04702_b200.harness import run_loop
from workload import CONFIGS, sample_trace
from tests.gpu_helpers import max_window_union, pinned_tables, run_parity

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _assert_tables(rep, exact=True):
    t = rep["tables"]
    assert t["max_rel"] <= TOL, t
    if exact:
        assert t["mismatch"] == 0, t


def test_tiny_config_parity():
    c = CONFIGS["tiny"]
    rep = run_parity(c.rows, c.slots, c.dim, c.batch, c.pooling, c.num_batches, 3, 2,
                     alpha=c.alpha, trace_seed=c.trace_seed, init_seed=c.init_seed,
                     gde=(c.gamma, c.delta, c.eta))
    assert rep["plans"] == c.num_batches and rep["pooled"] == c.num_batches
    assert rep["evictions"] > 0
    _assert_tables(rep)


@pytest.mark.parametrize("P,F", [(3, 2), (2, 1), (1, 1), (0, 0), (4, 3), (3, 0), (1, 2)])
def test_window_variants_policy_and_values(P, F):
    rows, D, N, L, nb = [300, 64, 1000], 8, 16, 3, 40
    tr = sample_trace(rows, N, L, 0.9, nb, 31 + P * 7 + F)
    slots = [max_window_union(tr.numpy(), t, P, F) + 2 for t in range(3)]
    slots = [min(s, R) for s, R in zip(slots, rows)]
    rep = run_parity(rows, slots, D, N, L, nb, P, F, trace=tr, gde=(0.5, 0.01, 0.02))
    assert rep["evictions"] > 0
    _assert_tables(rep)


def test_log_compaction_and_heavy_eviction():
    # log_factor=1: the LRU log ring is S_t + 4n entries and must compact often
    rows, D, N, L, nb = [500, 200], 16, 24, 2, 80
    tr = sample_trace(rows, N, L, 0.7, nb, 77)
    slots = [max_window_union(tr.numpy(), t, 3, 2) + 1 for t in range(2)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, log_factor=1)
    assert rep["evictions"] > 500
    _assert_tables(rep)


@pytest.mark.parametrize("D", [4, 12, 32, 64, 128, 256])
def test_dims(D):
    rows, N, L, nb = [400, 90], 8, 5, 16
    tr = sample_trace(rows, N, L, 1.0, nb, D)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 3) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.05))
    _assert_tables(rep)


def test_hot_segments_multichunk_backward():
    # 3-row table: every row occurs hundreds of times per batch -> multi-chunk
    rows, D, N, L, nb = [3, 7, 5000], 16, 256, 4, 10
    tr = sample_trace(rows, N, L, 1.05, nb, 5)
    slots = [3, 7, min(5000, max_window_union(tr.numpy(), 2, 3, 2) + 5)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr,
                     gde=(float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 0.5))
    _assert_tables(rep, exact=False)


def test_large_batch_radix_sort_path():
    # N*L = 16800 > 16384: the global-memory radix-sort dedup path
    rows, D, N, L, nb = [60000, 300], 8, 4200, 4, 9
    tr = sample_trace(rows, N, L, 0.9, nb, 9)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 10) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, check_slots=False,
                     gde=(float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 1.0))
    _assert_tables(rep, exact=False)


@pytest.mark.parametrize("index_dtype,on_device", [("int32", False), ("int64", True), ("int32", True)])
def test_index_formats(index_dtype, on_device):
    c = CONFIGS["tiny"]
    rep = run_parity(c.rows, c.slots, c.dim, c.batch, c.pooling, c.num_batches, 3, 2,
                     alpha=c.alpha, index_dtype=index_dtype, index_on_device=on_device)
    _assert_tables(rep)


def test_register_host_flag():
    c = CONFIGS["tiny"]
    rep = run_parity(c.rows, c.slots, c.dim, c.batch, c.pooling, 8, 3, 2, alpha=c.alpha,
                     register_host=True, profile=True)
    st = rep["stats"]
    assert st["kernel_timed"]["forward"] == 8 and st["kernel_ms"]["backward"] > 0
    _assert_tables(rep)


def test_host_alloc_tables():
    """Host tables from sp_host_alloc (THP-backed, registered by the library)."""
    c = CONFIGS["tiny"]
    rep = run_parity(c.rows, c.slots, c.dim, c.batch, c.pooling, c.num_batches, 3, 2,
                     alpha=c.alpha, host_alloc=True)
    _assert_tables(rep)


def test_host_alloc_near_numa_tables():
    """sp_host_alloc_near: the tables on the host NUMA node closest to the GPU
    (the node id is reported; -1 when the host has no NUMA information)."""
    from paper_2205_04702_b200 import HostTable
    h = HostTable(1000, 16, device=0)
    assert h.numa_node == -1 or 0 <= h.numa_node < 64
    h.tensor[7].fill_(3.0)
    assert float(h.tensor[7].sum()) == 48.0
    h.free()
    c = CONFIGS["tiny"]
    rep = run_parity(c.rows, c.slots, c.dim, c.batch, c.pooling, c.num_batches, 3, 2,
                     alpha=c.alpha, host_alloc="near")
    _assert_tables(rep)


def test_capacity_error_at_oracle_batch_and_table():
    rows, D, N, L, nb = [400, 400], 8, 8, 2, 40
    tr = sample_trace(rows, N, L, 0.5, nb, 3)
    slots = [200, 30]   # table 1 too small for its window working set
    pol = Policy(rows, slots, 3, 2)
    from oracle import OracleError
    want = None
    try:
        for b in range(nb):
            pol.plan(tr.numpy(), b)
    except OracleError as e:
        want = (e.batch, e.table)
    assert want is not None
    tables = pinned_tables(rows, D, 1)
    sp = ScratchPipe(rows, tables, D, slots, N, L)
    with pytest.raises(SpError) as ei:
        run_loop(sp, tr, 0.5, 0.01, 0.01)
    assert ei.value.status == SP_ERR_CAPACITY
    assert (ei.value.batch, ei.value.table) == want
    sp.close()


def test_index_range_error():
    rows, D, N, L, nb = [100, 50], 8, 4, 2, 12
    tr = sample_trace(rows, N, L, 1.0, nb, 4)
    tr[6, 1, 2, 1] = 50  # out of range for table 1
    tables = pinned_tables(rows, D, 1)
    sp = ScratchPipe(rows, tables, D, [60, 40], N, L)
    with pytest.raises(SpError) as ei:
        run_loop(sp, tr, 0.5, 0.01, 0.01)
    assert ei.value.status == SP_ERR_INDEX_RANGE
    assert (ei.value.batch, ei.value.table) == (6, 1)
    sp.close()


def test_call_order_errors():
    rows, D, N, L = [50], 4, 2, 1
    tables = pinned_tables(rows, D, 1)
    sp = ScratchPipe(rows, tables, D, [20], N, L)
    pooled = torch.empty((1, N, D), device="cuda")
    with pytest.raises(SpError):
        sp.forward(pooled)                  # nothing planned
    sp.plan(torch.zeros((1, N, L), dtype=torch.int64))
    with pytest.raises(SpError):
        sp.train(pooled, 0.1)               # train before forward
    sp.end_of_data()
    sp.forward(pooled)
    with pytest.raises(SpError):
        sp.forward(pooled)                  # forward twice
    sp.train(pooled, 0.0)
    sp.flush()
    sp.close()


def test_kaggle_full_size_parity_sampled():
    """BASELINE configs[1] at full size (26 Criteo-Kaggle tables, D=64,
    N=2048), int32 device indices as bench.py runs them, 1% slots so that
    evictions start within the checked batches; every plan record bit-exact,
    every pooled output bit-exact, sampled final rows within 1e-5."""
    c = CONFIGS["kaggle"]
    nb = 16
    tr = sample_trace(c.rows, c.batch, c.pooling, c.alpha, nb, c.trace_seed)
    # tightest safe Storage per table: evictions start within the checked batches
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 64) for t, R in enumerate(c.rows)]
    g, d, e = c.surrogate()
    rep = run_parity(c.rows, slots, c.dim, c.batch, c.pooling, nb, 3, 2, trace=tr,
                     init_seed=c.init_seed, gde=(g, d, e),
                     index_dtype="int32", index_on_device=True, check_slots=False,
                     sample_rows=4000)
    assert rep["plans"] == nb and rep["evictions"] > 1000
    _assert_tables(rep, exact=False)


def test_run_steps_graph_replay_matches_oracle():
    """sp_run_steps (C driver loop; CUDA-graph replay of the steady-state step
    after the first RING batches) gives the same plans, pooled values and
    final tables as the oracle."""
    from oracle import UncachedTrainer
    rows, D, N, L, nb = [2000, 300, 50], 16, 64, 2, 60
    tr = sample_trace(rows, N, L, 0.9, nb, 12)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 8) for t, R in enumerate(rows)]
    tables = pinned_tables(rows, D, 4702)
    sp = ScratchPipe(rows, tables, D, slots, N, L, index_dtype="int32", index_on_device=True)
    dev = tr.to(torch.int32).cuda().contiguous()
    pooled = torch.empty((3, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    g, d, e = 0.5, 0.01, 0.05
    sp.run_steps(dev, 25, pooled, grad, g, d, e)        # mixes eager and graph steps
    sp.run_steps(dev, nb - 25, pooled, grad, g, d, e)   # ... and the trace tail
    sp.flush()
    st = sp.stats()
    assert st["trained"] == nb
    orc = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        orc.step(tr.numpy()[b], g, d, e)
    for t, R in enumerate(rows):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        want = orc.rows_of(t, touched)
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-4)) <= TOL
    sp.close()


@pytest.mark.gpu
def test_run_steps_pinned_host_trace_matches_oracle():
    """sp_run_steps over a PINNED HOST trace (the plan kernel reads each batch
    over the host link; bench.py's e2e path), switched mid-run from a device
    trace and driven one step per call, gives the oracle's final tables."""
    from oracle import UncachedTrainer
    rows, D, N, L, nb = [2000, 300, 50], 16, 64, 2, 70
    tr = sample_trace(rows, N, L, 0.9, nb, 13)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 8) for t, R in enumerate(rows)]
    tables = pinned_tables(rows, D, 4702)
    sp = ScratchPipe(rows, tables, D, slots, N, L, index_dtype="int32", index_on_device=True)
    t32 = tr.to(torch.int32).contiguous()
    dev = t32.cuda()
    pooled = torch.empty((3, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    g, d, e = 0.5, 0.01, 0.05
    sp.run_steps(dev[:30], 20, pooled, grad, g, d, e)              # device trace, pushes up to 26
    j0 = sp.stats()["pushed"]
    host = t32[j0:].pin_memory()                                    # the rest from pinned host memory
    while sp.stats()["trained"] < nb:
        sp.run_steps(host, 1, pooled, grad, g, d, e, first_batch=j0)
    sp.flush()
    orc = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        orc.step(tr.numpy()[b], g, d, e)
    for t, R in enumerate(rows):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        want = orc.rows_of(t, touched)
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-4)) <= TOL
    with pytest.raises(Exception):  # pageable host memory is refused
        sp2 = ScratchPipe(rows, pinned_tables(rows, D, 4702), D, slots, N, L, index_dtype="int32",
                          index_on_device=True)
        try:
            sp2.run_steps(t32.clone(), 1, pooled, grad, g, d, e)
        finally:
            sp2.close()
    sp.close()


@pytest.mark.gpu
@pytest.mark.parametrize("D", [64, 128, 256, 512, 1024])
def test_hot_row_segments_last_arriver_fold(D):
    """Rows with more occurrences than one k_bwd segment (hs = 128 / 64 / 32 /
    16 / 16 for D = 64 / 128 / 256 / 512 / 1024; at hs = 16 a row with 17-32
    occurrences already has 2 segments, the worst case of the hot-record
    sizing): several CTAs fold segments, write fp64 partials,
    and the last to arrive folds them in segment order (plus plain chunk
    records from the large table in the same launch)."""
    rows, N, L, nb = [3, 5, 4000], 512, 4, 8
    tr = sample_trace(rows, N, L, 1.05, nb, 21 + D)
    slots = [3, 5, min(4000, max_window_union(tr.numpy(), 2, 3, 2) + 5)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr,
                     gde=(float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 0.5))
    _assert_tables(rep, exact=False)


@pytest.mark.gpu
@pytest.mark.parametrize("N,L", [(750, 4), (1500, 4)])
def test_smem_radix_tile_sizes(N, L):
    """n = N*L = 3000 and 6000: the 4- and 8-element-per-thread shared-memory
    radix passes of the dedup CTA (n = 2048 uses 2 per thread)."""
    rows, D, nb = [50000, 700], 16, 8
    tr = sample_trace(rows, N, L, 1.0, nb, N)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 10) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr,
                     gde=(float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 1.0))
    _assert_tables(rep, exact=False)


@pytest.mark.gpu
def test_stage_timing_and_plan_profile_introspection():
    """sp_set_stage_timing / sp_stage_times (events inside the recaptured step
    graphs) and sp_debug_plan_profile (per-CTA %globaltimer) report positive,
    self-consistent durations, and turning stage timing on and off does not
    change the results of the run."""
    from oracle import UncachedTrainer
    rows, D, N, L, nb = [3000, 400], 32, 128, 2, 80
    tr = sample_trace(rows, N, L, 1.0, nb, 31)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 8) for t, R in enumerate(rows)]
    tables = pinned_tables(rows, D, 4702)
    sp = ScratchPipe(rows, tables, D, slots, N, L, index_dtype="int32", index_on_device=True)
    dev = tr.to(torch.int32).cuda().contiguous()
    pooled = torch.empty((2, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    g, d, e = 0.5, 0.01, 0.05
    sp.run_steps(dev, 20, pooled, grad, g, d, e)
    sp.set_stage_timing(True)
    sp.run_steps(dev, 30, pooled, grad, g, d, e)          # recaptured with event nodes
    st = sp.stage_times()
    sp.set_stage_timing(False)
    for k in ("plan", "transfer", "forward", "surrogate", "backward"):
        assert st[k]["n"] > 0 and st[k]["ms"] > 0, (k, st[k])
    sp.set_profiling(True)
    sp.run_steps(dev, 10, pooled, grad, g, d, e)          # eager profiled steps
    prof = sp.debug_plan_profile()
    sp.set_profiling(False)
    pl = prof["per_launch"]
    assert len(pl["span_us"]) >= 5
    assert all(s > 0 for s in pl["span_us"])
    assert all(sp_ >= c - 1e-3 for sp_, c in zip(pl["span_us"], pl["plan_cta_max_us"]))
    sp.run_steps(dev, nb - 60, pooled, grad, g, d, e)
    sp.flush()
    orc = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        orc.step(tr.numpy()[b], g, d, e)
    for t, R in enumerate(rows):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        want = orc.rows_of(t, touched)
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-4)) <= TOL
    sp.close()


@pytest.mark.gpu
def test_prefill_all_resident_no_misses_matches_oracle():
    """sp_prefill (slots == rows, every row loaded before the first batch):
    no batch misses or evicts, and training still equals the oracle; prefill
    is refused when a table is not fully resident."""
    from oracle import UncachedTrainer
    rows, D, N, L, nb = [900, 60, 333], 16, 32, 3, 25
    tr = sample_trace(rows, N, L, 1.0, nb, 41)
    tables = pinned_tables(rows, D, 4702)
    sp = ScratchPipe(rows, tables, D, list(rows), N, L, index_dtype="int32", index_on_device=True)
    sp.prefill()
    dev = tr.to(torch.int32).cuda().contiguous()
    pooled = torch.empty((3, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    g, d, e = 0.5, 0.01, 0.05
    sp.run_steps(dev, nb, pooled, grad, g, d, e)
    sp.flush()
    st = sp.stats()
    assert st["misses"] == 0 and st["evictions"] == 0 and st["hits"] == st["uniques"] > 0
    orc = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        orc.step(tr.numpy()[b], g, d, e)
    for t, R in enumerate(rows):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        want = orc.rows_of(t, touched)
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-4)) <= TOL
    sp.close()
    sp2 = ScratchPipe(rows, pinned_tables(rows, D, 4702), D, [900, 60, 300], N, L)
    with pytest.raises(SpError):
        sp2.prefill()
    sp2.close()


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"SP_CPU_GATHER": "0"}, {"SP_CPU_GATHER": "1"},
                                 {"SP_CPU_GATHER": "1", "SP_GATHER_DMA": "1"},
                                 {"SP_CPU_GATHER": "0", "SP_WRITEBACK": "gpu"},
                                 {"SP_CPU_GATHER": "1", "SP_WRITEBACK": "gpu"},
                                 {"SP_CPU_GATHER": "0", "SP_WRITEBACK": "cpu"},
                                 {"SP_GATHER_FRAC": "0.5"}, {"SP_GATHER_FRAC": "0.3", "SP_WRITEBACK": "gpu"}])
def test_transfer_modes_match_oracle(env, monkeypatch):
    """Every transfer mode (GPU pull of random host rows, CPU gather into a
    pinned slot, CPU gather + copy-engine DMA) gives the oracle's plans,
    pooled values and final tables under heavy eviction; the default picks by
    batch size, so large configurations use the GPU pull."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rows, D, N, L, nb = [5000, 700, 90], 32, 96, 3, 40
    tr = sample_trace(rows, N, L, 0.9, nb, 51)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 4) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.05))
    assert rep["evictions"] > 200
    assert rep["stats"]["gpu_writeback"] == (env.get("SP_WRITEBACK") == "gpu")
    _assert_tables(rep)


@pytest.mark.gpu
def test_serial_strawman_schedule_matches_oracle(monkeypatch):
    """The paper's straw-man design point (Fig. 10: stages back to back, no
    overlap; bench --variant serial): every stage on the caller's stream
    (SP_DIAG_SERIAL=1) gives the same plans, pooled values and tables."""
    monkeypatch.setenv("SP_DIAG_SERIAL", "1")
    rows, D, N, L, nb = [3000, 250, 40], 16, 48, 2, 40
    tr = sample_trace(rows, N, L, 0.9, nb, 57)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 5) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.05))
    assert rep["evictions"] > 200
    _assert_tables(rep)
