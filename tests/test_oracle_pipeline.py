"""Pins for oracle Part C: the paper's 5-stage pipeline with values.

* cached == uncached training, bit for bit, with the paper's window (P=3, F=2)
  under several within-cycle stage orders
* Train always hits
* shrunken windows produce the RAW hazards of P:735-765 (negative tests)
"""
import numpy as np
import pytest

from oracle import OracleError, UncachedTrainer
from oracle.pipeline import PipelineSim
from workload import CONFIGS, init_rows_np, sample_trace

ORDERS = ["TICEP", "PCEIT", "CTPIE", "ITCPE"]


def _run_both(rows, slots, D, N, L, nb, P, F, seed, order, alpha=1.05, gde=(0.5, 0.01, 0.01)):
    g, d, e = gde
    tr = sample_trace(rows, N, L, alpha, nb, seed).numpy()
    init = [init_rows_np(4702, t, np.arange(R), D) for t, R in enumerate(rows)]
    sim = PipelineSim(rows, slots, D, N, L, P, F, 4702, g, d, e, order=order, init_tables=init)
    cpu = sim.run(tr)
    ref = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        ref.step(tr[b], g, d, e)
    want = [ref.rows_of(t, np.arange(R)) for t, R in enumerate(rows)]
    return sim, cpu, want


@pytest.mark.parametrize("order", ORDERS)
def test_tiny_config_cached_equals_uncached(order):
    c = CONFIGS["tiny"]
    sim, cpu, want = _run_both(c.rows, c.slots, c.dim, c.batch, c.pooling, c.num_batches,
                               3, 2, c.trace_seed, order, c.alpha)
    assert sim.hazards == []
    for t in range(2):
        assert np.array_equal(cpu[t], want[t])


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("order", ["TICEP", "PCEIT"])
def test_tight_storage_cached_equals_uncached(seed, order):
    # Storage just large enough: lots of evictions and refetches
    rows, D, N, L, nb = [64, 48], 4, 4, 2, 60
    sim, cpu, want = _run_both(rows, [40, 40], D, N, L, nb, 3, 2, seed, order, alpha=0.9)
    assert sim.hazards == []
    for t in range(2):
        assert np.array_equal(cpu[t], want[t])


def _adversarial_hazards(P, F, order, seeds=range(4)):
    found = []
    for seed in seeds:
        rows, D, N, L, nb = [64], 2, 4, 2, 120
        tr = sample_trace(rows, N, L, 0.6, nb, 100 + seed).numpy()
        for S in (20, 24, 28, 32):
            sim = PipelineSim(rows, [S], D, N, L, P, F, 4702, 0.5, 0.01, 0.05, order=order,
                              init_tables=[init_rows_np(4702, 0, np.arange(64), D)])
            try:
                sim.run(tr)
            except OracleError:
                pass  # CAPACITY ends the run; hazards seen before it still count
            found += sim.hazards
    return found


@pytest.mark.parametrize("order", ORDERS)
def test_paper_window_is_hazard_free_on_adversarial_traces(order):
    assert _adversarial_hazards(3, 2, order) == []


@pytest.mark.parametrize("order", ORDERS)
def test_no_window_is_unsafe_under_every_order(order):
    hz = _adversarial_hazards(1, 0, order)
    assert hz, "P=1, F=0 must expose RAW hazards"


def test_short_past_window_breaks_plan_collect_first_order():
    hz = _adversarial_hazards(2, 2, "PCEIT")
    assert any(h[0] == "evict-pending" for h in hz)
    assert _adversarial_hazards(2, 2, "TICEP") == []


def test_short_future_window_gives_stale_cpu_read():
    hz = _adversarial_hazards(3, 1, "PCEIT")
    assert any(h[0] == "stale-cpu-read" for h in hz)
