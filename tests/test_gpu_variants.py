"""GPU parity of the SURVEY §8(f) variants against the oracle (DESIGN.md
readings R23-R27): replacement policies (random eviction, LFU),
ragged bags (-1 padding and CSR offsets with per-table pooling; Fig. 2
P:257-263), and the static top-N partition (pinned rows).

Bar as for LRU: every Plan record (U, hit/miss, victim slots, evicted IDs) and
the per-slot state bit-exact, pooled outputs bit-exact, final tables within
1e-5 (bit-exact expected).
"""
import numpy as np
import pytest
import torch

from oracle import OracleError, Policy
from paper_2205_04702_b200 import SP_ERR_CAPACITY, ScratchPipe, SpError
from paper_2205_04702_b200.harness import run_loop
from tests.gpu_helpers import max_window_union, pinned_tables, run_parity
from workload import sample_trace

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _assert_exact(rep):
    t = rep["tables"]
    assert t["max_rel"] <= TOL and t["mismatch"] == 0, t


@pytest.mark.parametrize("policy", ["random", "lfu"])
@pytest.mark.parametrize("P,F", [(3, 2), (2, 1), (1, 0)])
def test_policy_parity(policy, P, F):
    rows, D, N, L, nb = [600, 90, 2000], 16, 24, 3, 60
    tr = sample_trace(rows, N, L, 0.9, nb, 500 + 10 * P + F)
    slots = [min(R, max_window_union(tr.numpy(), t, P, F) + 6) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, P, F, trace=tr, gde=(0.5, 0.01, 0.02),
                     policy_kw={"policy": policy, "policy_seed": 1234 + P})
    assert rep["evictions"] > 300
    _assert_exact(rep)


@pytest.mark.parametrize("policy", ["random", "lfu"])
def test_policy_heavy_eviction_log_compaction(policy):
    # LFU: class logs of 2*S + 4n entries wrap and compact; RANDOM: long draws
    rows, D, N, L, nb = [3000, 400], 32, 64, 2, 120
    tr = sample_trace(rows, N, L, 0.7, nb, 77)
    slots = [max_window_union(tr.numpy(), t, 3, 2) + 2 for t in range(2)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02),
                     policy_kw={"policy": policy, "policy_seed": 9})
    assert rep["evictions"] > 3000
    _assert_exact(rep)


@pytest.mark.parametrize("policy", ["random", "lfu"])
def test_policy_graph_mode_matches_oracle(policy):
    """sp_run_steps (CUDA-graph replay) with a non-LRU policy."""
    from oracle import UncachedTrainer
    rows, D, N, L, nb = [5000, 300, 40], 16, 128, 2, 80
    tr = sample_trace(rows, N, L, 0.9, nb, 88)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 10) for t, R in enumerate(rows)]
    tables = pinned_tables(rows, D, 4702)
    sp = ScratchPipe(rows, tables, D, slots, N, L, index_dtype="int32", index_on_device=True,
                     policy=policy, policy_seed=5)
    dev = tr.to(torch.int32).cuda().contiguous()
    pooled = torch.empty((3, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    sp.run_steps(dev, nb, pooled, grad, 0.5, 0.01, 0.05)
    pol = Policy(rows, slots, 3, 2, policy=policy, policy_seed=5)
    for b in range(nb):
        pol.plan(tr.numpy(), b)
    for t in range(3):
        res, lu = sp.debug_slots(t)
        ores, olu = pol.slot_state(t)
        assert np.array_equal(res, ores) and np.array_equal(lu, olu), t
    sp.flush()
    orc = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        orc.step(tr.numpy()[b], 0.5, 0.01, 0.05)
    for t in range(3):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        assert np.array_equal(got, orc.rows_of(t, touched)), t
    sp.close()


@pytest.mark.parametrize("policy", ["random", "lfu"])
def test_policy_capacity_error_at_oracle_batch(policy):
    rows, D, N, L, nb = [400, 400], 8, 8, 2, 40
    tr = sample_trace(rows, N, L, 0.5, nb, 3)
    slots = [200, 30]
    pol = Policy(rows, slots, 3, 2, policy=policy, policy_seed=2)
    want = None
    try:
        for b in range(nb):
            pol.plan(tr.numpy(), b)
    except OracleError as e:
        want = (e.batch, e.table)
    assert want is not None
    sp = ScratchPipe(rows, pinned_tables(rows, D, 1), D, slots, N, L, policy=policy, policy_seed=2)
    with pytest.raises(SpError) as ei:
        run_loop(sp, tr, 0.5, 0.01, 0.01)
    assert ei.value.status == SP_ERR_CAPACITY
    assert (ei.value.batch, ei.value.table) == want
    sp.close()


def _padded(tr, frac, seed, empty_bags=True):
    """-1 at a random `frac` of the positions; with empty_bags some bags lose
    every lookup (they pool to zeros)."""
    rng = np.random.default_rng(seed)
    a = tr.numpy().copy()
    mask = rng.random(a.shape) < frac
    if empty_bags:
        mask[:, :, ::7, :] = True
    a[mask] = -1
    return torch.from_numpy(a)


@pytest.mark.parametrize("policy", ["lru", "random", "lfu"])
def test_padding_ragged_bags_parity(policy):
    rows, D, N, L, nb = [800, 120, 3], 16, 32, 4, 40
    tr = _padded(sample_trace(rows, N, L, 1.0, nb, 61), 0.35, 1)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 6) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02), padding=True,
                     policy_kw={"policy": policy, "policy_seed": 3})
    assert rep["evictions"] > 100
    _assert_exact(rep)


def test_padding_large_n_global_radix_path():
    # n = 4200*4 = 16800 > 8192: the global-memory radix path with pad keys
    rows, D, N, L, nb = [60000, 300], 8, 4200, 4, 8
    tr = _padded(sample_trace(rows, N, L, 0.9, nb, 9), 0.25, 2)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 10) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, padding=True, check_slots=False,
                     gde=(float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 1.0))
    assert rep["tables"]["max_rel"] <= TOL, rep["tables"]


def test_csr_per_table_pooling_parity():
    """sp_plan_csr: table 0 has bags of 0-3 lookups, table 1 exactly 5, table
    2 exactly 1 (per-table pooling, max L = 5); the oracle sees the same bags
    as -1-padded [T][N][5] (expanded here independently)."""
    rows, D, N, L, nb = [900, 400, 50], 16, 24, 5, 30
    rng = np.random.default_rng(11)
    full = sample_trace(rows, N, L, 1.0, nb, 62).numpy()
    lens = np.zeros((nb, 3, N), np.int64)
    lens[:, 0] = rng.integers(0, 4, size=(nb, N))
    lens[:, 1] = 5
    lens[:, 2] = 1
    padded = full.copy()
    batches = []
    for b in range(nb):
        vals, offs = [], [0]
        for t in range(3):
            for s in range(N):
                k = int(lens[b, t, s])
                vals.extend(full[b, t, s, :k].tolist())
                padded[b, t, s, k:] = -1
                offs.append(len(vals))
        batches.append((np.array(vals, np.int64), np.array(offs, np.int64)))
    tr = torch.from_numpy(padded)
    slots = [min(R, max_window_union(padded, t, 3, 2) + 6) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02), padding=True,
                     push=lambda sp, j: sp.plan_csr(*batches[j]))
    assert rep["plans"] == nb and rep["pooled"] == nb
    _assert_exact(rep)
    # malformed CSR is rejected before anything is enqueued
    sp = ScratchPipe(rows, pinned_tables(rows, D, 1), D, slots, N, L, padding=True)
    v, o = batches[0]
    with pytest.raises(SpError):
        sp.plan_csr(v, np.concatenate([[0, 6], o[2:]]))      # a bag of 6 > pooling 5
    sp.close()


@pytest.mark.parametrize("policy", ["lru", "random", "lfu"])
def test_static_topn_pinned_rows_parity(policy):
    """Static top-N partition (the paper's static-cache design point from the
    same kernels): the most frequent rows of a profiling prefix are pinned in
    the last slots; they always hit and are never evicted."""
    rows, D, N, L, nb = [1500, 200], 16, 32, 2, 50
    tr = sample_trace(rows, N, L, 1.1, nb, 66)
    pinned, slots = [], []
    for t, R in enumerate(rows):
        ids, cnt = np.unique(tr.numpy()[:10, t], return_counts=True)
        top = np.sort(ids[np.argsort(-cnt, kind="stable")[:40]])
        pinned.append(top)
        slots.append(min(R, max_window_union(tr.numpy(), t, 3, 2) + 40 + 4))
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02), pinned=pinned,
                     policy_kw={"policy": policy, "policy_seed": 8})
    assert rep["evictions"] > 100
    _assert_exact(rep)
