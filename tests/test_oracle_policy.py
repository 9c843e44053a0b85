"""Pins for oracle Part B (reference scratchpad policy, IDs only).

Pins: the paper's Fig. 6 narrative, the window text
 checked by brute force over the trace, closed forms (no eviction
when Storage covers every ID), a reduction to textbook batch-granular LRU when
P = F = 0 (independent OrderedDict model), and brute-force capacity bounds
(P:1030-1035).
"""
import json
import os
from collections import OrderedDict

import numpy as np
import pytest

import oracle
from oracle import OracleError, Policy
from workload import sample_trace


def _trace(batches, T=1):
    """list of per-batch ID lists (one table, N=len, L=1) -> [nb][1][N][1]."""
    return np.array([[[[x] for x in b]] for b in batches], np.int64)


GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_fig6_hit_map_and_fifth_cycle_eviction():
    # Fig. 6: batch 1 queries {7089, 2021}; batch 2 {3010, 7089}: 3010 misses,
    # 7089 hits although Storage is still vacant; E[2021] is evicted at the 5th
    # cycle once its past holds expire.  (Paper counts from 1; we from 0.)
    g = json.load(open(os.path.join(GOLDEN, "fig6_hitmap.json")))
    tr = _trace(g["batches"])
    pol = Policy([10000], [g["slots"]], past=g["past"], future=g["future"])
    ex = g["expect"]
    r0 = pol.plan(tr, 0)[0]
    assert list(r0.uniq) == ex["cycle1_uniq"] and r0.misses == ex["cycle1_misses"]
    assert r0.evictions == 0
    r1 = pol.plan(tr, 1)[0]
    assert {int(k): bool(h) for k, h in zip(r1.uniq, r1.hit)} == {int(k): v for k, v in ex["cycle2_hit"].items()}
    assert r1.evictions == 0
    first = None
    for b in range(2, len(g["batches"])):
        r = pol.plan(tr, b)[0]
        if r.evictions and first is None:
            first = b + 1                              # paper's 1-based cycle
            assert list(r.evicted_ids) == ex["first_evicted"]
    assert first == ex["first_eviction_cycle"]


def test_fig6_not_evictable_before_fifth_cycle():
    batches = [[7089, 2021], [3010, 7089], [3010, 7089], [3010, 9999], [3010, 9999]]
    pol = Policy([10000], [3], past=3, future=2)
    tr = _trace(batches)
    for b in range(3):
        pol.plan(tr, b)
    with pytest.raises(OracleError) as e:        # 4th cycle: 2021 still held
        pol.plan(tr, 3)
    assert e.value.code == oracle.ORC_ERR_CAPACITY and e.value.table == 0


def _random_run(rows, slots, N, L, nb, P, F, seed, alpha=1.05):
    tr = sample_trace(rows, N, L, alpha, nb, seed).numpy()
    pol = Policy(rows, slots, P, F)
    recs = [pol.plan(tr, b) for b in range(nb)]
    return tr, pol, recs


@pytest.mark.parametrize("seed", range(6))
def test_window_superset_never_evicted(seed):
    """No evicted ID appears in B(b-P..b+F), brute force."""
    rows, slots, N, L, nb, P, F = [300, 120], [90, 60], 6, 3, 40, 3, 2
    tr, pol, recs = _random_run(rows, slots, N, L, nb, P, F, seed, alpha=0.9)
    evs = 0
    for b in range(nb):
        for t in range(2):
            window = set(tr[max(0, b - P):min(nb, b + F + 1), t].reshape(-1).tolist())
            ev = set(recs[b][t].evicted_ids.tolist())
            evs += len(ev)
            assert not (ev & window), (b, t, ev & window)
    assert evs > 50  # the test exercises evictions


@pytest.mark.parametrize("seed", range(4))
def test_hits_are_previous_residents_and_bijection(seed):
    rows, slots, N, L, nb = [200], [64], 5, 2, 50
    tr = sample_trace(rows, N, L, 1.0, nb, seed).numpy()
    pol = Policy(rows, slots, 3, 2)
    resident = set()
    for b in range(nb):
        r = pol.plan(tr, b)[0]
        U = set(tr[b, 0].reshape(-1).tolist())
        assert set(r.uniq.tolist()) == U and list(r.uniq) == sorted(U)
        assert set(r.uniq[r.hit].tolist()) == U & resident
        ev = set(r.evicted_ids.tolist())
        assert ev <= resident and not (ev & U)
        resident = (resident - ev) | U
        assert set(pol.resident(0).tolist()) == resident
        res_slots, _ = pol.slot_state(0)
        occupied = res_slots[res_slots >= 0]
        assert len(set(occupied.tolist())) == len(occupied) == len(resident)
        assert set(occupied.tolist()) == resident


def test_no_eviction_when_storage_covers_all_rows():
    rows, N, L, nb = [64, 40], 8, 2, 30
    tr = sample_trace(rows, N, L, 1.0, nb, 5).numpy()
    pol = Policy(rows, rows, 3, 2)
    seen = [set(), set()]
    for b in range(nb):
        recs = pol.plan(tr, b)
        for t in range(2):
            U = set(tr[b, t].reshape(-1).tolist())
            assert recs[t].evictions == 0
            assert set(recs[t].miss_ids.tolist()) == U - seen[t]
            seen[t] |= U


class TextbookBatchLRU:
    """Independent model: batch-granular LRU, vacant slots first (lowest slot),
    then least recently used; ties inside one batch by smaller ID."""

    def __init__(self, S):
        self.free = list(range(S))
        self.order = OrderedDict()  # id -> slot, least recent first
        self.slot = {}

    def step(self, ids):
        U = sorted(set(ids))
        hits = [x for x in U if x in self.slot]
        misses = [x for x in U if x not in self.slot]
        # victims are chosen among entries not touched by this batch
        evictable = [x for x in self.order if x not in hits]
        victims, evicted = [], []
        for _ in misses:
            if self.free:
                victims.append(self.free.pop(0)); evicted.append(-1)
            else:
                x = evictable.pop(0)
                victims.append(self.slot[x]); evicted.append(x)
        for x in evicted:
            if x >= 0:
                del self.order[x]; del self.slot[x]
        for x, s in zip(misses, victims):
            self.slot[x] = s
        # recency: this batch's IDs become most recent, in ascending ID order
        for x in U:
            if x in self.order:
                del self.order[x]
            self.order[x] = self.slot[x]
        return hits, misses, victims, evicted


@pytest.mark.parametrize("seed", range(5))
def test_p0_f0_is_textbook_batch_lru(seed):
    rows, S, N, L, nb = [80], 24, 4, 2, 60
    tr = sample_trace(rows, N, L, 0.9, nb, seed).numpy()
    pol = Policy(rows, [S], 0, 0)
    ref = TextbookBatchLRU(S)
    for b in range(nb):
        r = pol.plan(tr, b)[0]
        hits, misses, victims, evicted = ref.step(tr[b, 0].reshape(-1).tolist())
        assert list(r.uniq[r.hit]) == hits
        assert list(r.miss_ids) == misses
        assert list(r.victim_slots) == victims
        assert list(r.evicted[~r.hit]) == evicted


def _union(tr, t, lo, hi):
    lo, hi = max(0, lo), min(tr.shape[0] - 1, hi)
    return len(set(tr[lo:hi + 1, t].reshape(-1).tolist()))


@pytest.mark.parametrize("seed", range(4))
def test_capacity_bounds_bruteforce(seed):
    """CAPACITY never occurs when S >= max_b |U(b-P..b+F)| and always occurs
    when S < max_b |U(b-P..b)| (every ID of the last P+1 batches is resident
    at the end of Plan(b)); the failure point is monotone in S."""
    rows, N, L, nb, P, F = [120], 6, 2, 30, 3, 2
    tr = sample_trace(rows, N, L, 0.8, nb, seed).numpy()
    hi = max(_union(tr, 0, b - P, b + F) for b in range(nb))
    lo = max(_union(tr, 0, b - P, b) for b in range(nb))
    fail_at = {}
    for S in range(max(1, lo - 3), hi + 2):
        pol = Policy(rows, [S], P, F)
        try:
            for b in range(nb):
                pol.plan(tr, b)
            fail_at[S] = None
        except OracleError as e:
            assert e.code == oracle.ORC_ERR_CAPACITY
            fail_at[S] = e.batch
    for S, fb in fail_at.items():
        if S >= hi:
            assert fb is None
        if S < lo:
            assert fb is not None
    # more Storage never fails earlier
    prev = -1
    for S in sorted(fail_at):
        fb = fail_at[S]
        fbv = 10 ** 9 if fb is None else fb
        assert fbv >= prev
        prev = fbv


def test_tiny_config_never_hits_capacity():
    from workload import CONFIGS
    c = CONFIGS["tiny"]
    for seed in range(20):
        tr = sample_trace(c.rows, c.batch, c.pooling, c.alpha, c.num_batches, seed).numpy()
        pol = Policy(c.rows, c.slots, 3, 2)
        for b in range(c.num_batches):
            pol.plan(tr, b)


def test_worst_case_storage_formula():
    """(8 x 20 x 2048 x 128 x 4 B) x 6 = 960 MB (MiB)."""
    from paper_2205_04702_b200.sizing import worst_case_storage_bytes
    assert worst_case_storage_bytes(tables=8, pooling=20, batch=2048, dim=128, window=3) == 1006632960
    assert 1006632960 == 960 * 2 ** 20


@pytest.mark.parametrize("seed", range(4))
def test_partial_selection_equals_full_sort(seed):
    """The oracle's default picks the |misses| smallest candidates with a
    bounded heap; sorting every candidate must give identical plans."""
    rows, slots, N, L, nb = [2000, 500], [900, 300], 8, 2, 60
    tr = sample_trace(rows, N, L, 0.9, nb, 50 + seed).numpy()
    a, b = Policy(rows, slots, 3, 2), Policy(rows, slots, 3, 2, full_sort=True)
    for bb in range(nb):
        ra, rb = a.plan(tr, bb), b.plan(tr, bb)
        for x, y in zip(ra, rb):
            assert np.array_equal(x.slot, y.slot) and np.array_equal(x.evicted, y.evicted)
