"""Pins for the oracle's replacement-policy variants, padding and pinned
(static) slots (readings R23-R27).

PAPER.md P:1270-1278 swaps the default LRU for "a random eviction or LFU
(least-frequently-used) policy".  What the paper and the mathematics fix:
* every variant obeys the same window rules: no row of B(b-P..b+F) is ever
  evicted, checked by brute force over the trace;
* random eviction draws victims uniformly: over many seeds each occupied
  candidate is evicted with probability m/K (chi-square bound), and when
  every candidate is needed the victims are exactly the candidate set;
* LFU at P = F = 0 is the textbook frequency-ordered cache (ties by recency,
  then ID), cross-checked against an independent dict model with no slots;
* cold start takes vacant slots lowest first in every variant (R9);
* -1 padding (ragged bags) is "no lookup": a padded trace plans exactly like
  the trace with each pad replaced by a duplicate of a real ID of the same
  bag set (duplicates do not change U), and trains exactly like the trace
  with the padded positions removed;
* pinned rows (static partition) always hit and are never evicted.
"""
import numpy as np
import pytest

from oracle import LFU_FMAX, OracleError, Policy, UncachedTrainer
from workload import sample_trace

POLICIES = ["lru", "random", "lfu"]


def _tr(batches):
    """per-batch ID lists (one table, L=1) -> [nb][1][N][1]"""
    return np.array([[[[x] for x in b]] for b in batches], np.int64)


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("seed", range(4))
def test_window_superset_never_evicted(policy, seed):
    rows, slots, N, L, nb, P, F = [300, 120], [90, 60], 6, 3, 40, 3, 2
    tr = sample_trace(rows, N, L, 0.9, nb, 100 + seed).numpy()
    pol = Policy(rows, slots, P, F, policy=policy, policy_seed=seed)
    evs = 0
    for b in range(nb):
        recs = pol.plan(tr, b)
        for t in range(2):
            window = set(tr[max(0, b - P):min(nb, b + F + 1), t].reshape(-1).tolist())
            ev = set(recs[t].evicted_ids.tolist())
            evs += len(ev)
            assert not (ev & window), (policy, b, t)
            # always-hit invariant: after Plan(b) every ID of B(b) is resident
            assert set(tr[b, t].reshape(-1).tolist()) <= set(pol.resident(t).tolist())
    assert evs > 50


@pytest.mark.parametrize("policy", POLICIES)
def test_cold_start_vacant_slots_lowest_first(policy):
    pol = Policy([100], [10], 0, 0, policy=policy, policy_seed=7)
    r = pol.plan(_tr([[5, 3, 9, 1]]), 0)[0]
    assert list(r.uniq) == [1, 3, 5, 9] and list(r.slot) == [0, 1, 2, 3]


def test_random_victims_uniform_over_candidates():
    """Batch 0 fills all S slots; batch 1 brings m new IDs; P = F = 0 so every
    occupied slot is a candidate.  Over many seeds each slot is the k-th
    victim with probability 1/S and evicted with probability m/S."""
    S, m, seeds = 16, 4, 3000
    b0 = list(range(S))
    b1 = [100 + (i % m) for i in range(S)]
    tr = _tr([b0, b1])
    count = np.zeros(S)
    first = np.zeros(S)
    for sd in range(seeds):
        pol = Policy([1000], [S], 0, 0, policy="random", policy_seed=sd)
        pol.plan(tr, 0)
        r = pol.plan(tr, 1)[0]
        vs = r.victim_slots
        assert len(set(vs.tolist())) == m
        count[vs] += 1
        first[vs[0]] += 1     # victim of the smallest missed ID
    exp = seeds * m / S
    chi2 = np.sum((count - exp) ** 2 / exp)
    assert chi2 < 45, chi2     # 15 dof: p ~ 1e-4
    exp1 = seeds / S
    chi2f = np.sum((first - exp1) ** 2 / exp1)
    assert chi2f < 45, chi2f


def test_random_takes_every_candidate_when_all_needed():
    """When m equals the number of candidates, the victims are exactly the
    candidate set (brute force: slots whose resident is outside the window)."""
    S, P = 8, 1
    b0 = [0, 1, 2, 3, 4, 5, 6, 7]
    b1 = [0, 1, 2, 0, 1, 2, 0, 1]          # hits 0,1,2 (held through b=2 by P=1)
    b2 = [10, 11, 12, 13, 14, 10, 11, 12]  # 5 misses: candidates = slots of 3..7
    tr = _tr([b0, b1, b2])
    for sd in range(20):
        pol = Policy([100], [S], P, 0, policy="random", policy_seed=sd)
        pol.plan(tr, 0)
        pol.plan(tr, 1)
        r = pol.plan(tr, 2)[0]
        assert sorted(r.evicted_ids.tolist()) == [3, 4, 5, 6, 7]
    pol = Policy([100], [S - 1], P, 0, policy="random")
    with pytest.raises(OracleError):       # one slot short -> capacity at b = 2
        for b in range(3):
            pol.plan(_tr([b0[:7], b1[:7], b2[:7]]), b)


def _textbook_lfu(trace_np, S):
    """Independent batch-granular LFU cache (no slots): per batch, hits bump a
    saturating use count and recency; misses evict the residents not used in
    this batch with the smallest (count, last use, ID) until they fit."""
    res = {}   # id -> [count, last_use]
    out = []
    for b in range(trace_np.shape[0]):
        U = sorted(set(trace_np[b, 0].reshape(-1).tolist()))
        miss = [u for u in U if u not in res]
        for u in U:
            if u in res:
                res[u][0] = min(res[u][0] + 1, LFU_FMAX)
                res[u][1] = b
        ev = []
        free = S - len(res)
        need = max(0, len(miss) - free)
        if need:
            cand = sorted((c, lu, i) for i, (c, lu) in res.items() if lu != b)
            ev = sorted(i for _, _, i in cand[:need])
            for i in ev:
                del res[i]
        for u in miss:
            res[u] = [1, b]
        out.append((miss, ev, sorted(res)))
    return out


@pytest.mark.parametrize("seed", range(5))
def test_lfu_reduces_to_textbook_lfu_at_zero_window(seed):
    rows, S, N, L, nb = [200], 40, 8, 2, 60
    tr = sample_trace(rows, N, L, 1.1, nb, 300 + seed).numpy()
    pol = Policy(rows, [S], 0, 0, policy="lfu")
    want = _textbook_lfu(tr, S)
    for b in range(nb):
        r = pol.plan(tr, b)[0]
        miss, ev, res = want[b]
        assert r.miss_ids.tolist() == miss, b
        assert sorted(r.evicted_ids.tolist()) == ev, b
        assert pol.resident(0).tolist() == res, b


def test_lfu_keeps_the_frequent_row_lru_does_not():
    """Row 1 is used three times, then row 2 once (more recently); one slot
    must go: LFU evicts row 2 (fewer uses), LRU evicts row 1 (older)."""
    batches = [[1, 9], [1, 9], [1, 9], [2, 9], [3, 9]]   # P = F = 0, 3 slots
    tr = _tr(batches)
    got = {}
    for policy in ("lfu", "lru"):
        pol = Policy([100], [3], 0, 0, policy=policy)
        for b in range(4):
            pol.plan(tr, b)
        got[policy] = pol.plan(tr, 4)[0].evicted_ids.tolist()
    assert got == {"lfu": [2], "lru": [1]}


@pytest.mark.parametrize("policy", POLICIES)
def test_padding_plans_like_duplicates(policy):
    rows, slots, N, L, nb = [500, 80], [120, 60], 8, 4, 30
    tr = sample_trace(rows, N, L, 1.0, nb, 71).numpy()
    rng = np.random.default_rng(5)
    pad = tr.copy()
    dup = tr.copy()
    mask = rng.random(tr.shape) < 0.3
    mask[..., 0] = False                      # every bag keeps one real lookup
    pad[mask] = -1
    # a duplicate of the bag's first lookup: same unique set as the padded bag
    first = np.broadcast_to(tr[..., :1], tr.shape)
    dup[mask] = first[mask]
    pa = Policy(rows, slots, 3, 2, policy=policy, policy_seed=3, allow_padding=True)
    pb = Policy(rows, slots, 3, 2, policy=policy, policy_seed=3)
    for b in range(nb):
        ra, rb = pa.plan(pad, b), pb.plan(dup, b)
        for t in range(2):
            assert np.array_equal(ra[t].uniq, rb[t].uniq)
            assert np.array_equal(ra[t].slot, rb[t].slot)
            assert np.array_equal(ra[t].evicted, rb[t].evicted)
    with pytest.raises(OracleError):          # without the flag -1 is out of range
        Policy(rows, slots, 3, 2).plan(pad, 0)


def test_padding_trains_like_removed_positions():
    """Part A: a trailing -1 in every bag is "no lookup": pooled values and the
    trained tables equal those of the same bags without that position."""
    rows, D, N, nb = [300, 40], 8, 6, 12
    tr3 = sample_trace(rows, N, 3, 1.0, nb, 72).numpy()
    tr2 = tr3[..., :2].copy()
    pad = tr3.copy()
    pad[..., 2] = -1
    a = UncachedTrainer(rows, D, N, 3, 4702, allow_padding=True)
    b = UncachedTrainer(rows, D, N, 2, 4702)
    for k in range(nb):
        pa = a.step(pad[k], 0.5, 0.01, 0.05, want_pooled=True)
        pb = b.step(tr2[k], 0.5, 0.01, 0.05, want_pooled=True)
        assert np.array_equal(pa, pb)
    for t in range(2):
        ids = b.touched(t)
        assert np.array_equal(a.touched(t), ids)
        assert np.array_equal(a.rows_of(t, ids), b.rows_of(t, ids))


@pytest.mark.parametrize("policy", POLICIES)
def test_pinned_rows_always_hit_never_evicted(policy):
    rows, N, L, nb = [400], 12, 2, 50
    tr = sample_trace(rows, N, L, 1.2, nb, 81).numpy()
    ids, cnt = np.unique(tr[:, 0], return_counts=True)
    top = np.sort(ids[np.argsort(-cnt, kind="stable")[:10]])
    S = 10 + 2 * 3 * N * L
    pol = Policy(rows, [S], 3, 2, policy=policy, policy_seed=1, pinned=[top])
    res0, _ = pol.slot_state(0)
    assert res0[S - 10:].tolist() == top.tolist()
    for b in range(nb):
        r = pol.plan(tr, b)[0]
        assert not set(r.evicted_ids.tolist()) & set(top.tolist())
        assert not set(r.miss_ids.tolist()) & set(top.tolist())
        pinned_hits = set(r.uniq[r.hit].tolist()) & set(top.tolist())
        assert pinned_hits == set(r.uniq.tolist()) & set(top.tolist())
        res, _ = pol.slot_state(0)
        assert res[S - 10:].tolist() == top.tolist()
