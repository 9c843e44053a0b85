"""Pins for oracle Part A (uncached EmbeddingBag training + sparse SGD).

Each test checks the oracle against something other than itself: the paper's
Fig. 2 worked example, closed forms, or an independent numpy brute force.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import UncachedTrainer
from workload import init_rows_np, sample_trace

SEED = 4702


def test_fig2_worked_example():
    """Fig. 2: batch of 2 bags gathering rows
    {0,4} and {0,2,5}; G[0], G[1] routed back; row 0 receives G[0]+G[1],
    row 4 receives G[0], rows 2 and 5 receive G[1]; other rows untouched."""
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2_bags.json")))
    D = 4
    o = UncachedTrainer([8], D, 2, 3, SEED, allow_padding=True)
    E = init_rows_np(SEED, 0, np.arange(8), D)
    ids = np.array([[b + [-1] * (3 - len(b)) for b in g["bags"]]], np.int64)
    G = np.array([[[2 ** -6, -2 ** -7, 2 ** -8, 3 * 2 ** -9],
                   [-2 ** -5, 2 ** -6, 5 * 2 ** -10, 2 ** -7]]], np.float32)
    eta = 0.5
    pooled = o.step(ids, eta=eta, grad=G, want_pooled=True)
    assert np.array_equal(pooled[0, 0], E[0] + E[4])
    assert np.array_equal(pooled[0, 1], (E[0] + E[2]) + E[5])

    def upd(e, g):  # exact real value, rounded once to fp32 (= fmaf)
        return (e.astype(np.float64) - eta * g.astype(np.float64)).astype(np.float32)

    G0, G1 = G[0, 0].astype(np.float64), G[0, 1].astype(np.float64)
    assert np.array_equal(o.row(0, 0), upd(E[0], G0 + G1))
    assert np.array_equal(o.row(0, 4), upd(E[4], G0))
    assert np.array_equal(o.row(0, 2), upd(E[2], G1))
    assert np.array_equal(o.row(0, 5), upd(E[5], G1))
    Gs = {"G0": G0, "G1": G1}
    for r, names in g["gradients_per_row"].items():
        assert np.array_equal(o.row(0, int(r)), upd(E[int(r)], sum(Gs[n] for n in names)))
    for r in g["untouched_rows_of_8"]:
        assert np.array_equal(o.row(0, r), E[r])


def test_single_lookup_closed_form():
    """L=1, one bag: E' = (1 - eta*gamma) E - eta*delta."""
    gamma, delta, eta = 0.5, 0.01, 0.01
    o = UncachedTrainer([100], 16, 1, 1, SEED)
    E = init_rows_np(SEED, 0, np.array([42]), 16)[0].astype(np.float64)
    o.step(np.array([[[42]]]), gamma, delta, eta)
    want = (1 - eta * gamma) * E - eta * delta
    got = o.row(0, 42).astype(np.float64)
    assert np.allclose(got, want, rtol=0, atol=4 * np.spacing(np.float32(0.1)))


def test_gamma_zero_conservation():
    """gamma=0: every touched row changes by exactly -eta*delta*multiplicity
    (SPEC S:202); multiplicities counted independently with bincount."""
    R, N, L, D = 50, 8, 4, 8
    delta, eta = 2.0 ** -6, 2.0 ** -3
    ids = sample_trace([R], N, L, 1.05, 1, 11)[0].numpy()
    o = UncachedTrainer([R], D, N, L, SEED)
    o.step(ids, 0.0, delta, eta)
    mult = np.bincount(ids.reshape(-1), minlength=R)
    E = init_rows_np(SEED, 0, np.arange(R), D).astype(np.float64)
    for r in range(R):
        want = (E[r] - eta * delta * mult[r]).astype(np.float32)
        assert np.array_equal(o.row(0, r), want), r


def test_eta_zero_is_identity():
    R, N, L, D = 30, 4, 3, 4
    ids = sample_trace([R, R], N, L, 1.0, 1, 3)[0].numpy()
    o = UncachedTrainer([R, R], D, N, L, SEED)
    o.step(ids, 0.5, 0.01, 0.0)
    for t in range(2):
        assert np.array_equal(o.rows_of(t, np.arange(R)), init_rows_np(SEED, t, np.arange(R), D))


def test_duplicate_in_bag_counts_twice():
    o = UncachedTrainer([10], 4, 1, 2, SEED)
    E = init_rows_np(SEED, 0, np.array([3]), 4)[0]
    pooled = o.step(np.array([[[3, 3]]]), 0.0, 0.0, 0.0, want_pooled=True)
    assert np.array_equal(pooled[0, 0], E + E)


def _numpy_bruteforce(tables, trace, gamma, delta, eta):
    """Independent numpy implementation: gather, fp32 p-fold, surrogate,
    per-occurrence fp64 scatter-add (np.add.at), one fp32 SGD step."""
    tables = [t.copy() for t in tables]
    for ids_b in trace:
        for t, ids in enumerate(ids_b):
            N, L = ids.shape
            W = tables[t]
            pooled = W[ids[:, 0]].copy()
            for p in range(1, L):
                pooled = pooled + W[ids[:, p]]
            g = oracle.fmaf32(np.float32(gamma), pooled, np.float32(delta))
            acc = np.zeros((W.shape[0], W.shape[1]), np.float64)
            np.add.at(acc, ids.reshape(-1), np.repeat(g.astype(np.float64), L, axis=0))
            touched = np.unique(ids)
            W[touched] = oracle.fmaf32(np.float32(-eta), acc[touched].astype(np.float32), W[touched])
    return tables


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_multi_batch_matches_numpy_bruteforce(seed):
    rows, D, N, L, nb = [40, 17], 8, 6, 3, 12
    gamma, delta, eta = 0.5, 0.01, 0.05
    trace = sample_trace(rows, N, L, 1.1, nb, seed).numpy()
    init = [init_rows_np(SEED, t, np.arange(R), D) for t, R in enumerate(rows)]
    want = _numpy_bruteforce(init, trace, gamma, delta, eta)
    o = UncachedTrainer(rows, D, N, L, SEED)
    for b in range(nb):
        o.step(trace[b], gamma, delta, eta)
    for t, R in enumerate(rows):
        got = o.rows_of(t, np.arange(R))
        # the fp64 accumulation order differs (add.at vs sorted fold): equal
        # after rounding to fp32 except at an fp32 rounding boundary
        assert np.max(np.abs(got - want[t])) <= 2 * np.spacing(np.float32(0.2))
        assert np.mean(got == want[t]) > 0.999


def test_index_range_error():
    o = UncachedTrainer([10, 20], 4, 2, 1, SEED)
    with pytest.raises(oracle.OracleError) as e:
        o.step(np.array([[[1], [2]], [[3], [20]]]), 0.5, 0.0, 0.1)
    assert e.value.code == oracle.ORC_ERR_INDEX and e.value.table == 1
    assert np.array_equal(o.row(0, 1), init_rows_np(SEED, 0, np.array([1]), 4)[0])
