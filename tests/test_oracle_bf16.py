"""Pins for the oracle's bf16 Storage mode (reading R28).

The scratchpad holds each resident row rounded to bf16 (round to nearest,
ties to even) on fill and after every SGD update; the forward folds the
widened values in fp32, the coalescing stays fp64, host tables stay fp32.
Pinned against things other than the oracle itself:

* the rounding against torch's own fp32 -> bfloat16 conversion (an
  independent implementation) on random values over the whole exponent
  range, constructed ties, subnormals, infinities and NaN;
* first touch: with eta = 0 a touched row equals the rounding of its fp32
  initial value, an untouched row keeps its fp32 value, and the pooled
  output is the fp32 left fold of the rounded rows;
* the L = 1 closed form iterated with torch's rounding:
  w <- bf16(fmaf(-eta, (1/N)(gamma*w + delta)... ) for a row alone in its bags;
* cached (Part C, 5-stage pipeline) == uncached bit for bit in bf16 mode,
  under several within-cycle stage orders, with evictions and refetches.
"""
import numpy as np
import pytest
import torch

from oracle import UncachedTrainer, bf16_round, fmaf32, init_value
from oracle.pipeline import PipelineSim
from workload import CONFIGS, init_rows_np, sample_trace


def _torch_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


def test_rounding_matches_torch_bfloat16():
    rng = np.random.default_rng(28)
    bits = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    # constructed exact ties (low 16 bits = 0x8000) with even and odd kept mantissas
    ties = ((rng.integers(0, 2**16, size=4096, dtype=np.uint32) << 16) | 0x8000).view(np.float32)
    edge = np.array([0.0, -0.0, 1e-45, -1e-45, 1.17549435e-38, 3.4028235e38, -3.4028235e38,
                     np.inf, -np.inf, 1.0, 1.00390625, 1.01171875], np.float32)
    for v in (x, ties, edge):
        got, want = bf16_round(v), _torch_bf16(v)
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(got), nan)
        assert np.array_equal(got[~nan].view(np.uint32), want[~nan].view(np.uint32))


def test_first_touch_rounds_rows_and_forward_folds_rounded_values():
    rows, D, N, L = [500, 40], 16, 8, 3
    tr = sample_trace(rows, N, L, 1.05, 1, 7).numpy()
    o = UncachedTrainer(rows, D, N, L, 4702, bf16=True)
    pooled = o.step(tr[0], 0.5, 0.01, 0.0, want_pooled=True)   # eta = 0: no update
    for t, R in enumerate(rows):
        touched = set(np.unique(tr[0][t]).tolist())
        for r in range(R):
            init = np.array([init_value(4702, t, r, j) for j in range(D)], np.float32)
            want = _torch_bf16(init) if r in touched else init
            assert np.array_equal(o.row(t, r), want), (t, r)
        for s in range(N):
            acc = None
            for p in range(L):
                v = _torch_bf16(init_rows_np(4702, t, np.array([tr[0][t][s][p]]), D)[0])
                acc = v if acc is None else (acc + v).astype(np.float32)
            assert np.array_equal(pooled[t][s], acc), (t, s)


def test_single_lookup_closed_form_with_rounded_updates():
    # one table, L = 1, every bag looks up row 3: after dedup the row's coalesced
    # gradient is sum_s (gamma*w + delta) = N*(gamma*w + delta) in fp32/fp64, so
    # w_{k+1} = bf16(fmaf(-eta, float(N*fp64(fmaf(gamma, w, delta))), w_k))
    rows, D, N = [10], 8, 4
    g, d, e = 0.5, 0.01, 0.05
    o = UncachedTrainer(rows, D, N, 1, 4702, bf16=True)
    ids = np.full((1, N, 1), 3, np.int64)
    w = _torch_bf16(np.array([init_value(4702, 0, 3, j) for j in range(D)], np.float32))
    for _ in range(25):
        o.step(ids, g, d, e)
        gs = fmaf32(np.float32(g), w, np.float32(d))
        acc = (gs.astype(np.float64) * N).astype(np.float32)   # N equal fp32 terms summed exactly in fp64
        w = _torch_bf16(fmaf32(np.float32(-e), acc, w))
        assert np.array_equal(o.row(0, 3), w)


@pytest.mark.parametrize("order", ["TICEP", "PCEIT", "CTPIE"])
def test_cached_equals_uncached_bf16(order):
    rows, D, N, L, nb = [64, 48], 4, 4, 2, 60
    S = [40, 40]   # just above the window working set: evictions and refetches
    tr = sample_trace(rows, N, L, 0.9, nb, 11).numpy()
    init = [init_rows_np(4702, t, np.arange(R), D) for t, R in enumerate(rows)]
    sim = PipelineSim(rows, S, D, N, L, 3, 2, 4702, 0.5, 0.01, 0.05, order=order, init_tables=init, bf16=True)
    cpu = sim.run(tr)
    assert sim.hazards == []
    ref = UncachedTrainer(rows, D, N, L, 4702, bf16=True)
    for b in range(nb):
        ref.step(tr[b], 0.5, 0.01, 0.05)
    for t, R in enumerate(rows):
        assert np.array_equal(cpu[t], ref.rows_of(t, np.arange(R))), t
    # the bf16 run really differs from fp32 training
    ref32 = UncachedTrainer(rows, D, N, L, 4702)
    for b in range(nb):
        ref32.step(tr[b], 0.5, 0.01, 0.05)
    assert not np.array_equal(ref32.rows_of(0, np.arange(64)), ref.rows_of(0, np.arange(64)))
