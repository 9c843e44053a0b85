"""GPU parity of the bf16 Storage variant (DESIGN.md reading
R28) against the oracle's bf16 mode (`UncachedTrainer(bf16=True)`, pinned in
tests/test_oracle_bf16.py).

With SP_FLAG_BF16 the scratchpad holds every resident row rounded to bf16
(nearest even) on fill and after each SGD update; the forward widens and
folds in fp32, the gradient coalescing stays fp64, the host tables stay fp32
and a write-back widens exactly.  Bar: every Plan record and the per-slot
state bit-exact (the policy does not see the values), pooled outputs
bit-exact (the fold reads the same bf16 values in the same order), final
tables bit-exact except where the fp64 pieces of a row spanning backward
tiles round differently than the oracle's sequential sum (R7); such a
difference can move a stored value by at most one bf16 unit (relative
2^-7), so that is the table tolerance, with the mismatch count bounded.
"""
import numpy as np
import pytest
import torch

from oracle import UncachedTrainer
from paper_2205_04702_b200 import ScratchPipe, SpError
from tests.gpu_helpers import max_window_union, pinned_tables, run_parity
from workload import sample_trace

pytestmark = pytest.mark.gpu
BF16_TOL = 2.0 ** -7


def _assert_bf16(rep, max_mismatch_frac=1e-3):
    t = rep["tables"]
    assert t["max_rel"] <= BF16_TOL, t
    assert t["mismatch"] <= max_mismatch_frac * max(1, t["rows"]) * 1, t


def _bf16_valued(x: np.ndarray) -> bool:
    return bool(np.all((x.view(np.uint32) & 0xFFFF) == 0))


@pytest.mark.parametrize("D", [8, 24, 64, 128, 256, 1024])
def test_bf16_parity_dims(D):
    """D = 8 / 24: bulk-copy staging (no tile::gather4 for bf16 rows unless
    D % 16 == 0), D = 24 the generic forward; D = 64 / 128 / 256 gather4;
    D = 1024: two rows per tile, 64 KB of k_bwd_rows partials."""
    rows, N, L, nb = [5000, 700, 90], 96, 3, 40
    tr = sample_trace(rows, N, L, 0.9, nb, 51)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 4) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.05), bf16=True)
    assert rep["evictions"] > 200 and rep["pooled"] == nb
    _assert_bf16(rep)


@pytest.mark.parametrize("env", [{"SP_CPU_GATHER": "0"}, {"SP_CPU_GATHER": "1"},
                                 {"SP_CPU_GATHER": "0", "SP_WRITEBACK": "gpu"},
                                 {"SP_GATHER_FRAC": "0.5"},
                                 {"SP_BWD_G4": "0"}, {"SP_BWD_TMA": "0"},
                                 {"SP_XFER": "warp"}, {"SP_BWD": "rec"}])
def test_bf16_transfer_and_backward_modes(env, monkeypatch):
    """Every transfer mode converts in k_pullfill (GPU pull, CPU gather,
    hybrid, the kernel's own write-back of widened victims); every staging
    mode of the tiled backward; SP_XFER=warp / SP_BWD=rec fall back to the
    kernels that handle bf16 rows."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rows, D, N, L, nb = [5000, 700, 90], 32, 96, 3, 40
    tr = sample_trace(rows, N, L, 0.9, nb, 52)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 4) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.05), bf16=True)
    assert rep["evictions"] > 200
    _assert_bf16(rep)


def test_bf16_rows_spanning_tiles():
    """L = 1 with a steep Zipf head: the hottest rows span many backward
    tiles (fp64 pieces folded in tile order, groups of 8 above 8 pieces)."""
    rows, D, N, L, nb = [200000, 3000], 64, 4096, 1, 12
    tr = sample_trace(rows, N, L, 1.2, nb, 53)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 64) for t, R in enumerate(rows)]
    gde = (float(np.float32(0.5 / N)), float(np.float32(0.01 / N)), 1.0)
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=gde, bf16=True)
    _assert_bf16(rep, max_mismatch_frac=1e-2)


def test_bf16_padding_ragged_bags():
    rows, D, N, L, nb = [800, 120, 3], 16, 32, 4, 40
    tr = sample_trace(rows, N, L, 1.0, nb, 61).numpy().copy()
    rng = np.random.default_rng(1)
    mask = rng.random(tr.shape) < 0.35
    mask[:, :, ::7, :] = True
    tr[mask] = -1
    tr = torch.from_numpy(tr)
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 6) for t, R in enumerate(rows)]
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02), padding=True, bf16=True)
    assert rep["evictions"] > 100
    _assert_bf16(rep)


def test_bf16_pinned_rows():
    rows, D, N, L, nb = [1500, 200], 16, 32, 2, 50
    tr = sample_trace(rows, N, L, 1.1, nb, 66)
    pinned, slots = [], []
    for t, R in enumerate(rows):
        ids, cnt = np.unique(tr.numpy()[:10, t], return_counts=True)
        pinned.append(np.sort(ids[np.argsort(-cnt, kind="stable")[:40]]))
        slots.append(min(R, max_window_union(tr.numpy(), t, 3, 2) + 44))
    rep = run_parity(rows, slots, D, N, L, nb, 3, 2, trace=tr, gde=(0.5, 0.01, 0.02), pinned=pinned, bf16=True)
    _assert_bf16(rep)


def test_bf16_prefill_graph_replay():
    """sp_prefill rounds every row on the GPU; sp_run_steps replays graphs."""
    rows, D, N, L, nb = [900, 60, 333], 16, 32, 3, 25
    tr = sample_trace(rows, N, L, 1.0, nb, 41)
    tables = pinned_tables(rows, D, 4702)
    sp = ScratchPipe(rows, tables, D, list(rows), N, L, index_dtype="int32", index_on_device=True, bf16=True)
    sp.prefill()
    st0 = sp.debug_storage(1)
    assert _bf16_valued(st0)
    want0 = tables[1].numpy()
    from oracle import bf16_round
    assert np.array_equal(st0, bf16_round(want0))  # the GPU's rounding == the oracle's
    dev = tr.to(torch.int32).cuda().contiguous()
    pooled = torch.empty((3, N, D), device="cuda")
    grad = torch.empty_like(pooled)
    g, d, e = 0.5, 0.01, 0.05
    sp.run_steps(dev, nb, pooled, grad, g, d, e)
    sp.flush()
    orc = UncachedTrainer(rows, D, N, L, 4702, bf16=True)
    for b in range(nb):
        orc.step(tr.numpy()[b], g, d, e)
    for t in range(3):
        touched = orc.touched(t)
        got = tables[t][torch.from_numpy(touched)].numpy()
        want = orc.rows_of(t, touched)
        assert _bf16_valued(got)
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-4)) <= BF16_TOL
    sp.close()


def test_bf16_rounding_ties_and_specials():
    """Rows with values on bf16 ties (round half to even), subnormals, huge
    magnitudes, +-0 and +-inf: the GPU rounding (k_rows_to_bf16, the same
    SRow<true>::nar as k_pullfill and k_bwd_tile) equals the oracle's
    (and torch's) bit for bit."""
    R, D = 64, 16
    h = torch.empty((R, D), dtype=torch.float32).pin_memory()
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2 ** 32, size=(R, D), dtype=np.uint64).astype(np.uint32)
    bits[0, :8] = np.array([0x3F808000, 0x3F818000, 0x3F80C000, 0x3F817FFF, 0x00008000, 0x00018000,
                            0x7F7FFFFF, 0x80000000], np.uint32)  # ties, subnormal ties, max, -0
    bits[0, 8:10] = np.array([0x7F800000, 0xFF800000], np.uint32)  # +-inf
    vals = bits.view(np.float32).copy()
    vals[np.isnan(vals)] = 1.0  # (no NaN payload cases)
    h.copy_(torch.from_numpy(vals))
    sp = ScratchPipe([R], [h], D, [R], 4, 1, bf16=True)
    sp.prefill()
    got = sp.debug_storage(0)
    from oracle import bf16_round
    want = bf16_round(vals)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(want, torch.from_numpy(vals).to(torch.bfloat16).float().numpy())
    sp.close()


def test_bf16_rejects_dim_not_multiple_of_8():
    rows, D = [100], 12
    with pytest.raises(SpError):
        ScratchPipe(rows, pinned_tables(rows, D, 1), D, [50], 4, 1, bf16=True)
