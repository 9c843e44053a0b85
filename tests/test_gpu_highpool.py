"""GPU parity at the high-pooling shape (BASELINE configs[3]): n = N*L =
2048 x 80 = 163,840 lookups per table per batch (the dedup CTA's global-memory
radix path, 25-bit keys of 20M-row tables: four 8-bit passes), Zipf 0.8,
D = 128.  Two of the config's eight 20M-row tables (the other six are the
same shape; 20 GB of host tables instead of 82 GB) with Storage just above the
window working set: every Plan record and the per-slot state bit-exact, every
pooled output bit-exact, sampled final rows within 1e-5.
"""
import numpy as np
import pytest
import torch

from tests.gpu_helpers import max_window_union, run_parity
from workload import CONFIGS, sample_trace

pytestmark = pytest.mark.gpu


def test_highpool_size_global_radix_path():
    c = CONFIGS["highpool"]
    rows = c.rows[:2]
    nb = 10
    assert c.batch * c.pooling == 163_840 and rows[0] >= 1 << 24
    tr = sample_trace(rows, c.batch, c.pooling, c.alpha, nb, c.trace_seed, device="cuda").cpu()
    slots = [min(R, max_window_union(tr.numpy(), t, 3, 2) + 256) for t, R in enumerate(rows)]
    g, d, e = c.surrogate()
    rep = run_parity(rows, slots, c.dim, c.batch, c.pooling, nb, 3, 2, trace=tr,
                     init_seed=c.init_seed, gde=(g, d, e), index_dtype="int32", index_on_device=True,
                     check_slots=True, sample_rows=3000, host_alloc=True)
    assert rep["plans"] == nb and rep["pooled"] == nb
    assert rep["evictions"] > 100_000, rep["evictions"]
    assert rep["tables"]["max_rel"] <= 1e-5, rep["tables"]
