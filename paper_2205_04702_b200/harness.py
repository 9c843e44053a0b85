"""The training loop around a ScratchPipe context (harness, not the method).

``run_loop`` drives the library the way a trainer would:
push F+P+1 batches ahead, then per iteration push the next batch (or signal
end of data), forward, the MLP stand-in (surrogate gradient kernel), train.
Callbacks let tests inspect every Plan record and pooled output;
``on_plan(b, newest)`` gets newest=True when Plan(b) is the latest Plan
enqueued (so slot-level state reflects exactly Plan(b)).
"""
from __future__ import annotations

from typing import Callable, Optional

import torch


def run_loop(sp, trace, gamma: float, delta: float, eta: float,
             on_plan: Optional[Callable[[int, bool], None]] = None,
             on_pooled: Optional[Callable[[int, torch.Tensor], None]] = None,
             flush: bool = True, num_batches: Optional[int] = None,
             push: Optional[Callable] = None):
    """trace: indexable by batch -> [T][N][L] tensor (CPU or CUDA per the
    context's index placement; or anything `push(sp, j)` understands, e.g. a
    CSR batch list for sp_plan_csr).  Returns the number of batches trained."""
    nb = len(trace) if num_batches is None else num_batches
    ahead = sp.F + sp.P + 1
    pooled = torch.empty((sp.T, sp.N, sp.D), dtype=torch.float32, device=f"cuda:{sp.device}")
    grad = torch.empty_like(pooled)
    planned = 0

    def do_push(j):
        nonlocal planned
        if push is None:
            sp.plan(trace[j])
        else:
            push(sp, j)
        while planned <= j - sp.F - 1:  # Plan(b) runs at push(b+F+1)
            if on_plan:  # second argument: this Plan is the newest one enqueued
                on_plan(planned, planned == j - sp.F - 1)
            planned += 1

    for j in range(min(ahead, nb)):
        do_push(j)
    eod = False
    for b in range(nb):
        j = b + ahead
        if j < nb:
            do_push(j)
        elif not eod:
            sp.end_of_data()
            eod = True
            while planned < nb:
                if on_plan:
                    on_plan(planned, planned == nb - 1)
                planned += 1
        sp.forward(pooled)
        if on_pooled:
            on_pooled(b, pooled)
        sp.surrogate(pooled, gamma, delta, out=grad)
        sp.train(grad, eta)
    if not eod:
        sp.end_of_data()
    if flush:
        sp.flush()
    return nb
