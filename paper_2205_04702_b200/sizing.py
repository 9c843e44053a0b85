"""Storage sizing rules (host logic, no device code).

worst_case_storage_bytes: PAPER.md §6.4, P:1207-1213 — Storage must hold every
embedding gathered by the mini-batches inside the sliding window:
(tables x gathers per table x batch x dim x 4 B) x (batches in window), with
P + 1 + F = 2w batches in the window (P = w past, F = w - 1 future; Fig. 8
caption P:806-811).  The paper's default model gives 960 MB (MiB).
"""
from __future__ import annotations

import math
from typing import List, Sequence


def window_batches(window: int) -> int:
    """Batches inside the sliding window: past P=w, current, future F=w-1."""
    return window + 1 + (window - 1)


def worst_case_storage_bytes(tables: int, pooling: int, batch: int, dim: int,
                             window: int = 3, elem_bytes: int = 4) -> int:
    return tables * pooling * batch * dim * elem_bytes * window_batches(window)


def slots_for_fraction(rows: Sequence[int], frac: float, batch: int, pooling: int,
                       window: int = 3) -> List[int]:
    """S_t = min(R_t, max(ceil(frac*R_t), 2w*N*L)) (SURVEY.md §8.0 slot rule):
    never fewer slots than the worst-case window working set of one table."""
    floor = window_batches(window) * batch * pooling
    return [min(int(R), max(math.ceil(frac * R), floor)) for R in rows]
