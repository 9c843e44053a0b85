"""The BASELINE.json configurations as concrete synthetic workloads.

Cardinalities: the public Criteo-Kaggle (DLRM) and MLPerf Criteo-1TB lists
(not in /root/reference; SURVEY.md §8.0 allows "any list with the same caps").
Slot rule: S_t = min(R_t, max(ceil(x*R_t), 2w*N*L)); tiny uses
128 slots per table (per-table pools).
Surrogate gradient (MLP stand-in): g = fmaf(gamma, pooled, delta);
large configs fold the 1/N mean into gamma/delta.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

CRITEO_KAGGLE = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145,
                 5683, 8351593, 3194, 27, 14992, 5461306, 10, 5652, 2173, 4,
                 7046547, 18, 15, 286181, 105, 142572]
CRITEO_TB = [39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63, 38532951,
             2953546, 403346, 10, 2208, 11938, 155, 4, 976, 14, 39979771,
             25641295, 39664984, 585935, 12972, 108, 36]


@dataclass
class WorkloadConfig:
    name: str
    rows: List[int]
    dim: int
    batch: int
    pooling: int
    alpha: float
    slot_frac: Optional[float] = None
    slots_fixed: Optional[List[int]] = None
    window: int = 3
    num_batches: int = 20
    trace_seed: int = 2205
    init_seed: int = 4702
    gamma: float = 0.5
    delta: float = 0.01
    eta: float = 0.01
    mean_surrogate: bool = False
    preroll: int = 0          # untimed batches to reach steady state in bench
    description: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def num_tables(self) -> int:
        return len(self.rows)

    @property
    def slots(self) -> List[int]:
        if self.slots_fixed is not None:
            return list(self.slots_fixed)
        floor = 2 * self.window * self.batch * self.pooling
        return [min(R, max(math.ceil(self.slot_frac * R), floor)) for R in self.rows]

    def surrogate(self):
        """(gamma', delta', eta) as float32-representable Python floats."""
        import numpy as np
        if self.mean_surrogate:
            g = float(np.float32(self.gamma / self.batch))
            d = float(np.float32(self.delta / self.batch))
        else:
            g = float(np.float32(self.gamma))
            d = float(np.float32(self.delta))
        return g, d, float(np.float32(self.eta))

    def with_(self, **kw) -> "WorkloadConfig":
        import dataclasses
        return dataclasses.replace(self, **kw)


CONFIGS = {
    "tiny": WorkloadConfig(
        name="tiny", rows=[1000, 1000], dim=16, batch=8, pooling=4, alpha=1.05,
        slots_fixed=[128, 128], window=3, num_batches=20,
        description="2 tables x 1,000 rows x dim 16, batch 8, pooling 4, Zipf 1.05, 128 slots, window 3, 20 batches"),
    "kaggle": WorkloadConfig(
        name="kaggle", rows=[min(r, 10_000_000) for r in CRITEO_KAGGLE], dim=64,
        batch=2048, pooling=1, alpha=1.1, slot_frac=0.10, window=3,
        eta=1.0, mean_surrogate=True, preroll=6000,
        description="Criteo-Kaggle-shaped: 26 tables (<=10M rows), dim 64, batch 2048, pooling 1, Zipf 1.1, 10% slots"),
    "terabyte": WorkloadConfig(
        name="terabyte", rows=list(CRITEO_TB), dim=128, batch=4096, pooling=1,
        alpha=1.05, slot_frac=0.05, window=3, eta=1.0, mean_surrogate=True,
        preroll=6000,
        description="Criteo-Terabyte-shaped: 26 tables (<=40M rows), dim 128, batch 4096, pooling 1, Zipf 1.05, 5% slots"),
    "highpool": WorkloadConfig(
        name="highpool", rows=[20_000_000] * 8, dim=128, batch=2048, pooling=80,
        alpha=0.8, slot_frac=0.10, window=3, eta=1.0, mean_surrogate=True,
        preroll=50,
        description="high-pooling low-locality: 8 x 20M rows, dim 128, batch 2048, pooling 80, Zipf 0.8, 10% slots"),
    "sharded64": WorkloadConfig(
        name="sharded64", rows=[10_000_000] * 64, dim=128, batch=8192, pooling=20,
        alpha=1.05, slots_fixed=[1_000_000] * 64, window=3, eta=0.25,
        mean_surrogate=True, preroll=100,
        description="8-GPU table-wise sharded: 64 x 10M x dim 128, batch 8192, pooling 20, 1M slots per table"),
}


def get_config(name: str) -> WorkloadConfig:
    return CONFIGS[name]
