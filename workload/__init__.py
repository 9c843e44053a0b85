"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the ScratchPipe method (no dedup, no
policy, no gather/reduce, no SGD).  It only produces the two inputs the method
consumes:

* sparse-ID traces: i.i.d. Zipf ranks ("use these PDFs to
  generate ... access traces"; SURVEY.md §8(c) reading 16) scattered through a
  per-table Feistel bijection rank -> row ("per-table seeded
  random permutation mapping rank -> row ID");
* initial embedding values: uniform in [-0.1, 0.1) from a counter hash of
  (seed, table, row, col) (SURVEY.md §8(c) reading 17).

Both are pure functions of their seeds.  The oracle re-implements the same
counter-based init generator in C (allowed: "each side implements the same
counter-based generator"); ``tests/test_workload.py`` pins the two together.
"""
from .gen import (  # noqa: F401
    splitmix64_np,
    init_rows_np,
    init_table,
    zipf_cdf,
    feistel_perm,
    sample_trace,
)
from .configs import CONFIGS, WorkloadConfig, get_config  # noqa: F401
