"""Counter-based generators for traces and initial tables (inputs only).

Formulas (both numpy and torch paths compute the same IEEE operations; the
oracle's C ``orc_init_value`` re-implements ``init``):

    sm(x)        = splitmix64 finaliser (Steele et al.), all arithmetic mod 2^64
    init(s,t,r,c)= f32( f64(sm(sm(sm(sm(s) ^ t) ^ r) ^ c) >> 40) * (0.2 / 2^24) - 0.1 )
    u(s,t,b,i)   = (sm(sm(sm(sm(s ^ TRACE_SALT) ^ t) ^ b) ^ i) >> 11) * 2^-53
    rank         = #{ r : cdf[r] <= u }   (inverse CDF of p(r) ∝ (r+1)^-alpha)
    row          = feistel_t(rank)        (4-round balanced Feistel + cycle walking)

The Zipf family stands in for the paper's empirical PDFs (
SURVEY.md §8(c) reading 16).  The generated trace is laid out [nb][T][N][L],
sample-major inside each table.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

MASK64 = (1 << 64) - 1
C0 = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB
TRACE_SALT = 0x5452414345  # "TRACE"
PERM_SALT = 0x5045524D     # "PERM"
INIT_SCALE = 0.2 / 16777216.0


def _sm_int(x: int) -> int:
    """splitmix64 on a Python int (scalar helper)."""
    x = (x + C0) & MASK64
    x = ((x ^ (x >> 30)) * C1) & MASK64
    x = ((x ^ (x >> 27)) * C2) & MASK64
    return x ^ (x >> 31)


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(C0)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(C1)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(C2)
        return x ^ (x >> np.uint64(31))


def _s64(c: int) -> int:
    """Reinterpret an unsigned 64-bit constant as signed int64."""
    c &= MASK64
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 tensor viewed as uint64."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64_torch(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 over int64 tensors (two's-complement wrap == mod 2^64)."""
    x = x + _s64(C0)
    x = (x ^ _lsr(x, 30)) * _s64(C1)
    x = (x ^ _lsr(x, 27)) * _s64(C2)
    return x ^ _lsr(x, 31)


# ----------------------------------------------------------------------------
# initial embedding values
# ----------------------------------------------------------------------------

def _init_prefix(seed: int, t: int) -> int:
    return _sm_int(_sm_int(seed & MASK64) ^ (t & MASK64))


def init_rows_np(seed: int, t: int, rows: np.ndarray, dim: int) -> np.ndarray:
    """Initial values of the given rows of table t, float32 [len(rows)][dim]."""
    h2 = np.uint64(_init_prefix(seed, t))
    rows = np.asarray(rows, dtype=np.uint64).reshape(-1, 1)
    h3 = splitmix64_np(h2 ^ rows)
    cols = np.arange(dim, dtype=np.uint64).reshape(1, -1)
    h4 = splitmix64_np(h3 ^ cols)
    u24 = (h4 >> np.uint64(40)).astype(np.float64)
    return (u24 * INIT_SCALE - 0.1).astype(np.float32)


def init_table(seed: int, t: int, num_rows: int, dim: int,
               device: str | torch.device = "cpu",
               out: torch.Tensor | None = None,
               chunk_rows: int = 1 << 20) -> torch.Tensor:
    """Whole table t as float32 [num_rows][dim] (torch; CPU or CUDA).

    If ``out`` is given (e.g. a pinned host tensor) the rows are written there,
    generated on ``device`` chunk by chunk.
    """
    if out is None:
        out = torch.empty((num_rows, dim), dtype=torch.float32, device=device)
    h2 = _s64(_init_prefix(seed, t))
    cols = torch.arange(dim, dtype=torch.int64, device=device).view(1, -1)
    for r0 in range(0, num_rows, chunk_rows):
        r1 = min(num_rows, r0 + chunk_rows)
        rows = torch.arange(r0, r1, dtype=torch.int64, device=device).view(-1, 1)
        h3 = splitmix64_torch(rows ^ h2)
        h4 = splitmix64_torch(h3 ^ cols)
        u24 = _lsr(h4, 40).to(torch.float64)
        vals = (u24 * INIT_SCALE - 0.1).to(torch.float32)
        out[r0:r1].copy_(vals, non_blocking=False)
    return out


# ----------------------------------------------------------------------------
# Zipf traces
# ----------------------------------------------------------------------------

def zipf_cdf(num_rows: int, alpha: float) -> np.ndarray:
    """Normalised CDF of p(r) ∝ (r+1)^-alpha, r = 0..R-1 (float64)."""
    w = np.arange(1, num_rows + 1, dtype=np.float64) ** (-float(alpha))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    cdf[-1] = 1.0
    return cdf


def _feistel_params(num_rows: int, seed: int, t: int):
    k = max(2, math.ceil(math.log2(max(num_rows, 2))))
    if k % 2:
        k += 1
    half = k // 2
    base = _sm_int(_sm_int((seed ^ PERM_SALT) & MASK64) ^ t)
    keys = [_s64(_sm_int(base ^ r)) for r in range(4)]
    return half, keys


def feistel_perm(x: torch.Tensor, num_rows: int, seed: int, t: int) -> torch.Tensor:
    """Seeded bijection on [0, num_rows) (4-round Feistel + cycle walking)."""
    half, keys = _feistel_params(num_rows, seed, t)
    mask = (1 << half) - 1

    def once(v: torch.Tensor) -> torch.Tensor:
        lo = v & mask
        hi = (v >> half) & mask
        for key in keys:
            f = _lsr(splitmix64_torch(lo ^ key), 64 - half)
            hi, lo = lo, hi ^ f
        return (hi << half) | lo

    y = once(x)
    bad = y >= num_rows
    while bool(bad.any()):
        y[bad] = once(y[bad])
        bad = y >= num_rows
    return y


_CDF_CACHE: dict = {}


def _cdf_tensor(num_rows: int, alpha: float, device) -> torch.Tensor:
    key = (num_rows, float(alpha), str(device))
    c = _CDF_CACHE.get(key)
    if c is None:
        c = torch.from_numpy(zipf_cdf(num_rows, alpha)).to(device)
        if len(_CDF_CACHE) > 64:
            _CDF_CACHE.clear()
        _CDF_CACHE[key] = c
    return c


def sample_trace(rows: Sequence[int], batch: int, pooling: int, alpha: float,
                 num_batches: int, seed: int, *, first_batch: int = 0,
                 device: str | torch.device = "cpu",
                 dtype: torch.dtype = torch.int64) -> torch.Tensor:
    """Trace [num_batches][T][N][L] of sparse IDs (batches first_batch.. ).

    Batch b, table t, flat lookup i = s*L + p draws u(seed,t,b,i) and maps it
    through the table's Zipf inverse CDF and Feistel bijection.
    """
    T = len(rows)
    n = batch * pooling
    out = torch.empty((num_batches, T, n), dtype=dtype, device=device)
    salt = (seed ^ TRACE_SALT) & MASK64
    idx = torch.arange(n, dtype=torch.int64, device=device).view(1, -1)
    bvec = torch.arange(first_batch, first_batch + num_batches, dtype=torch.int64,
                        device=device).view(-1, 1)
    for t, R in enumerate(rows):
        cdf = _cdf_tensor(int(R), alpha, device)
        h2 = _s64(_sm_int(_sm_int(salt) ^ t))
        h3 = splitmix64_torch(bvec ^ h2)          # [nb,1]
        h4 = splitmix64_torch(h3 ^ idx)           # [nb,n]
        u = _lsr(h4, 11).to(torch.float64) * (2.0 ** -53)
        rank = torch.searchsorted(cdf, u, right=True).clamp_(max=int(R) - 1)
        out[:, t, :] = feistel_perm(rank, int(R), seed, t).to(dtype)
    return out.view(num_batches, T, batch, pooling)
