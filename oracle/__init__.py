"""CPU oracle for ScratchPipe (arXiv 2205.04702) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2205_04702_b200`` never imports it and shares no code with it.

* ``liboracle.so`` (sp_oracle.c): Part A (uncached EmbeddingBag training with
  sparse SGD) and Part B (reference scratchpad policy), plain C.
* ``pipeline.py``: Part C, the paper's cycle-level 5-stage pipeline with values
  and a RAW-hazard checker (pure Python, small cases only).

Parity pins live in tests/test_oracle_*.py; see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORC_OK, ORC_ERR_ARG, ORC_ERR_CAPACITY, ORC_ERR_INDEX = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sp_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64p = ctypes.POINTER(ctypes.c_int64)
        f32p = ctypes.POINTER(ctypes.c_float)
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.orc_version.restype = ctypes.c_int32
        L.orc_init_value.restype = ctypes.c_float
        L.orc_init_value.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32]
        L.orc_train_create.restype = P
        L.orc_train_create.argtypes = [ctypes.c_int32, i64p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_uint64]
        L.orc_train_destroy.argtypes = [P]
        L.orc_train_step.restype = ctypes.c_int32
        L.orc_train_step.argtypes = [P, i64p, f32p, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                     f32p, i32p]
        L.orc_train_get_row.argtypes = [P, ctypes.c_int32, ctypes.c_int64, f32p]
        L.orc_train_set_padding.argtypes = [P, ctypes.c_int32]
        L.orc_train_set_table_ids.argtypes = [P, P]
        L.orc_train_set_bf16.argtypes = [P, ctypes.c_int32]
        L.orc_bf16_round_array.argtypes = [ctypes.c_int64, P, P]
        L.orc_train_touched.restype = ctypes.c_int64
        L.orc_train_touched.argtypes = [P, ctypes.c_int32, i64p, ctypes.c_int64]
        L.orc_policy_create.restype = P
        L.orc_policy_create.argtypes = [ctypes.c_int32, i64p, i64p, ctypes.c_int32, ctypes.c_int32]
        L.orc_policy_destroy.argtypes = [P]
        L.orc_policy_plan.restype = ctypes.c_int32
        L.orc_policy_plan.argtypes = [P, i64p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int64, i64p, i64p, i64p, i64p, i64p, i32p]
        L.orc_policy_resident.restype = ctypes.c_int64
        L.orc_policy_resident.argtypes = [P, ctypes.c_int32, i64p, ctypes.c_int64]
        L.orc_policy_slots.argtypes = [P, ctypes.c_int32, i64p, i64p]
        L.orc_policy_set_full_sort.argtypes = [P, ctypes.c_int32]
        L.orc_policy_set_kind.argtypes = [P, ctypes.c_int32, ctypes.c_uint64]
        L.orc_policy_set_padding.argtypes = [P, ctypes.c_int32]
        L.orc_policy_pin.restype = ctypes.c_int32
        L.orc_policy_pin.argtypes = [P, ctypes.c_int32, i64p, ctypes.c_int64]
        L.orc_policy_freq.argtypes = [P, ctypes.c_int32, i64p]
        L.orc_fmaf_array.argtypes = [ctypes.c_int64, f32p, f32p, f32p, f32p]
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def fmaf32(a, b, c) -> np.ndarray:
    """Element-wise float32 fmaf (single rounding, C99 libm) with numpy broadcasting."""
    a, b, c = np.broadcast_arrays(np.asarray(a, np.float32), np.asarray(b, np.float32),
                                  np.asarray(c, np.float32))
    a, b, c = (np.ascontiguousarray(x, dtype=np.float32) for x in (a, b, c))
    out = np.empty(a.shape, np.float32)
    lib().orc_fmaf_array(a.size, _p(a, ctypes.c_float), _p(b, ctypes.c_float),
                         _p(c, ctypes.c_float), _p(out, ctypes.c_float))
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """The oracle's bf16 round-to-nearest-even (reading R28), widened to fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    lib().orc_bf16_round_array(x.size, _p(x, ctypes.c_float), _p(out, ctypes.c_float))
    return out


def init_value(seed: int, t: int, row: int, col: int) -> float:
    return float(lib().orc_init_value(seed, t, row, col))


class OracleError(RuntimeError):
    def __init__(self, code: int, batch: int, table: int):
        super().__init__(f"oracle error code={code} batch={batch} table={table}")
        self.code, self.batch, self.table = code, batch, table


class UncachedTrainer:
    """Part A: uncached EmbeddingBag training with sparse SGD (ground truth)."""

    def __init__(self, rows: Sequence[int], dim: int, batch: int, pooling: int, init_seed: int,
                 allow_padding: bool = False, table_ids: Optional[Sequence[int]] = None,
                 bf16: bool = False):
        self.rows = np.asarray(rows, dtype=np.int64)
        self.T, self.D, self.N, self.L = len(rows), dim, batch, pooling
        self._h = lib().orc_train_create(self.T, _p(self.rows, ctypes.c_int64), dim, batch,
                                         pooling, init_seed)
        if not self._h:
            raise ValueError("bad oracle config")
        if allow_padding:
            lib().orc_train_set_padding(self._h, 1)
        if bf16:  # bf16 Storage (reading R28)
            lib().orc_train_set_bf16(self._h, 1)
        if table_ids is not None:  # global table ids (table-wise sharding)
            self._gid = np.ascontiguousarray(table_ids, dtype=np.int32)
            lib().orc_train_set_table_ids(self._h, _p(self._gid, ctypes.c_int32))
        self.step_count = 0

    def close(self):
        if self._h:
            lib().orc_train_destroy(self._h)
            self._h = None

    __del__ = close

    def step(self, ids: np.ndarray, gamma: float = 0.0, delta: float = 0.0, eta: float = 0.0,
             grad: Optional[np.ndarray] = None, want_pooled: bool = False):
        ids = np.ascontiguousarray(ids, dtype=np.int64).reshape(self.T, self.N, self.L)
        pooled = np.empty((self.T, self.N, self.D), np.float32) if want_pooled else None
        g = None if grad is None else np.ascontiguousarray(grad, dtype=np.float32)
        err = ctypes.c_int32(-1)
        rc = lib().orc_train_step(self._h, _p(ids, ctypes.c_int64),
                                  None if g is None else _p(g, ctypes.c_float),
                                  gamma, delta, eta,
                                  None if pooled is None else _p(pooled, ctypes.c_float),
                                  ctypes.byref(err))
        if rc != ORC_OK:
            raise OracleError(rc, self.step_count, err.value)
        self.step_count += 1
        return pooled

    def row(self, t: int, r: int) -> np.ndarray:
        out = np.empty(self.D, np.float32)
        lib().orc_train_get_row(self._h, t, r, _p(out, ctypes.c_float))
        return out

    def rows_of(self, t: int, rows: np.ndarray) -> np.ndarray:
        return np.stack([self.row(t, int(r)) for r in rows]) if len(rows) else np.empty((0, self.D), np.float32)

    def touched(self, t: int) -> np.ndarray:
        n = lib().orc_train_touched(self._h, t, None, 0)
        out = np.empty(n, np.int64)
        lib().orc_train_touched(self._h, t, _p(out, ctypes.c_int64), n)
        return out


class PlanRecord:
    """Part B output for one (batch, table)."""
    __slots__ = ("U", "hits", "misses", "evictions", "uniq", "slot", "hit", "evicted")

    def __init__(self, counts, uniq, slot, hit, evicted):
        self.U, self.hits, self.misses, self.evictions = (int(c) for c in counts)
        U = self.U
        self.uniq, self.slot, self.hit, self.evicted = uniq[:U].copy(), slot[:U].copy(), hit[:U].astype(bool), evicted[:U].copy()

    @property
    def miss_ids(self):
        return self.uniq[~self.hit]

    @property
    def victim_slots(self):
        return self.slot[~self.hit]

    @property
    def evicted_ids(self):
        e = self.evicted[~self.hit]
        return e[e >= 0]


POLICIES = {"lru": 0, "random": 1, "lfu": 2}
LFU_FMAX = 8


class Policy:
    """Part B: reference scratchpad policy (IDs only).

    policy: "lru" (default), "random" or "lfu" (readings
    R23-R25); policy_seed: the RANDOM draw seed; allow_padding: -1 entries are
    not lookups (ragged bags, R27); pinned: per table, rows held in the
    table's last slots for the whole run (static partition, R26)."""

    def __init__(self, rows: Sequence[int], slots: Sequence[int], past: int, future: int,
                 full_sort: bool = False, policy: str = "lru", policy_seed: int = 0,
                 allow_padding: bool = False, pinned=None):
        self.rows = np.asarray(rows, dtype=np.int64)
        self.slots = np.asarray(slots, dtype=np.int64)
        self.T = len(rows)
        self.P, self.F = past, future
        self._h = lib().orc_policy_create(self.T, _p(self.rows, ctypes.c_int64),
                                          _p(self.slots, ctypes.c_int64), past, future)
        if not self._h:
            raise ValueError("bad policy config")
        if full_sort:
            lib().orc_policy_set_full_sort(self._h, 1)
        lib().orc_policy_set_kind(self._h, POLICIES[policy], policy_seed & ((1 << 64) - 1))
        if allow_padding:
            lib().orc_policy_set_padding(self._h, 1)
        if pinned is not None:
            for t, ids in enumerate(pinned):
                if ids is None or len(ids) == 0:
                    continue
                a = np.ascontiguousarray(ids, dtype=np.int64)
                if lib().orc_policy_pin(self._h, t, _p(a, ctypes.c_int64), len(a)) != ORC_OK:
                    raise ValueError(f"bad pinned rows for table {t}")

    def close(self):
        if self._h:
            lib().orc_policy_destroy(self._h)
            self._h = None

    __del__ = close

    def plan(self, trace: np.ndarray, b: int):
        """trace: [nb][T][N][L] int64 -> list of PlanRecord per table."""
        trace = np.ascontiguousarray(trace, dtype=np.int64)
        nb, T, N, L = trace.shape
        n = N * L
        counts = np.zeros(4 * T, np.int64)
        uniq = np.empty(T * n, np.int64)
        slot = np.empty(T * n, np.int64)
        hit = np.empty(T * n, np.int64)
        ev = np.empty(T * n, np.int64)
        err = ctypes.c_int32(-1)
        rc = lib().orc_policy_plan(self._h, _p(trace, ctypes.c_int64), nb, N, L, b,
                                   _p(counts, ctypes.c_int64), _p(uniq, ctypes.c_int64),
                                   _p(slot, ctypes.c_int64), _p(hit, ctypes.c_int64),
                                   _p(ev, ctypes.c_int64), ctypes.byref(err))
        if rc != ORC_OK:
            raise OracleError(rc, b, err.value)
        return [PlanRecord(counts[4 * t:4 * t + 4], uniq[t * n:(t + 1) * n], slot[t * n:(t + 1) * n],
                           hit[t * n:(t + 1) * n], ev[t * n:(t + 1) * n]) for t in range(T)]

    def resident(self, t: int) -> np.ndarray:
        n = lib().orc_policy_resident(self._h, t, None, 0)
        out = np.empty(n, np.int64)
        lib().orc_policy_resident(self._h, t, _p(out, ctypes.c_int64), n)
        return out

    def freq(self, t: int) -> np.ndarray:
        out = np.empty(int(self.slots[t]), np.int64)
        lib().orc_policy_freq(self._h, t, _p(out, ctypes.c_int64))
        return out

    def slot_state(self, t: int):
        S = int(self.slots[t])
        res = np.empty(S, np.int64)
        lu = np.empty(S, np.int64)
        lib().orc_policy_slots(self._h, t, _p(res, ctypes.c_int64), _p(lu, ctypes.c_int64))
        return res, lu
