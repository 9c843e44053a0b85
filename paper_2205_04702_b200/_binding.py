"""Thin ctypes binding over libscratchpipe.so (include/scratchpipe.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  There is no CPU fallback: if the library is missing this
module raises at import, and a context cannot be created without a CUDA
device.
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libscratchpipe.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "scratchpipe.h")

SP_OK, SP_ERR_INVALID_ARG, SP_ERR_CAPACITY, SP_ERR_INDEX_RANGE, SP_ERR_STATE, SP_ERR_CUDA, \
    SP_ERR_NCCL, SP_ERR_OOM = range(8)
STATUS_NAMES = {0: "SP_OK", 1: "SP_ERR_INVALID_ARG", 2: "SP_ERR_CAPACITY", 3: "SP_ERR_INDEX_RANGE",
                4: "SP_ERR_STATE", 5: "SP_ERR_CUDA", 6: "SP_ERR_NCCL", 7: "SP_ERR_OOM"}
SP_FLAG_REGISTER_HOST = 1 << 0
SP_FLAG_INDEX_I32 = 1 << 1
SP_FLAG_INDEX_DEVICE = 1 << 2
SP_FLAG_PROFILE = 1 << 3
SP_FLAG_PADDING = 1 << 4
SP_FLAG_BF16 = 1 << 5
POLICIES = {"lru": 0, "random": 1, "lfu": 2}
KERNEL_KINDS = ["plan", "transfer", "forward", "backward", "surrogate", "flush", "h2d", "d2h"]
KERNEL_ONLY = ["plan", "transfer", "forward", "backward", "surrogate", "flush"]
RING = 16  # batches in flight inside the library (sp_internal.cuh)


class SpDesc(ctypes.Structure):
    _fields_ = [
        ("num_tables", ctypes.c_int32),
        ("rows", ctypes.POINTER(ctypes.c_int64)),
        ("host_tables", ctypes.POINTER(ctypes.c_void_p)),
        ("dim", ctypes.c_int32),
        ("slots", ctypes.POINTER(ctypes.c_int64)),
        ("window", ctypes.c_int32),
        ("past", ctypes.c_int32),
        ("future", ctypes.c_int32),
        ("batch_size", ctypes.c_int32),
        ("pooling", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("flags", ctypes.c_uint32),
        ("log_factor", ctypes.c_int32),
        ("host_threads", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("reserved", ctypes.c_uint32),
        ("policy_seed", ctypes.c_uint64),
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("num_tables_all", ctypes.c_int32),
        ("reserved2", ctypes.c_int32),
        ("table_owner", ctypes.POINTER(ctypes.c_int32)),
        ("table_ids", ctypes.POINTER(ctypes.c_int32)),
    ]


class SpStats(ctypes.Structure):
    _fields_ = [
        ("pushed", ctypes.c_int64), ("planned", ctypes.c_int64), ("transferred", ctypes.c_int64),
        ("forwarded", ctypes.c_int64), ("trained", ctypes.c_int64),
        ("uniques", ctypes.c_int64), ("hits", ctypes.c_int64), ("misses", ctypes.c_int64),
        ("evictions", ctypes.c_int64),
        ("h2d_index_bytes", ctypes.c_int64), ("h2d_row_bytes", ctypes.c_int64),
        ("d2h_row_bytes", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64 * 8), ("kernel_ms", ctypes.c_double * 8),
        ("kernel_timed", ctypes.c_int64 * 8),
        ("host_gather_ms", ctypes.c_double), ("host_scatter_ms", ctypes.c_double),
        ("host_rows_gathered", ctypes.c_int64), ("host_rows_scattered", ctypes.c_int64),
        ("wait_xfer_ms", ctypes.c_double), ("wait_list_ms", ctypes.c_double),
        ("graph_steps", ctypes.c_int64), ("graph_step_host_ms", ctypes.c_double),
        ("transfer_mode", ctypes.c_int32), ("engine_threads", ctypes.c_int32),
        ("gpu_writeback", ctypes.c_int32), ("backward_kernels", ctypes.c_int32),
        ("gather_share", ctypes.c_double),
    ]


XFER_MODES = {0: "gpu_pull", 1: "cpu_gather", 2: "cpu_gather_dma", 3: "hybrid"}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i64p = ctypes.POINTER(ctypes.c_int64)
    P = ctypes.c_void_p
    S = ctypes.c_int
    L.sp_abi_version.restype = ctypes.c_int32
    L.sp_create.argtypes = [ctypes.POINTER(SpDesc), ctypes.POINTER(ctypes.c_void_p)]
    L.sp_create.restype = S
    for name, args in [("sp_plan", [P, P]), ("sp_plan_device", [P, P]),
                       ("sp_copy_batch_stats", [P, ctypes.c_int64, P]),
                       ("sp_set_profiling", [P, ctypes.c_int32]),
                       ("sp_run_steps", [P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, P, P,
                                         ctypes.c_float, ctypes.c_float, ctypes.c_float, P]),
                       ("sp_get_timeline", [P, P, P, P, P, ctypes.c_int64, i64p]), ("sp_end_of_data", [P]), ("sp_forward", [P, P]),
                       ("sp_train", [P, P, ctypes.c_float]),
                       ("sp_surrogate_grad", [P, P, P, ctypes.c_int64, ctypes.c_float, ctypes.c_float]),
                       ("sp_flush", [P]), ("sp_destroy", [P]), ("sp_prefill", [P]),
                       ("sp_plan_csr", [P, P, P]), ("sp_pin_rows", [P, ctypes.c_int32, P, ctypes.c_int64]),
                       ("sp_last_error_batch", [P, i64p, ctypes.POINTER(ctypes.c_int32)]),
                       ("sp_get_stats", [P, ctypes.POINTER(SpStats)]),
                       ("sp_debug_plan", [P, ctypes.c_int64, ctypes.c_int32, i64p, i64p, i64p, i64p, i64p]),
                       ("sp_debug_resident", [P, ctypes.c_int32, i64p, ctypes.c_int64, i64p]),
                       ("sp_debug_slots", [P, ctypes.c_int32, i64p, i64p]),
                       ("sp_debug_storage", [P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, P]),
                       ("sp_debug_plan_profile", [P, P]), ("sp_stage_times", [P, P, P]),
                       ("sp_set_stage_timing", [P, ctypes.c_int32]), ("sp_stage_events", [P, P]),
                       ("sp_set_span_timing", [P, ctypes.c_int32]), ("sp_span_times", [P, P])]:
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = S
    L.sp_nccl_unique_id.argtypes = [P]
    L.sp_nccl_unique_id.restype = S
    i32p = ctypes.POINTER(ctypes.c_int32)
    L.sp_shard_plan.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, i32p, i32p, i64p, i32p, i64p]
    L.sp_shard_plan.restype = S
    L.sp_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    L.sp_host_alloc.restype = S
    L.sp_host_alloc_near.argtypes = [ctypes.c_size_t, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p),
                                     ctypes.POINTER(ctypes.c_int32)]
    L.sp_host_alloc_near.restype = S
    L.sp_host_free.argtypes = [P, ctypes.c_size_t]
    L.sp_host_free.restype = S
    L.sp_error_string.argtypes = [P]
    L.sp_error_string.restype = ctypes.c_char_p
    return L


lib = _load()


def header_symbols() -> List[str]:
    """Every function the public header declares."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z_]+)\s*\(", src)))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for a sharded context (sp_nccl_unique_id)."""
    buf = ctypes.create_string_buffer(128)
    st = lib.sp_nccl_unique_id(buf)
    if st != SP_OK:
        raise SpError(st, "sp_nccl_unique_id failed (NCCL library not loadable)")
    return buf.raw


def shard_plan(world: int, rank: int, owner):
    """Host-only message lists of the sharded exchange (sp_shard_plan):
    sends [(peer, local table, global table)], recvs [(peer, global table)]."""
    own = np.ascontiguousarray(owner, dtype=np.int32)
    ns, nr = ctypes.c_int64(0), ctypes.c_int64(0)
    i32 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    st = lib.sp_shard_plan(world, rank, len(own), i32(own), None, ctypes.byref(ns), None, ctypes.byref(nr))
    if st != SP_OK:
        raise SpError(st, "sp_shard_plan failed")
    snd = np.zeros(3 * ns.value, np.int32)
    rcv = np.zeros(2 * nr.value, np.int32)
    lib.sp_shard_plan(world, rank, len(own), i32(own), i32(snd), ctypes.byref(ns), i32(rcv), ctypes.byref(nr))
    return [tuple(x) for x in snd.reshape(-1, 3).tolist()], [tuple(x) for x in rcv.reshape(-1, 2).tolist()]


class HostTable:
    """A host embedding table from sp_host_alloc (THP-backed, CUDA-registered);
    `.tensor` is a float32 CPU torch view [rows][dim].  With `device`, the
    pages go to the host NUMA node closest to that GPU (sp_host_alloc_near;
    `.numa_node` is the node used, -1 for none)."""

    def __init__(self, rows: int, dim: int, device: int | None = None):
        import torch
        self.bytes = int(rows) * int(dim) * 4
        p = ctypes.c_void_p()
        self.numa_node = -1
        if device is None:
            st = lib.sp_host_alloc(self.bytes, ctypes.byref(p))
        else:
            nn = ctypes.c_int32(-1)
            st = lib.sp_host_alloc_near(self.bytes, int(device), ctypes.byref(p), ctypes.byref(nn))
            self.numa_node = nn.value
        if st != SP_OK:
            raise SpError(st, "sp_host_alloc failed")
        self.ptr = p.value
        buf = (ctypes.c_byte * self.bytes).from_address(self.ptr)
        self.tensor = torch.frombuffer(buf, dtype=torch.float32).view(int(rows), int(dim))

    def data_ptr(self):
        return self.ptr

    def free(self):
        if self.ptr:
            self.tensor = None
            lib.sp_host_free(ctypes.c_void_p(self.ptr), self.bytes)
            self.ptr = None

    __del__ = free


class SpError(RuntimeError):
    def __init__(self, status: int, msg: str, batch: int = -1, table: int = -1):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status, self.batch, self.table = status, batch, table


def _i64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class ScratchPipe:
    """One scratchpad context (the embedding tables of one GPU).

    host_tables: list of pinned CPU float32 torch tensors [rows_t, dim] (or any
    objects exposing data_ptr()).  With register_host=True ordinary host memory
    is registered by the library instead.
    """

    def __init__(self, rows: Sequence[int], host_tables, dim: int, slots: Sequence[int],
                 batch_size: int, pooling: int, window: int = 3, past: int = -1, future: int = -1,
                 device: int = 0, stream=None, index_dtype: str = "int64", index_on_device: bool = False,
                 register_host: bool = False, profile: bool = False, log_factor: int = 0,
                 host_threads: int = 0, policy: str = "lru", policy_seed: int = 0,
                 padding: bool = False, world: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                 table_owner=None, table_ids=None, bf16: bool = False):
        """world > 1 (or nccl_id given): table-wise sharding inside the library
        -- this context owns the global tables `table_ids` (ascending) of the
        `table_owner` map; forward / train exchange with NCCL and use the
        batch-sharded [T_all][N/world][D] layout.  bf16=True: bf16 Storage
        (SP_FLAG_BF16, reading R28)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("ScratchPipe needs a CUDA device (no CPU fallback)")
        self.T, self.D, self.N, self.L = len(rows), dim, batch_size, pooling
        self.device = device
        self._rows = np.ascontiguousarray(rows, dtype=np.int64)
        self._slots = np.ascontiguousarray(slots, dtype=np.int64)
        self._tables = list(host_tables)  # keep alive
        self._hp = (ctypes.c_void_p * self.T)(*[t.data_ptr() for t in self._tables])
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        flags = 0
        if register_host:
            flags |= SP_FLAG_REGISTER_HOST
        if index_dtype == "int32":
            flags |= SP_FLAG_INDEX_I32
        if index_on_device:
            flags |= SP_FLAG_INDEX_DEVICE
        if profile:
            flags |= SP_FLAG_PROFILE
        if padding:
            flags |= SP_FLAG_PADDING
        if bf16:
            flags |= SP_FLAG_BF16
        self.index_dtype, self.index_on_device = index_dtype, index_on_device
        self.world, self.rank = world, rank
        self.T_all = self.T
        own = ids = None
        self._nid = None
        if nccl_id is not None or world > 1:
            own = np.ascontiguousarray(table_owner, dtype=np.int32)
            ids = np.ascontiguousarray(table_ids, dtype=np.int32)
            self.T_all = len(own)
            self._own, self._ids = own, ids
            self._nid = ctypes.create_string_buffer(bytes(nccl_id), 128)
        i32 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)) if a is not None else None
        d = SpDesc(self.T, _i64(self._rows), self._hp, dim, _i64(self._slots), window, past, future,
                   batch_size, pooling, device, ctypes.c_void_p(stream.cuda_stream), flags, log_factor,
                   host_threads, POLICIES[policy], 0, policy_seed & ((1 << 64) - 1), world, rank,
                   ctypes.cast(self._nid, ctypes.c_void_p) if self._nid is not None else None,
                   self.T_all, 0, i32(own), i32(ids))
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            st = lib.sp_create(ctypes.byref(d), ctypes.byref(h))
        if st != SP_OK:
            raise SpError(st, "sp_create failed")
        self._h = h
        if past < 0 or future < 0:
            past, future = window, max(window - 1, 0)
        self.P, self.F = past, future
        self._pooled = None
        import collections
        self._idx_refs = collections.deque(maxlen=RING + 2)

    # ------------------------------------------------------------------ core
    def _keep(self, idx):
        """Keep a pushed index tensor alive until its batch's Plan has run:
        k_push reads it on the library's plan stream, up to RING (16) batches
        after sp_plan returns, so a temporary must not be recycled by torch's
        caching allocator before then (RING + 2 newest references are kept)."""
        self._idx_refs.append(idx)

    def _check(self, st: int):
        if st != SP_OK:
            b = ctypes.c_int64(-1)
            t = ctypes.c_int32(-1)
            lib.sp_last_error_batch(self._h, ctypes.byref(b), ctypes.byref(t))
            raise SpError(st, lib.sp_error_string(self._h).decode(), b.value, t.value)

    def plan(self, idx):
        """Push the next batch [T][N][L] (torch tensor or numpy array)."""
        import torch
        if isinstance(idx, np.ndarray):
            idx = torch.from_numpy(idx)
        want = torch.int32 if self.index_dtype == "int32" else torch.int64
        if idx.dtype != want:
            raise TypeError(f"indices must be {want}")
        if idx.numel() != self.T * self.N * self.L:
            raise ValueError("indices must have T*N*L elements")
        if self.index_on_device != idx.is_cuda:
            raise ValueError("index device does not match index_on_device")
        idx = idx.contiguous()
        self._keep(idx)  # device indices are read asynchronously on the plan stream
        self._check(lib.sp_plan(self._h, ctypes.c_void_p(idx.data_ptr())))

    def plan_device(self, idx):
        """Push a device-resident batch (any context): read on the plan stream."""
        want = "int32" if self.index_dtype == "int32" else "int64"
        if not idx.is_cuda or str(idx.dtype) != f"torch.{want}" or not idx.is_contiguous():
            raise TypeError(f"device indices must be contiguous cuda {want}")
        self._keep(idx)
        self._check(lib.sp_plan_device(self._h, ctypes.c_void_p(idx.data_ptr())))

    def plan_csr(self, values, offsets):
        """Push a ragged batch in CSR form: values int64 [nnz], offsets int64
        [T*N+1] (bag t*N+s = values[offsets[k]:offsets[k+1]]), host arrays
        (needs padding=True; sp_plan_csr)."""
        v = np.ascontiguousarray(values, dtype=np.int64)
        o = np.ascontiguousarray(offsets, dtype=np.int64)
        if o.size != self.T * self.N + 1:
            raise ValueError("offsets must have T*N+1 entries")
        self._check(lib.sp_plan_csr(self._h, v.ctypes.data_as(ctypes.c_void_p) if v.size else None,
                                    o.ctypes.data_as(ctypes.c_void_p)))

    def pin_rows(self, t: int, ids):
        """Static partition: rows `ids` of table t held in its last slots for
        the whole run (before the first plan; sp_pin_rows)."""
        a = np.ascontiguousarray(ids, dtype=np.int64)
        self._check(lib.sp_pin_rows(self._h, t, a.ctypes.data_as(ctypes.c_void_p) if a.size else None, a.size))

    def copy_batch_stats(self, b: int, host_out):
        """Async D2H of batch b's per-table (U, hits, misses, evictions) into a
        pinned int32 tensor [T][4], ordered on the context's stream."""
        self._check(lib.sp_copy_batch_stats(self._h, b, ctypes.c_void_p(host_out.data_ptr())))

    def run_steps(self, trace_dev, steps: int, pooled, grad, gamma: float, delta: float, lr: float,
                  stats_out=None, first_batch: int = 0):
        """C driver loop over a trace [nb][T][N][L] (see sp_run_steps) in device
        memory or pinned host memory.  trace[i] is batch first_batch + i."""
        if not trace_dev.is_contiguous() or not (trace_dev.is_cuda or trace_dev.is_pinned()):
            raise TypeError("trace must be a contiguous CUDA tensor or pinned host tensor")
        self._last_idx = trace_dev
        stride = trace_dev[0].numel() * trace_dev.element_size()
        base = trace_dev.data_ptr() - first_batch * stride  # batch j at base + j*stride
        self._check(lib.sp_run_steps(self._h, ctypes.c_void_p(base), first_batch + trace_dev.shape[0],
                                     stride, steps, ctypes.c_void_p(pooled.data_ptr()),
                                     ctypes.c_void_p(grad.data_ptr()), float(gamma), float(delta), float(lr),
                                     None if stats_out is None else ctypes.c_void_p(stats_out.data_ptr())))

    def set_profiling(self, on: bool):
        self._check(lib.sp_set_profiling(self._h, 1 if on else 0))

    def timeline(self):
        """[(kind, batch, start_ms, end_ms)] of profiled launches (synchronises)."""
        n = ctypes.c_int64(0)
        self._check(lib.sp_get_timeline(self._h, None, None, None, None, 0, ctypes.byref(n)))
        k = np.empty(n.value, np.int32)
        b = np.empty(n.value, np.int64)
        s0 = np.empty(n.value, np.float64)
        s1 = np.empty(n.value, np.float64)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        self._check(lib.sp_get_timeline(self._h, ptr(k), ptr(b), ptr(s0), ptr(s1), n.value, ctypes.byref(n)))
        return [(KERNEL_KINDS[int(k[i])], int(b[i]), float(s0[i]), float(s1[i])) for i in range(n.value)]

    def end_of_data(self):
        self._check(lib.sp_end_of_data(self._h))

    def pooled_shape(self):
        """[T][N][D], or [T_all][N/world][D] when sharded."""
        if self._nid is not None:
            return (self.T_all, self.N // self.world, self.D)
        return (self.T, self.N, self.D)

    def forward(self, out=None):
        import torch
        if out is None:
            out = torch.empty(self.pooled_shape(), dtype=torch.float32, device=f"cuda:{self.device}")
        self._check(lib.sp_forward(self._h, ctypes.c_void_p(out.data_ptr())))
        return out

    def train(self, grad, lr: float):
        self._check(lib.sp_train(self._h, ctypes.c_void_p(grad.data_ptr()), float(lr)))

    def surrogate(self, pooled, gamma: float, delta: float, out=None):
        import torch
        if out is None:
            out = torch.empty_like(pooled)
        if not (pooled.is_contiguous() and out.is_contiguous() and out.numel() == pooled.numel()):
            raise ValueError("surrogate: contiguous tensors of equal size required")
        self._check(lib.sp_surrogate_grad(self._h, ctypes.c_void_p(pooled.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), pooled.numel(),
                                          float(gamma), float(delta)))
        return out

    def flush(self):
        self._check(lib.sp_flush(self._h))

    def prefill(self):
        """All rows resident before the first batch (needs slots == rows)."""
        self._check(lib.sp_prefill(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib.sp_destroy(self._h)
            self._h = None

    __del__ = close

    def stats(self) -> dict:
        s = SpStats()
        st = lib.sp_get_stats(self._h, ctypes.byref(s))
        out = {k: getattr(s, k) for k, _ in SpStats._fields_[:12]}
        out["kernel_launches"] = dict(zip(KERNEL_KINDS, list(s.kernel_launches)))
        out["kernel_ms"] = dict(zip(KERNEL_KINDS, list(s.kernel_ms)))
        out["kernel_timed"] = dict(zip(KERNEL_KINDS, list(s.kernel_timed)))
        for k in ("host_gather_ms", "host_scatter_ms", "host_rows_gathered", "host_rows_scattered",
                  "wait_xfer_ms", "wait_list_ms", "graph_steps", "graph_step_host_ms", "engine_threads",
                  "gpu_writeback", "gather_share", "backward_kernels"):
            out[k] = getattr(s, k)
        out["transfer_mode"] = XFER_MODES.get(s.transfer_mode, str(s.transfer_mode))
        out["status"] = st
        return out

    # --------------------------------------------------------- introspection
    def debug_plan(self, b: int, t: int) -> dict:
        n = self.N * self.L
        counts = np.zeros(4, np.int64)
        uniq, slot, hit, ev = (np.empty(n, np.int64) for _ in range(4))
        self._check(lib.sp_debug_plan(self._h, b, t, _i64(counts), _i64(uniq), _i64(slot), _i64(hit), _i64(ev)))
        U = int(counts[0])
        return {"U": U, "hits": int(counts[1]), "misses": int(counts[2]), "evictions": int(counts[3]),
                "uniq": uniq[:U].copy(), "slot": slot[:U].copy(), "hit": hit[:U].astype(bool),
                "evicted": ev[:U].copy()}

    def debug_resident(self, t: int) -> np.ndarray:
        n = ctypes.c_int64(0)
        self._check(lib.sp_debug_resident(self._h, t, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, np.int64)
        self._check(lib.sp_debug_resident(self._h, t, _i64(out), n.value, ctypes.byref(n)))
        return out

    def debug_slots(self, t: int):
        S = int(self._slots[t])
        res, lu = np.empty(S, np.int64), np.empty(S, np.int64)
        self._check(lib.sp_debug_slots(self._h, t, _i64(res), _i64(lu)))
        return res, lu

    def set_stage_timing(self, on: bool):
        self._check(lib.sp_set_stage_timing(self._h, 1 if on else 0))

    def stage_times(self) -> dict:
        """Mean ms per step of each stage over the last 16 steps (events inside
        the step graphs / around each transfer; sp_stage_times)."""
        ms = np.zeros(5, np.float64)
        n = np.zeros(5, np.int32)
        self._check(lib.sp_stage_times(self._h, ms.ctypes.data_as(ctypes.c_void_p), n.ctypes.data_as(ctypes.c_void_p)))
        names = ["plan", "transfer", "forward", "surrogate", "backward"]
        return {k: {"ms": float(ms[i]), "n": int(n[i])} for i, k in enumerate(names)}

    def stage_events(self) -> np.ndarray:
        """[16][8] ms of the stage events of the last 16 timed steps relative
        to the earliest plan start (NaN: not recorded); sp_stage_events."""
        out = np.zeros(RING * 8, np.float64)
        self._check(lib.sp_stage_events(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out.reshape(RING, 8)

    def set_span_timing(self, on: bool):
        self._check(lib.sp_set_span_timing(self._h, 1 if on else 0))

    def span_times(self) -> np.ndarray:
        """[5 kinds][16 ring slots][start, end] ms (plan, transfer, forward,
        surrogate, backward) of the last launch per slot, from the kernels'
        own %globaltimer stamps (NaN: not recorded); sp_span_times."""
        out = np.zeros(5 * RING * 2, np.float64)
        self._check(lib.sp_span_times(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out.reshape(5, RING, 2)

    def debug_plan_profile(self) -> dict:
        """k_push per-CTA wall time while profiling: mean us per launch of the
        Plan CTA and of the dedup CTA of each table (sp_debug_plan_profile)."""
        T = len(self._slots)
        out = np.zeros(18 * T + 2 + 4096, np.uint64)
        self._check(lib.sp_debug_plan_profile(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        sp = out[18 * T + 2:].reshape(4, 1024)
        ok = (sp[1] > 0) & (sp[0] != np.uint64(0xFFFFFFFFFFFFFFFF))
        spans = {"span_us": ((sp[1][ok] - sp[0][ok]).astype(np.float64) / 1e3).tolist(),
                 "plan_cta_max_us": (sp[2][ok].astype(np.float64) / 1e3).tolist(),
                 "dedup_cta_max_us": (sp[3][ok].astype(np.float64) / 1e3).tolist()}
        npl, nde = max(1, int(out[2 * T]) // T), max(1, int(out[2 * T + 1]) // T)
        ph = out[2 * T + 2:18 * T + 2].astype(np.float64).reshape(2, T, 8)
        return {"plan_us": (out[:T].astype(np.float64) / npl / 1e3).tolist(),
                "dedup_us": (out[T:2 * T].astype(np.float64) / nde / 1e3).tolist(),
                "plan_phase_us": (ph[0] / npl / 1e3).tolist(), "dedup_phase_us": (ph[1] / nde / 1e3).tolist(),
                "launches": [int(out[2 * T]) // T, int(out[2 * T + 1]) // T], "per_launch": spans}

    def debug_storage(self, t: int, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = int(self._slots[t]) - first
        out = np.empty((count, self.D), np.float32)
        self._check(lib.sp_debug_storage(self._h, t, first, count, out.ctypes.data_as(ctypes.c_void_p)))
        return out
