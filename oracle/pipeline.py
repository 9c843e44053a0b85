"""Part C: the paper's cycle-level ScratchPipe pipeline with values and a RAW
hazard checker — TEST INFRASTRUCTURE ONLY (pure Python; small cases only).

Stages and their lags (Fig. 8):
    Plan(c)  Collect(c-1)  Exchange(c-2)  Insert(c-3)  Train(c-4)
within each cycle in a configurable order (a permutation of "PCEIT").

* Plan      Part B policy (oracle.Policy) decides hits, misses, victims.
* Collect   reads missed rows from the CPU tables and victims from Storage
            (P:688-696).
* Exchange  moves them (no value change here).
* Insert    writes victims back into the CPU tables and fills Storage
            (P:702-704).
* Train     gathers from Storage through the slot map frozen at Plan,
            forward (fp32 left fold over p), surrogate g = fmaf(gamma, pooled,
            delta), coalesce (fp64 sum, rounded to fp32), SGD fmaf(-eta, g, w)
            into Storage.

Hazards reported (RAW dependencies 1-4 of P:735-765):
* ``train-miss``     Train found a slot whose tag is not the planned ID
                     (the "always hits" claim)
* ``evict-pending``  Collect read a victim slot that an earlier batch still has
                     to write (its Train or its Insert): RAW-2 / RAW-3
* ``stale-cpu-read`` Collect read a CPU row whose write-back is still pending:
                     RAW-4
After the drain, every resident slot is written back (reading R10) and the CPU
tables are returned; with a hazard-free window they must equal Part A bit for
bit.
"""
from __future__ import annotations

import numpy as np

from . import Policy, bf16_round, fmaf32, init_value


class PipelineSim:
    STAGES = "PCEIT"

    def __init__(self, rows, slots, dim, batch, pooling, past, future, init_seed,
                 gamma, delta, eta, order="TICEP", init_tables=None, bf16=False):
        assert sorted(order) == sorted(self.STAGES)
        self.rows, self.slots = list(rows), list(slots)
        self.T, self.D, self.N, self.L = len(rows), dim, batch, pooling
        self.P, self.F = past, future
        self.order = order
        # bf16 Storage (reading R28): the scratchpad holds rows rounded to bf16,
        # on Insert and after every update; the CPU tables stay fp32
        self.rnd = bf16_round if bf16 else (lambda v: v)
        self.gamma, self.delta, self.eta = np.float32(gamma), np.float32(delta), np.float32(eta)
        if init_tables is None:
            init_tables = [np.array([[init_value(init_seed, t, r, j) for j in range(dim)]
                                     for r in range(R)], np.float32) for t, R in enumerate(rows)]
        self.cpu = [np.array(x, np.float32, copy=True) for x in init_tables]
        self.storage = [np.zeros((S, dim), np.float32) for S in slots]
        self.tag = [np.full(S, -1, np.int64) for S in slots]
        self.policy = Policy(rows, slots, past, future)
        self.hazards = []
        self.plans = {}
        self.pending_wb = [dict() for _ in rows]          # row -> batch that evicted it
        self.pending_slot_writes = [dict() for _ in rows]  # slot -> set of (batch, stage)

    # ------------------------------------------------------------------ stages
    def _plan(self, trace, b):
        recs = self.policy.plan(trace, b)
        plan = []
        for t, r in enumerate(recs):
            slot_of = dict(zip(r.uniq.tolist(), r.slot.tolist()))
            fills = [(int(i), int(s), int(o)) for i, s, o, h in zip(r.uniq, r.slot, r.evicted, r.hit) if not h]
            plan.append({"slot_of": slot_of, "fills": fills})
            for (_, s, o) in fills:
                if o >= 0:
                    self.pending_wb[t][o] = b
                self.pending_slot_writes[t].setdefault(s, set()).add((b, "I"))
            for s in set(slot_of.values()):
                self.pending_slot_writes[t].setdefault(s, set()).add((b, "T"))
        self.plans[b] = {"tables": plan}

    def _collect(self, b):
        pl = self.plans[b]
        for t, tp in enumerate(pl["tables"]):
            fill_vals, evict_vals = [], []
            for (x, s, o) in tp["fills"]:
                wb = self.pending_wb[t].get(x)
                if wb is not None and wb < b:
                    self.hazards.append(("stale-cpu-read", b, t, x))
                fill_vals.append(self.cpu[t][x].copy())
                if o >= 0:
                    pend = [w for w in self.pending_slot_writes[t].get(s, ()) if w[0] < b]
                    if pend:
                        self.hazards.append(("evict-pending", b, t, s))
                    evict_vals.append(self.storage[t][s].copy())
                else:
                    evict_vals.append(None)
            tp["fill_vals"], tp["evict_vals"] = fill_vals, evict_vals

    def _exchange(self, b):
        pass  # values already in the per-batch buffers (Exchange moves them)

    def _insert(self, b):
        pl = self.plans[b]
        for t, tp in enumerate(pl["tables"]):
            for (x, s, o), fv, ev in zip(tp["fills"], tp["fill_vals"], tp["evict_vals"]):
                if o >= 0:
                    self.cpu[t][o] = ev
                    if self.pending_wb[t].get(o) == b:
                        del self.pending_wb[t][o]
                self.storage[t][s] = self.rnd(fv)
                self.tag[t][s] = x
                self.pending_slot_writes[t][s].discard((b, "I"))

    def _train(self, trace, b):
        pl = self.plans.pop(b)
        ids_b = trace[b]
        for t, tp in enumerate(pl["tables"]):
            ids = ids_b[t].reshape(self.N, self.L)
            slot_of = tp["slot_of"]
            for x, s in slot_of.items():
                if self.tag[t][s] != x:
                    self.hazards.append(("train-miss", b, t, x))
            st = self.storage[t]
            pooled = np.empty((self.N, self.D), np.float32)
            for s_ in range(self.N):
                acc = st[slot_of[int(ids[s_, 0])]].copy()
                for p in range(1, self.L):
                    acc = (acc + st[slot_of[int(ids[s_, p])]]).astype(np.float32)
                pooled[s_] = acc
            g = fmaf32(self.gamma, pooled, self.delta)
            for x in sorted(slot_of):
                acc = np.zeros(self.D, np.float64)
                for occ in np.nonzero(ids.reshape(-1) == x)[0]:
                    acc += g[occ // self.L].astype(np.float64)
                s = slot_of[x]
                st[s] = self.rnd(fmaf32(-self.eta, acc.astype(np.float32), st[s]))
            for s in set(slot_of.values()):
                self.pending_slot_writes[t][s].discard((b, "T"))

    # ------------------------------------------------------------------- run
    def run(self, trace):
        trace = np.ascontiguousarray(trace, dtype=np.int64)
        nb = trace.shape[0]
        lag = {"P": 0, "C": 1, "E": 2, "I": 3, "T": 4}
        for c in range(nb + 4):
            for st in self.order:
                b = c - lag[st]
                if not (0 <= b < nb):
                    continue
                if st == "P":
                    self._plan(trace, b)
                elif st == "C":
                    self._collect(b)
                elif st == "E":
                    self._exchange(b)
                elif st == "I":
                    self._insert(b)
                else:
                    self._train(trace, b)
        # flush: every resident slot is dirty and written back
        for t in range(self.T):
            for s in range(self.slots[t]):
                if self.tag[t][s] >= 0:
                    self.cpu[t][self.tag[t][s]] = self.storage[t][s]
        return self.cpu
