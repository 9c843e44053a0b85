"""Shared GPU-vs-oracle parity driver for the -m gpu tests."""
from __future__ import annotations

import numpy as np
import torch

from oracle import Policy, UncachedTrainer
from paper_2205_04702_b200 import ScratchPipe
from paper_2205_04702_b200.harness import run_loop
from workload import init_rows_np, init_table, sample_trace


def pinned_tables(rows, D, seed, device="cuda", pin=True, host_alloc=False):
    out = []
    for t, R in enumerate(rows):
        if host_alloc:  # sp_host_alloc: THP-backed, registered by the library allocator
            from paper_2205_04702_b200 import HostTable
            ht = HostTable(R, D, device=0 if host_alloc == "near" else None)  # "near": sp_host_alloc_near
            init_table(seed, t, R, D, device=device, out=ht.tensor)
            out.append(ht)
            continue
        h = torch.empty((R, D), dtype=torch.float32)
        if pin:
            h = h.pin_memory()
        init_table(seed, t, R, D, device=device, out=h)
        out.append(h)
    return out


def max_window_union(trace_np, t, P, F):
    nb = trace_np.shape[0]
    best = 0
    for b in range(nb):
        lo, hi = max(0, b - P), min(nb - 1, b + F)
        best = max(best, len(np.unique(trace_np[lo:hi + 1, t])))
    return best


def compare_tables(got: np.ndarray, want: np.ndarray, init: np.ndarray):
    """SURVEY §8(c) metric: max |x-ref| / max(|ref|, 1e-4) and the error
    relative to the update size (sensitive to a lost update)."""
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-4)
    upd = np.max(np.abs(want - init)) if want.size else 0.0
    return {
        "max_rel": float(rel.max()) if rel.size else 0.0,
        "mismatch": int(np.sum(got != want)),
        "rel_to_update": float(np.max(np.abs(got - want)) / upd) if upd > 0 else 0.0,
    }


def run_parity(rows, slots, D, N, L, nb, P, F, alpha=1.05, trace_seed=2205, init_seed=4702,
               gde=(0.5, 0.01, 0.01), index_dtype="int64", index_on_device=False, log_factor=0,
               check_plans=True, check_slots=True, check_pooled=True, trace=None,
               register_host=False, profile=False, sample_rows=None, host_alloc=False,
               tables=None, policy_kw=None, padding=False, pinned=None, push=None, sp_kw=None,
               bf16=False):
    """tables: pre-allocated host tables (HostTable or pinned tensors), already
    holding init(init_seed) values; policy_kw: extra ScratchPipe / Policy
    arguments of a replacement-policy variant (policy, policy_seed); padding:
    -1 entries are "no lookup" on both sides; pinned: per table, rows pinned
    in the last slots (sp_pin_rows / the oracle's static partition); push:
    optional push(sp, j) replacing sp.plan(trace[j]) (e.g. sp_plan_csr);
    bf16: bf16 Storage on both sides (SP_FLAG_BF16 / the oracle's bf16 mode,
    reading R28)."""
    g, d, e = gde
    if trace is None:
        trace = sample_trace(rows, N, L, alpha, nb, trace_seed)
    trace_np = trace.numpy()
    if tables is None:
        tables = pinned_tables(rows, D, init_seed, pin=not register_host, host_alloc=host_alloc)
    views = [getattr(t, "tensor", t) for t in tables]
    feed = trace.to(torch.int32 if index_dtype == "int32" else torch.int64)
    if index_on_device:
        feed = feed.cuda()
    pkw = dict(policy_kw or {})
    sp = ScratchPipe(rows, tables, D, slots, N, L, past=P, future=F, index_dtype=index_dtype,
                     index_on_device=index_on_device, log_factor=log_factor,
                     register_host=register_host, profile=profile, padding=padding, bf16=bf16, **pkw,
                     **(sp_kw or {}))
    if pinned is not None:
        for t, ids in enumerate(pinned):
            if ids is not None and len(ids):
                sp.pin_rows(t, ids)
    pol = Policy(rows, slots, P, F, allow_padding=padding, pinned=pinned, **pkw) \
        if (check_plans or check_slots) else None
    orc = UncachedTrainer(rows, D, N, L, init_seed, allow_padding=padding, bf16=bf16)
    report = {"plans": 0, "evictions": 0, "pooled": 0}

    def on_plan(b, newest=True):
        if pol is None:
            return
        recs = pol.plan(trace_np, b)
        for t in range(len(rows)):
            r = recs[t]
            report["evictions"] += r.evictions
            if check_plans:
                gp = sp.debug_plan(b, t)
                assert (gp["U"], gp["hits"], gp["misses"], gp["evictions"]) == \
                    (r.U, r.hits, r.misses, r.evictions), (b, t)
                assert np.array_equal(gp["uniq"], r.uniq), (b, t)
                assert np.array_equal(gp["hit"], r.hit), (b, t)
                assert np.array_equal(gp["slot"], r.slot), (b, t)
                assert np.array_equal(gp["evicted"], r.evicted), (b, t)
            if check_slots and newest:
                res, lu = sp.debug_slots(t)
                ores, olu = pol.slot_state(t)
                assert np.array_equal(res, ores), (b, t)
                assert np.array_equal(lu, olu), (b, t)
        report["plans"] += 1

    def on_pooled(b, pooled):
        want = orc.step(trace_np[b], g, d, e, want_pooled=check_pooled)
        if check_pooled:
            got = pooled.cpu().numpy()
            assert np.array_equal(got, want), (b, float(np.max(np.abs(got - want))))
            report["pooled"] += 1

    run_loop(sp, feed, g, d, e, on_plan=on_plan, on_pooled=on_pooled, push=push)
    # final host tables after sp_flush vs the oracle's uncached training
    worst = {"max_rel": 0.0, "mismatch": 0, "rel_to_update": 0.0, "rows": 0}
    for t, R in enumerate(rows):
        touched = orc.touched(t)
        if sample_rows is not None and len(touched) > sample_rows:
            touched = np.sort(np.random.default_rng(t).choice(touched, sample_rows, replace=False))
        if len(touched):
            want = orc.rows_of(t, touched)
            got = views[t][torch.from_numpy(touched)].numpy()
            c = compare_tables(got, want, init_rows_np(init_seed, t, touched, D))
            worst["max_rel"] = max(worst["max_rel"], c["max_rel"])
            worst["mismatch"] += c["mismatch"]
            worst["rel_to_update"] = max(worst["rel_to_update"], c["rel_to_update"])
            worst["rows"] += len(touched)
        # untouched rows keep their initial values
        untouched = np.setdiff1d(np.arange(min(R, 512)), orc.touched(t))
        if len(untouched):
            assert np.array_equal(views[t][torch.from_numpy(untouched)].numpy(),
                                  init_rows_np(init_seed, t, untouched, D))
    report["tables"] = worst
    report["stats"] = sp.stats()
    sp.close()
    return report
