#!/usr/bin/env python
"""bench.py — the ScratchPipe hot path on B200 (BASELINE.json metric).

One "step" = one pass of the whole hot path over one synthetic mini-batch:
sp_plan (index ingest + dedup + Hit-Map probe + hit/miss + window-safe victim
selection + bookkeeping), the Collect/Exchange/Insert transfer (CPU threads
gather the missed rows into pinned memory, one kernel moves them into the
freed slots and stages the victims in pinned memory, CPU threads scatter the
victims into their host rows),
sp_forward (EmbeddingBag gather-reduce), the MLP stand-in
(surrogate gradient kernel) and sp_train (coalescing segmented reduce + fused
SGD).  Workload at N=1: BASELINE configs[2], Criteo-Terabyte-shaped (the
shape north_star names for the 1- and 8-GPU headline; it fits one B200), in
steady state: `preroll` untimed batches first fill the scratchpad (cold start
is not the paper's regime), then W warm-up steps, then K timed steps.  The
other BASELINE configs are parity-test cases and extra runs (--config kaggle |
highpool | tiny).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config terabyte]

Prints ONE JSON line on rank 0.  `value` times device-resident int32 indices
(inputs in HBM); `e2e` times the same steps one library call per step with
the indices in pinned host memory (their H2D inside the timed region) plus a
D2H read of every step's Plan counters that the host waits for.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "embedding training iters/s at 1/2/4/8 B200; Train-stage HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="terabyte")
    ap.add_argument("--policy", default="lru", choices=["lru", "random", "lfu"],
                    help="replacement policy among the window-safe candidates (P:1270-1278)")
    ap.add_argument("--policy-seed", type=int, default=2205)
    ap.add_argument("--dim", type=int, default=0, help="sensitivity sweep: override D (P:1248-1258)")
    ap.add_argument("--pooling", type=int, default=0, help="sensitivity sweep: override L (P:1259-1268)")
    ap.add_argument("--batch", type=int, default=0, help="sensitivity sweep: override N")
    ap.add_argument("--slot-frac", type=float, default=0.0, help="sensitivity sweep: slots as a fraction of rows")
    ap.add_argument("--gather-frac", type=float, default=-1.0,
                    help="share of each batch's missed rows gathered by CPU threads (hybrid transfer); "
                         "-1: the library's default")
    ap.add_argument("--host-threads", type=int, default=0, help="transfer-engine helper threads per pool")
    ap.add_argument("--writeback", default="", choices=["", "gpu", "cpu"],
                    help="victims' write-back: GPU bulk stores into host rows, or CPU scatter (default: library's)")
    ap.add_argument("--variant", default="pipelined", choices=["pipelined", "serial", "resident", "gpuonly", "static"],
                    help="design points of PAPER.md Fig. 10 / Table 1 from the same kernels: "
                         "pipelined (ScratchPipe), serial (straw-man: every stage on one stream, "
                         "no overlap), resident (slots = rows, cold start), gpuonly (slots = rows "
                         "and every row loaded before the first batch: no misses at all), static (the "
                         "paper's static top-N cache from the same kernels: the hottest rows of a profiling "
                         "prefix pinned in the slot budget, a window-sized scratchpad for the rest)")
    ap.add_argument("--storage", default="f32", choices=["f32", "bf16"],
                    help="Storage row format (SURVEY 8(f) f4): f32 (the paper's), or bf16 (SP_FLAG_BF16, "
                         "reading R28: rows rounded to bf16 in HBM, host tables, pooled and gradients fp32)")
    ap.add_argument("--preroll", type=int, default=-1, help="untimed steady-state fill batches (-1: config)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=200)
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + clock-event reasons during a timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.0005):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # warm the query path: the first calls can take tens of ms, longer
            # than a whole timed region at ~50 us/step
            for _ in range(3):
                pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": [n for bit, n in self.REASONS.items() if self.reasons & bit]}


# --------------------------------------------------------------------------- helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def host_cpu_info():
    """nproc and the lscpu model name of this box (cpu_baseline context)."""
    info = {"nproc": os.cpu_count()}
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "NUMA node(s)", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception as e:  # pragma: no cover
        info["lscpu"] = f"unavailable: {e}"
    return info


def host_mem_available():
    """MemAvailable of this node in bytes (None if unknown)."""
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return None


def link_peaks(dev, mib=256, reps=5):
    """Host-link peaks measured in this run: pinned cudaMemcpyAsync of `mib`
    MiB, best of `reps`, H2D, D2H and both directions at once (two streams),
    CUDA events.  The roofline denominators of the transfer stage."""
    import torch
    n = mib << 18  # float32 elements
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h2 = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def once(kind):
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        with torch.cuda.stream(s1):
            if kind in ("h2d", "bidir"):
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
        if kind == "bidir":
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            s1.wait_stream(s2)
        b.record(s1)
        b.synchronize()
        return a.elapsed_time(b) * 1e-3

    out = {}
    for kind in ("h2d", "d2h", "bidir"):
        once(kind)
        t = min(once(kind) for _ in range(reps))
        out[kind + "_GBs"] = round((2 if kind == "bidir" else 1) * n * 4 / t / 1e9, 2)
    out["how"] = f"pinned cudaMemcpyAsync of {mib} MiB, best of {reps}, CUDA events (bidir: both directions on two streams, bytes summed)"
    del h, h2, d, d2
    return out


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle (plain CPU program, as it stands) on this box's host cores:
    each step = one oracle iteration (reference policy Plan + uncached
    EmbeddingBag SGD) over one batch of the same workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import torch
    from oracle import Policy, UncachedTrainer
    from workload import CONFIGS, sample_trace
    cfg = CONFIGS[args.config]
    g, d, e = cfg.surrogate()
    nb = args.warmup + args.steps
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    tr = sample_trace(cfg.rows, cfg.batch, cfg.pooling, cfg.alpha, nb, cfg.trace_seed,
                      device=dev, dtype=torch.int64).cpu().numpy()
    pol = Policy(cfg.rows, cfg.slots, cfg.window, max(cfg.window - 1, 0))
    orc = UncachedTrainer(cfg.rows, cfg.dim, cfg.batch, cfg.pooling, cfg.init_seed)

    def step(b):
        pol.plan(tr, b)
        orc.step(tr[b], g, d, e)

    for b in range(args.warmup):
        step(b)
    t0 = time.perf_counter()
    for b in range(args.warmup, nb):
        step(b)
    el = time.perf_counter() - t0
    v = args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg.description, "note": "oracle from a cold scratchpad"},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle", "host": host_cpu_info(),
                             "sample": f"{args.steps} consecutive batches after {args.warmup} warm-up, "
                                       "reference policy + uncached EmbeddingBag SGD, single thread"},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def cpu_baseline(cfg, trace_dev, seconds):
    """Oracle on a bounded sample of the same trace (cold start), 1 thread."""
    import torch
    from oracle import Policy, UncachedTrainer
    g, d, e = cfg.surrogate()
    pol = Policy(cfg.rows, cfg.slots, cfg.window, max(cfg.window - 1, 0))
    orc = UncachedTrainer(cfg.rows, cfg.dim, cfg.batch, cfg.pooling, cfg.init_seed)
    chunk = 1024
    tr = trace_dev[:chunk].to(torch.int64).cpu().numpy()
    n = 0
    t0 = time.perf_counter()
    while True:
        if n >= tr.shape[0]:
            break
        pol.plan(tr, n)
        orc.step(tr[n], g, d, e)
        n += 1
        if time.perf_counter() - t0 > seconds and n >= 3:
            break
    el = time.perf_counter() - t0
    return {"value": n / el, "unit": "iters/s", "cores": 1, "kind": "oracle", "host": host_cpu_info(),
            "sample": f"first {n} batches of the bench trace from a cold scratchpad: reference policy "
                      f"(Part B) + uncached EmbeddingBag SGD (Part A), single thread, {el:.1f} s"}


def _union_us(iv):
    """Total length (us) of the union of [a, b] intervals given in ms."""
    iv = sorted((a, b) for a, b in iv if a == a and b == b and b >= a)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        tot += cur[1] - cur[0]
    return tot * 1e3


def _stream_busy(ev):
    """Per-step busy time of each stream over the stage-event window of the
    last 16 steps (sp_stage_events): union of that stream's intervals / steps."""
    import numpy as np
    rows = [r for r in range(ev.shape[0]) if not np.isnan(ev[r, 0])]
    nst = max(1, len(rows))
    plan = [(ev[r, 0], ev[r, 1]) for r in rows]
    comp = [(ev[r, 2], ev[r, 5]) for r in rows]
    xfer = [(ev[r, 6], ev[r, 7]) for r in range(ev.shape[0]) if not np.isnan(ev[r, 6])]
    lo = np.nanmin(ev[rows][:, [0, 2]]) if rows else 0.0
    hi = np.nanmax(ev[rows][:, [1, 5]]) if rows else 0.0
    # the step period of THIS pass (event nodes in the graphs slow it down a
    # little against the timed region): spacing of consecutive Train ends
    ends = sorted(ev[r, 5] for r in rows)
    step = (ends[-1] - ends[0]) * 1e3 / (len(ends) - 1) if len(ends) > 1 else float("nan")
    return {"plan": _union_us(plan) / nst, "compute": _union_us(comp) / nst,
            "transfer": _union_us(xfer) / max(1, len(xfer)),
            "window_us_per_step": (hi - lo) * 1e3 / nst, "step_us": step, "steps": nst}


def _overlap(kernels, step_us, busy=None):
    """Stage overlap in the steady state.  busy: per-step busy
    time of each stream = the union of its event intervals over the last 16
    steps / 16 (so two transfers in flight on the two alternating transfer
    streams count once), all measured in the stage-timing pass; its own step
    period is the comparison (the timed region's step is reported beside it).
    Full overlap: step <= 1.05 x the busiest stream.  Busy spans include
    waiting for SM resources beside the other stages, so they can only
    overstate a stage; each is <= the pass's step by construction."""
    if busy is None:
        return None
    streams = {k: busy[k] for k in ("plan", "transfer", "compute")}
    tot, mx = sum(streams.values()), max(streams.values())
    bound = max(streams, key=streams.get)
    pstep = busy["step_us"] if busy["step_us"] == busy["step_us"] else step_us
    return {"step_us": round(step_us, 2), "timing_pass_step_us": round(pstep, 2),
            "stream_busy_us_per_step": {k: round(v, 2) for k, v in streams.items()},
            "event_window_us_per_step": round(busy["window_us_per_step"], 2),
            "serial_sum_us": round(tot, 2), "busiest_stream": bound,
            "busiest_over_step": round(mx / pstep, 3) if pstep else None,
            "step_over_busiest": round(pstep / mx, 3) if mx else None,
            "full_overlap": bool(mx and pstep <= 1.05 * mx),
            "transfer_hidden_behind_compute": bool(streams["transfer"] <= 1.05 * streams["compute"]),
            "source": "sp_stage_events: CUDA events on each stage's own stream inside the step graphs, "
                      "union of intervals per stream over the last %d steps" % busy["steps"]}


def _span_summary(sp_ms):
    """In-kernel span stamps of the last 16 steps (sp_span_times: [kind][slot]
    [start, end] ms): per stage the median in-situ duration (first CTA start to
    last CTA end), per stream the busy time per step (union of its intervals /
    steps), and the step period from consecutive backward ends."""
    import numpy as np
    kinds = ["plan", "transfer", "forward", "surrogate", "backward"]
    iv = {k: [(a, b) for a, b in sp_ms[i] if a == a and b == b] for i, k in enumerate(kinds)}
    dur = {k: float(np.median([(b - a) * 1e3 for a, b in v])) if v else None for k, v in iv.items()}
    ends = sorted(b for _, b in iv["backward"])
    step = (ends[-1] - ends[0]) * 1e3 / (len(ends) - 1) if len(ends) > 1 else float("nan")
    nst = max(1, len(iv["backward"]))
    busy = {"plan": _union_us(iv["plan"]) / max(1, len(iv["plan"])),
            "transfer": _union_us(iv["transfer"]) / max(1, len(iv["transfer"])),
            "compute": _union_us(iv["forward"] + iv["surrogate"] + iv["backward"]) / nst}
    return {"raw_ms": [[[round(x, 4) if x == x else None for x in ab] for ab in sp_ms[i]] for i in range(5)],
            "duration_us": {k: (round(v, 2) if v is not None else None) for k, v in dur.items()},
            "stream_busy_us_per_step": {k: round(v, 2) for k, v in busy.items()},
            "step_us": round(step, 2), "steps": nst,
            "source": "%globaltimer stamps of every CTA of the five stage kernels in the graph-mode "
                      "steady state (sp_set_span_timing; no events in the graphs), last 16 steps"}


def _plan_roles(p0, p1):
    """k_push critical chain: mean per-launch wall time of each table's Plan
    CTA and dedup CTA over the profiling window (globaltimer, in-kernel)."""
    out = {}
    for role, key, li in (("plan", "plan_us", 0), ("dedup", "dedup_us", 1)):
        n0, n1 = p0["launches"][li], p1["launches"][li]
        if n1 <= n0:
            continue
        per = [(b * n1 - a * n0) / (n1 - n0) for a, b in zip(p0[key], p1[key])]
        tm = int(max(range(len(per)), key=lambda i: per[i]))
        pk = role + "_phase_us"
        phases = [round((b * n1 - a * n0) / (n1 - n0), 2) for a, b in zip(p0[pk][tm], p1[pk][tm])]
        out[role] = {"max_table_us": round(max(per), 2), "mean_us": round(sum(per) / len(per), 2),
                     "argmax_table": tm, "phases_us_of_argmax": phases[:6 if role == "plan" else 5]}
    pl = p1.get("per_launch", {})
    if pl.get("span_us"):
        import numpy as np
        q = lambda v: [round(float(np.percentile(v, x)), 2) for x in (50, 90, 99)]
        out["per_launch_p50_p90_p99_us"] = {"kernel_span": q(pl["span_us"]), "slowest_plan_cta": q(pl["plan_cta_max_us"]),
                                            "slowest_dedup_cta": q(pl["dedup_cta_max_us"]),
                                            "launches": len(pl["span_us"])}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2205_04702_b200 import ScratchPipe
    from paper_2205_04702_b200.sharding import (lpt_assign,
                                                table_weights, tables_of)
    from workload import CONFIGS, init_table, sample_trace

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    over = {k: v for k, v in (("dim", args.dim), ("pooling", args.pooling), ("batch", args.batch)) if v}
    if args.slot_frac:
        over.update(slot_frac=args.slot_frac, slots_fixed=None)
    if over:
        cfg = cfg.with_(**over)
    if args.writeback:
        os.environ["SP_WRITEBACK"] = args.writeback
    if args.gather_frac >= 0:
        os.environ["SP_GATHER_FRAC"] = str(args.gather_frac)
    if args.variant in ("resident", "gpuonly"):
        cfg = cfg.with_(slot_frac=1.0, slots_fixed=None)
    if args.variant == "serial":
        os.environ["SP_DIAG_SERIAL"] = "1"
    T, D, N, L = cfg.num_tables, cfg.dim, cfg.batch, cfg.pooling
    slots_all = cfg.slots
    owner = lpt_assign(table_weights(cfg.rows, slots_all, N * L, D), world)
    mine = tables_of(owner, rank)
    shard_kw = {}
    if world > 1:  # table-wise sharding inside the library: NCCL comm from a shared unique id
        from paper_2205_04702_b200 import nccl_unique_id
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        shard_kw = dict(world=world, rank=rank, nccl_id=box[0], table_owner=owner, table_ids=mine)
    rows = [cfg.rows[t] for t in mine]
    slots = [slots_all[t] for t in mine]
    g_, d_, e_ = cfg.surrogate()
    W, K = max(3, args.warmup), args.steps
    KP = min(K, args.profile_steps)
    pre = cfg.preroll if args.preroll < 0 else args.preroll
    P, F = cfg.window, max(cfg.window - 1, 0)
    ahead = P + F + 1
    KS = 48 if world == 1 else 0       # graph-mode stage-timing pass (16 recaptures + 32 timed), and again for spans
    nb_dev = pre + W + K + 2 * KS + KP  # device-index phase (incl. the `ahead` pushed first)
    WE = max(W, 18)                    # e2e warm-up: also (re)captures the 16 step graphs
    nb_host = WE + K                   # host-index (e2e) phase
    nb = nb_dev + ahead + nb_host

    # ---- inputs: host tables (pinned), trace (device int32; host int32 part pinned)
    from paper_2205_04702_b200 import HostTable
    need = sum(cfg.rows[t] for t in mine) * D * 4
    avail = host_mem_available()
    if avail is not None and need > 0.9 * avail:
        raise SystemExit(f"host RAM: this rank's tables need {need / 1e9:.1f} GB of pinned memory, the node has "
                         f"{avail / 1e9:.1f} GB available (MemAvailable): run {args.config} on more GPUs or a larger node")
    tables = []   # THP-backed, CUDA-registered host tables (sp_host_alloc)
    for t in mine:
        h = HostTable(cfg.rows[t], D, device=local)  # NUMA-local to this rank's GPU
        init_table(cfg.init_seed, t, cfg.rows[t], D, device=dev, out=h.tensor)
        tables.append(h)
    trace = torch.empty((nb, len(mine), N, L), dtype=torch.int32, device=dev)
    CH = 512
    for b0 in range(0, nb, CH):
        b1 = min(nb, b0 + CH)
        full = sample_trace(cfg.rows, N, L, cfg.alpha, b1 - b0, cfg.trace_seed, first_batch=b0,
                            device=dev, dtype=torch.int32)
        trace[b0:b1] = full[:, mine]
        del full
    host_trace = trace[nb_dev + ahead:].cpu().pin_memory()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)
    sp = ScratchPipe(rows, tables, D, slots, N, L, window=cfg.window, device=local, stream=stream,
                     index_dtype="int32", index_on_device=False, policy=args.policy,
                     host_threads=args.host_threads,
                     policy_seed=args.policy_seed, bf16=args.storage == "bf16", **shard_kw)
    pinned_rows = 0
    if args.variant == "static":
        # static top-N partition: the hottest rows of the first 200 batches of
        # the trace fill the slot budget except a window-sized scratchpad
        # (2w*N*L slots: the minimum the look-forward window needs)
        prof = trace[:min(200, nb)]
        for k, t in enumerate(mine):
            pool = min(slots[k], 2 * cfg.window * N * L)
            ids, cnt = torch.unique(prof[:, k].reshape(-1), return_counts=True)
            top = ids[torch.argsort(cnt, descending=True, stable=True)[:slots[k] - pool]]
            sp.pin_rows(k, top.cpu().numpy())
            pinned_rows += int(top.numel())
    if args.variant == "gpuonly":
        sp.prefill()
    pooled = torch.empty(sp.pooled_shape(), dtype=torch.float32, device=dev)  # [T_all][N/G][D] if sharded
    grad = torch.empty_like(pooled)
    stats_host = torch.zeros((K + max(W, 18) + 8, len(mine), 4), dtype=torch.int32).pin_memory()
    state = {"pushed": 0, "trained": 0}

    def push_dev():
        j = state["pushed"]
        sp.plan_device(trace[j])
        state["pushed"] = j + 1

    def push_host():
        j = state["pushed"]
        sp.plan(host_trace[j - nb_dev - ahead])
        state["pushed"] = j + 1

    def train_step(push, read_stats_slot=None):
        push()
        sp.forward(pooled)          # sharded: NCCL exchange inside the library
        sp.surrogate(pooled, g_, d_, out=grad)
        sp.train(grad, e_)
        if read_stats_slot is not None:
            sp.copy_batch_stats(state["trained"], stats_host[read_stats_slot])
        state["trained"] += 1

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, n, sampler_index=None):
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(sampler_index) if sampler_index is not None else None
        if sampler:
            sampler.__enter__()
        s.record(stream)
        for k in range(n):
            fn(k)
        e.record(stream)
        barrier()
        if sampler:
            sampler.__exit__()
        ms = torch.tensor([s.elapsed_time(e)], device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item()), sampler

    # ---- preroll + warm-up + timed value loop: device-resident indices, the
    # library's C driver loop (sp_run_steps: plan / forward / surrogate / train)
    dev_trace = trace[:nb_dev + ahead]
    t_pre = time.perf_counter()
    sp.run_steps(dev_trace, pre + W, pooled, grad, g_, d_, e_)  # sharded: eager steps, NCCL in the library
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t_pre
    st0 = sp.stats()

    def value_loop(n):
        sp.run_steps(dev_trace, n, pooled, grad, g_, d_, e_)

    # ---- timed: value (inputs resident in HBM)
    barrier()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    sampler.__enter__()
    t_host = time.perf_counter()
    s_ev.record(stream)
    value_loop(K)
    e_ev.record(stream)
    t_host_issue = time.perf_counter() - t_host
    barrier()
    sampler.__exit__()
    ms_t = torch.tensor([s_ev.elapsed_time(e_ev)], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    st1 = sp.stats()
    stage_t = stage_busy = spans = None
    if world == 1:  # same graph-mode steady state, step graphs recaptured with event nodes
        evspan = os.environ.get("SP_BENCH_EVSPAN") == "1"  # diagnostic: spans stamped in the event pass too
        sp.set_stage_timing(True)
        if evspan:
            sp.set_span_timing(True)
        value_loop(KS)
        stage_t = sp.stage_times()   # events of the last 16 steps, on each stage's own stream
        stage_busy = _stream_busy(sp.stage_events())
        if evspan:
            print("evspan events", {k: round(v["ms"] * 1e3, 2) for k, v in stage_t.items()},
                  "spans", _span_summary(sp.span_times())["duration_us"], file=sys.stderr)
            sp.set_span_timing(False)
        sp.set_stage_timing(False)
        sp.set_span_timing(True)    # the same steady state, kernels stamping their own spans
        value_loop(KS)
        spans = _span_summary(sp.span_times())
        sp.set_span_timing(False)
    st1p = sp.stats()  # baseline of the (eager) profiling pass
    value = K / (ms / 1e3)   # iterations of the global batch per second (max over ranks)
    ms_per_step = ms / K
    from paper_2205_04702_b200._binding import KERNEL_ONLY
    launches = {k: st1["kernel_launches"][k] - st0["kernel_launches"][k] for k in st1["kernel_launches"]}
    gpu_launches = sum(v for k, v in launches.items() if k in KERNEL_ONLY)
    # a backward launch is two kernels with the two-phase backward (k_bwd_tile + k_bwd_rows)
    gpu_launches += launches.get("backward", 0) * (int(st1.get("backward_kernels", 1) or 1) - 1)
    # ---- profiling pass: per-kernel CUDA-event durations (separate from the timed region)
    sp.set_profiling(True)
    pp0 = sp.debug_plan_profile()
    value_loop(KP)
    sp.set_profiling(False)
    pp1 = sp.debug_plan_profile()
    st2 = sp.stats()
    if os.environ.get("SP_TIMELINE"):
        json.dump(sp.timeline(), open(os.environ["SP_TIMELINE"], "w"))
    state["pushed"] = nb_dev + ahead
    state["trained"] = nb_dev
    # ---- e2e: host indices (pinned) through the public API, and a D2H of every
    # step's result (its Plan counters) that the host waits for and reads one
    # step later (lag 1 keeps the pipeline full)
    evs = [torch.cuda.Event() for _ in range(2)]
    hits_seen = []
    h0 = nb_dev + ahead  # host_trace[i] is batch h0 + i

    def e2e_one(slot):
        # the library's step call: the plan kernel reads B(j) over the host link
        sp.run_steps(host_trace, 1, pooled, grad, g_, d_, e_, first_batch=h0)
        state["pushed"] += 1
        sp.copy_batch_stats(state["trained"], stats_host[slot])
        state["trained"] += 1
        evs[slot % 2].record(stream)

    for k in range(WE):
        e2e_one(k)
    torch.cuda.synchronize()

    e2e_host_t = []

    def e2e_step(k):
        e2e_one(WE + k)
        if k >= 1:
            evs[(WE + k - 1) % 2].synchronize()
            hits_seen.append(int(stats_host[WE + k - 1, :, 1].sum()))
        e2e_host_t.append(time.perf_counter())
    ms_e2e, _ = timed(e2e_step, K)
    e2e_gaps = [1e6 * (b - a) for a, b in zip(e2e_host_t, e2e_host_t[1:])]
    hits_seen.append(int(stats_host[WE + K - 1, :, 1].sum()))
    e2e_value = K / (ms_e2e / 1e3)
    st3 = sp.stats()
    idx_bytes = len(mine) * N * L * 4
    stats_bytes = len(mine) * 4 * 4

    # ---- per-kernel accounting (profiling window)
    def delta(key):
        return st2[key] - st1p[key]
    steps_p = KP
    U = delta("uniques") / steps_p
    m = delta("misses") / steps_p
    ev = delta("evictions") / steps_p
    Tg = len(mine)
    n = N * L
    kms = {k: st2["kernel_ms"][k] - st1p["kernel_ms"][k] for k in st2["kernel_ms"]}
    kcount = {k: st2["kernel_timed"][k] - st1p["kernel_timed"][k] for k in st2["kernel_timed"]}
    avg_ms = {k: (kms[k] / kcount[k] if kcount[k] else 0.0) for k in kms}
    es = 2 if args.storage == "bf16" else 4  # bytes per Storage element
    alg_bytes = {
        # slot map + gathered rows + pooled out (nominal TBE bytes)
        "forward": 4 * Tg * n + es * D * Tg * n + 4 * D * Tg * N,
        # pooled grad in + occurrence list + per-unique segment/slot words + SGD read+write
        "backward": 4 * D * Tg * N + 4 * Tg * n + 16 * U + 2 * es * D * U,
        "surrogate": 8 * D * Tg * N,
        # k_pullfill, host-link bytes: missed rows pulled (H2D) + victims written
        # to the pinned staging slot (D2H); HBM: the same rows written / read
        "transfer": 4 * D * m + 4 * D * ev,
        "plan": 4 * Tg * n,
    }
    peak, peak_kind = peaks()
    traffic = load_traffic()
    total_ms = sum(kms.values()) or 1.0
    kernels = {}
    # per-stage duration: CUDA events on each stage's own stream inside the
    # step graphs of the TIMED region (last 16 steps), else the profiling pass
    timed_src = bool(stage_t) and all(stage_t[k]["n"] > 0 for k in ["forward", "backward", "surrogate"])
    for k in ["plan", "transfer", "forward", "backward", "surrogate"]:
        us = stage_t[k]["ms"] * 1e3 if timed_src and stage_t[k]["n"] else avg_ms[k] * 1e3
        gbs = alg_bytes[k] / (us * 1e-6) / 1e9 if us else None
        kernels[k] = {"avg_us": round(us, 3),
                      "span_us": spans["duration_us"][k] if spans else None,
                      "share_profiling_pass": round(kms[k] / total_ms, 4),
                      "profiling_pass_us": round(avg_ms[k] * 1e3, 3),
                      "alg_bytes_per_launch": int(alg_bytes[k]), "alg_GBs": None if gbs is None else round(gbs, 1)}
    # dominant HBM-bound kernel (the Train stage: forward or backward)
    dom = max(["forward", "backward"], key=lambda k: kernels[k]["avg_us"])
    ach = kernels[dom]["alg_GBs"] or 0.0
    # ncu DRAM traffic applies to the configuration it was captured on
    tkey = args.config if args.storage == "f32" else f"{args.config}:{args.storage}"
    tr_bytes = traffic.get(tkey, {}).get(dom)  # per config (captured on that workload)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "duration_source": ("CUDA events around the kernel on its stream inside the step graphs "
                                    "of a graph-mode pass right after the timed region (mean of 16 steps; that "
                                    "pass launches without programmatic dependent launch so each event pair "
                                    "brackets one kernel)")
                                   if timed_src else
                                   "CUDA events around each launch in a separate profiling pass",
                "traffic": tr_bytes,
                "bytes_per_launch": int(alg_bytes[dom]),
                "bytes_formula": (("4*T*n + %d*D*T*n + 4*D*T*N" % es) if dom == "forward"
                                  else ("4*D*T*N + 4*T*n + 16*U + %d*D*U" % (2 * es)))}
    if spans and spans["duration_us"].get(dom):
        # cross-check: the same bytes over the kernel's own first-CTA-start to
        # last-CTA-end span in the same steady state
        sa = alg_bytes[dom] / (spans["duration_us"][dom] * 1e-6) / 1e9
        roofline["span_achieved"] = round(sa, 1)
        roofline["span_frac"] = round(sa / peak, 4)
    train_ms = (kernels["forward"]["avg_us"] + kernels["backward"]["avg_us"]) * 1e-3
    train_bytes = alg_bytes["forward"] + alg_bytes["backward"]
    # host link: the transfer stream's busy time per step (union of its event
    # intervals: two transfers may be in flight on the alternating streams)
    xs = (stage_busy["transfer"] if stage_busy else kernels["transfer"]["avg_us"]) * 1e-6
    link_GBs = 4 * D * m / xs / 1e9 if xs else None
    wb_GBs = 4 * D * ev / xs / 1e9 if xs else None
    lp = link_peaks(dev)
    mode = st2.get("transfer_mode", "?")
    path = {"gpu_pull": "k_pullfill pulls each missed row from its host row (TMA bulk copy per row, "
                        "zero-copy over the link) into the freed Storage slot and writes the victims "
                        "contiguously to pinned staging; CPU threads scatter them into their host rows",
            "cpu_gather": "CPU threads gather the missed rows into a contiguous pinned slot; k_pullfill "
                          "moves it into the freed slots and writes the victims contiguously to pinned "
                          "staging (TMA bulk copies); CPU threads scatter them into their host rows",
            "cpu_gather_dma": "CPU gather into a pinned slot, copy-engine DMA of the slot, k_pullfill "
                              "fills the slots and stages the victims; CPU scatter",
            "hybrid": "CPU threads gather a share (%.2f) of each batch's missed rows into a contiguous "
                      "pinned slot while k_pullfill pulls the rest from their host rows (TMA bulk "
                      "copies); the victims are staged contiguously and scattered by CPU threads"
                      % st2.get("gather_share", 0.0)}.get(mode, mode)
    if st2.get("gpu_writeback"):
        path += " [write-back: k_pullfill stores each victim straight into its host row]"

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "iters/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.description, "config_key": args.config, "tables": T, "dim": D,
                   "batch": N, "pooling": L, "zipf_alpha": cfg.alpha, "slots_total": sum(slots_all),
                   "window": cfg.window, "preroll_batches": pre, "index_input": "device int32 (value)",
                   "l2": "no flush: inputs larger than L2 (Storage %.2f GB, Hit-Map %.0f MB, host tables "
                         "%.1f GB); every step reads a fresh batch" % (
                             sum(slots_all) * D * es / 1e9, sum(cfg.rows) * 4 / 1e6, sum(cfg.rows) * D * 4 / 1e9),
                   "parallelism": f"table-wise x{world}" if world > 1 else "single GPU",
                   "variant": args.variant, "policy": args.policy, "storage": args.storage,
                   **({"pinned_rows": pinned_rows} if args.variant == "static" else {})},
        "roofline": roofline,
        "train_stage": {"avg_us": round(train_ms * 1e3, 3), "alg_bytes": int(train_bytes),
                        "alg_GBs": round(train_bytes / (train_ms * 1e-3) / 1e9, 1) if train_ms else None},
        "host_link": {"path": path, "transfer_mode": mode, "engine_threads": st2.get("engine_threads"),
                      "gather_share": st2.get("gather_share"), "gpu_writeback": st2.get("gpu_writeback"),
                      "h2d_bytes_per_batch": int(4 * D * m),
                      "h2d_GBs": None if link_GBs is None else round(link_GBs, 2),
                      "d2h_bytes_per_batch": int(4 * D * ev),
                      "d2h_GBs": None if wb_GBs is None else round(wb_GBs, 2),
                      "peak_h2d_GBs": lp["h2d_GBs"], "peak_d2h_GBs": lp["d2h_GBs"], "peak_bidir_GBs": lp["bidir_GBs"],
                      "h2d_frac": None if link_GBs is None else round(link_GBs / lp["h2d_GBs"], 4),
                      "d2h_frac": None if wb_GBs is None else round(wb_GBs / lp["d2h_GBs"], 4),
                      "bidir_frac": None if link_GBs is None else round((link_GBs + wb_GBs) / lp["bidir_GBs"], 4),
                      "peak_source": "measured in this run: " + lp["how"],
                      "busy_source": "transfer-stream busy time per step (union of its event intervals)"
                                     if stage_busy else "transfer kernel span (profiling pass)"},
        # stage overlap in the graph-mode steady state: 1.0 = the step costs
        # only its slowest stream, 0.0 = the stages run back to back
        "overlap": _overlap(kernels, ms_per_step * 1e3, stage_busy) if timed_src else None,
        "spans": spans,
        "kernels": kernels,
        "plan_ctas": _plan_roles(pp0, pp1),
        "host_engine": {"scatter_us_per_batch": round(1e3 * (st2["host_scatter_ms"] - st1p["host_scatter_ms"]) / KP, 2),
                        "gather_us_per_batch": round(1e3 * (st2["host_gather_ms"] - st1p["host_gather_ms"]) / KP, 2),
                        "threads": "1 scatter thread + row-copy helpers"},
        "host_waits_us_per_step": {"list_slot": round(1e3 * (st1["wait_list_ms"] - st0["wait_list_ms"]) / K, 2)},
        "per_step": {"uniques": round(U, 1), "misses": round(m, 1), "evictions": round(ev, 1)},
        "gpu_launches": int(gpu_launches),
        "launches_per_step": {k: v / K for k, v in launches.items()},
        "clocks": sampler.summary(),
        "host_issue_us_per_step": round(1e6 * t_host_issue / K, 2),
        "graph_steps": st1["graph_steps"] - st0["graph_steps"],
        "graph_step_host_us": round(1e3 * (st1["graph_step_host_ms"] - st0["graph_step_host_ms"]) /
                                    max(1, st1["graph_steps"] - st0["graph_steps"]), 2),
        "e2e": {"value": round(e2e_value, 2), "unit": "iters/s", "h2d_bytes_per_step": idx_bytes,
                "d2h_bytes_per_step": stats_bytes, "ms_per_step": round(ms_e2e / K, 5),
                "host_step_us_first5": [round(x, 1) for x in e2e_gaps[:5]],
                "host_step_us_median": round(statistics.median(e2e_gaps), 1) if e2e_gaps else None,
                "path": "sp_run_steps(1 step) on pinned host int32 indices (the plan kernel reads "
                        "the batch over the host link); sp_copy_batch_stats D2H each step, waited "
                        "for and read one step later" + ("; pooled rows and gradients exchanged "
                                                         "with NCCL inside the library" if world > 1 else "")},
        "preroll_s": round(t_pre, 2),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, trace, args.cpu_seconds)
    sp.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
