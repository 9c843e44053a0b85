"""Summarise one round_measure.sh pass into profiles/:

    python tools/ncu_summary.py gpurun_out/<tag> <round-tag>

  launches.csv (ncu --metrics gpu__time_duration.sum, serialised, cold cache)
      -> per-kernel median / mean / share of the step
  full.ncu-rep (ncu --set full)
      -> per launch: duration, DRAM bytes read/written, occupancy, L2 hit rate
      -> profiles/ncu_traffic.json: DRAM bytes per launch of the Train-stage
         kernels, as bench.py's roofline "traffic" ({"forward": B, "backward": B})
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# kernel name prefix -> bench stage
STAGE = {"k_fwd": "forward", "k_bwd_hot": "backward", "k_bwd": "backward", "k_bwd_tile": "backward", "k_bwd_rows": "backward", "k_push": "plan",
         "k_xfer_warp": "transfer", "k_fwd_pad": "forward",
         "k_pullfill": "transfer", "k_surrogate": "surrogate"}


def stage_of(name: str) -> str:
    base = name.replace("void ", "").split("(")[0].split("<")[0].strip()
    return STAGE.get(base, base)


def kname(name: str) -> str:
    return name.replace("void ", "").split("(")[0].strip()


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                out[kname(d["Kernel Name"])].append(float(d["Metric Value"]) / 1e3)
    return out


def full_raw(path):
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
               "launch__grid_size", "launch__registers_per_thread"]
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base",
                          "--metrics", ",".join(metrics)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        out.append({"kernel": kname(d["Kernel Name"]), "stage": stage_of(d["Kernel Name"]),
                    **{m: float(d[m]) for m in metrics if d.get(m) not in (None, "")}})
    return out


def main():
    src, tag = sys.argv[1], sys.argv[2]
    lines = [f"# {tag}: ncu evidence from {src} (bench.py, steady state)"]
    lp = os.path.join(src, "launches.csv")
    ll = launch_list(lp) if os.path.exists(lp) else {}
    tot = sum(sum(v) for v in ll.values()) or 1.0
    lines.append("# launch list: ncu --metrics gpu__time_duration.sum --clock-control none "
                 "(serialised, cold cache: compare SHARES, not absolute times)")
    for k, v in sorted(ll.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:28s} n={len(v):4d} median={statistics.median(v):7.1f}us "
                     f"mean={statistics.mean(v):7.1f}us share={100 * sum(v) / tot:5.1f}%")
    full = full_raw(os.path.join(src, "full.ncu-rep"))
    lines.append("# ncu --set full, per launch: duration us | DRAM read MB | DRAM write MB | "
                 "achieved GB/s (DRAM) | warps active % | L2 hit % | grid | regs")
    per_stage = collections.defaultdict(list)
    for i, d in enumerate(full):
        us = d["gpu__time_duration.sum"] / 1e3
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        lines.append(f"{i:3d} {d['kernel']:24s} {us:8.2f} {rd / 1e6:9.3f} {wr / 1e6:9.3f} "
                     f"{(rd + wr) / (us * 1e-6) / 1e9:9.1f} {d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):6.1f} "
                     f"{d.get('lts__t_sector_hit_rate.pct', 0):6.1f} {int(d.get('launch__grid_size', 0)):6d} "
                     f"{int(d.get('launch__registers_per_thread', 0)):4d}")
        per_stage[(d["stage"], d["kernel"])].append(rd + wr)
    # per-launch DRAM traffic of each stage = sum over its kernels of the mean per launch
    traffic = collections.defaultdict(float)
    for (st, k), v in per_stage.items():
        traffic[st] += statistics.mean(v)
    traffic = {k: int(v) for k, v in traffic.items()}
    traffic["source"] = f"{src}/full.ncu-rep (dram__bytes_read.sum + dram__bytes_write.sum, mean per launch)"
    cfg = sys.argv[3] if len(sys.argv) > 3 else "terabyte"
    lines.append(f"# DRAM bytes per launch by stage ({cfg}): " + json.dumps(traffic))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.txt"), "w").write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt[cfg] = traffic  # bench.py reads the entry of the config it runs
    json.dump(allt, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
