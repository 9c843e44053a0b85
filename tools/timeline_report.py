"""Summarise a bench timeline dump (SP_TIMELINE=...): per-kernel in-situ
durations, per-stream busy fraction, and the step-critical chain."""
import json
import sys
from collections import defaultdict

tl = json.load(open(sys.argv[1]))
tl.sort(key=lambda r: r[2])
t0, t1 = tl[0][2], max(r[3] for r in tl)
span = t1 - t0
by = defaultdict(list)
for k, b, s, e in tl:
    by[k].append((b, s, e))
print(f"span {span*1e3:.0f} us, batches {len(by['backward'])}, step {span*1e3/len(by['backward']):.1f} us")
for k, v in by.items():
    d = sorted((e - s) * 1e3 for _, s, e in v)
    busy = sum((e - s) for _, s, e in v) / span
    print(f"{k:10s} n={len(v):4d} median={d[len(d)//2]:6.1f}us p90={d[int(len(d)*.9)]:6.1f}us  busy={busy:5.2f}")
# per batch: forward start - transfer end (waiting), train end -> next forward start gap
fw = {b: (s, e) for b, s, e in by['forward']}
bw = {b: (s, e) for b, s, e in by['backward']}
xf = {b: (s, e) for b, s, e in by['transfer']}
su = {b: (s, e) for b, s, e in by['surrogate']}
gaps = defaultdict(list)
for b in sorted(fw):
    if b - 1 in bw:
        gaps['bwd(b-1).end->fwd(b).start'].append((fw[b][0] - bw[b - 1][1]) * 1e3)
    if b in xf:
        gaps['xfer(b).end->fwd(b).start'].append((fw[b][0] - xf[b][1]) * 1e3)
    if b in su:
        gaps['fwd.end->surr.start'].append((su[b][0] - fw[b][1]) * 1e3)
    if b in su and b in bw:
        gaps['surr.end->bwd.start'].append((bw[b][0] - su[b][1]) * 1e3)
for k, v in gaps.items():
    v.sort()
    print(f"{k:28s} median={v[len(v)//2]:6.1f}us p10={v[len(v)//10]:6.1f} p90={v[int(len(v)*.9)]:6.1f}")
