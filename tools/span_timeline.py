"""Per-batch timeline of the steady state from a bench line's in-kernel span
stamps (spans.raw_ms: [plan, transfer, forward, surrogate, backward][slot]
[start, end] ms).  Slot r holds the last launch for a batch = r (mod 16);
Plan / Transfer slots may already hold batch + 16, recognised by starting
after that slot's forward.  Prints, per trained batch in order, each stage's
start / end (us, relative to the first forward) and the gaps that bound the
step.   python tools/span_timeline.py bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
raw = d["spans"]["raw_ms"]
names = ["plan", "xfer", "fwd", "surr", "bwd"]
slots = [r for r in range(16) if raw[2][r][0] is not None and raw[4][r][1] is not None]
slots.sort(key=lambda r: raw[2][r][0])
t0 = raw[2][slots[0]][0]
print("%4s " % "slot" + " ".join("%17s" % n for n in names) + "   xfer.end->fwd  bwd(prev).end->fwd")
prev_bwd = None
for r in slots:
    row = []
    for k in range(5):
        a, b = raw[k][r]
        if a is None:
            row.append("%17s" % "-")
            continue
        if k < 2 and a > raw[2][r][0]:  # already the launch for batch + 16
            row.append("%17s" % "(next)")
            continue
        row.append("%8.1f-%8.1f" % ((a - t0) * 1e3, (b - t0) * 1e3))
    xa, xb = raw[1][r]
    slack = (raw[2][r][0] - xb) * 1e3 if xb is not None and xa is not None and xa < raw[2][r][0] else float("nan")
    gap = (raw[2][r][0] - prev_bwd) * 1e3 if prev_bwd is not None else float("nan")
    print("%4d " % r + " ".join(row) + "   %8.1f       %8.1f" % (slack, gap))
    prev_bwd = raw[4][r][1]
