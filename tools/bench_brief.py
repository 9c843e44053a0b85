"""One line per bench JSON: value, e2e, step, per-stage us (timed pass / profiling pass), roofline."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        k = d["kernels"]
        st = " ".join("%s %.1f/%.1f" % (x[:4], k[x]["avg_us"], k[x]["profiling_pass_us"]) for x in k)
        print("%-40s %8.0f e2e %8.0f step %6.1f | %s | roof %s %.3f" % (
            p, d["value"], d["e2e"]["value"], d["ms_per_step"] * 1e3, st, d["roofline"]["kernel"],
            d["roofline"]["frac"]))
    except Exception as e:
        print(p, "parse error", e)
