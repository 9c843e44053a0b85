#!/bin/bash
# Transfer-engine A/B on the TB bench: r2_xsweep.sh TAG STEPS "label|ENV=.. ENV=..|bench args" ...
TAG=$1; STEPS=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
for spec in "$@"; do
  IFS='|' read -r label envs args <<< "$spec"
  env $envs timeout 600 python bench.py --steps $STEPS --warmup 20 --no-cpu-baseline $args > $O/$label.json 2> $O/$label.err
  echo "== $label: env[$envs] args[$args] $(python tools/bench_brief.py $O/$label.json | cut -c40-)" >> $O/sweep.log
  python - "$O/$label.json" >> $O/sweep.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    sp = d.get("spans") or {}
    print("   spans", sp.get("duration_us"), "busy", sp.get("stream_busy_us_per_step"), "step", sp.get("step_us"),
          "| eng", {k: v for k, v in d["host_engine"].items() if k != "threads"},
          "| link h2d %.1f d2h %.1f GB/s" % (d["host_link"]["h2d_GBs"], d["host_link"]["d2h_GBs"]))
except Exception as e:
    print("   parse error", e)
PY
done
cat $O/sweep.log
