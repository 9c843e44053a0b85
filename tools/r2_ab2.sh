#!/bin/bash
# A/B of compile-time knobs + env + bench args, span summary per run:
#   r2_ab2.sh TAG STEPS "label|-DFLAGS|ENV=.. ENV=..|bench args" ...
TAG=$1; STEPS=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
for spec in "$@"; do
  IFS='|' read -r label flags envs args <<< "$spec"
  SP_NVCC_EXTRA="$flags" python -c "
import importlib.util
s = importlib.util.spec_from_file_location('b', 'paper_2205_04702_b200/build.py'); m = importlib.util.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)" >> $O/build.log 2>&1
  env $envs timeout 600 python bench.py --steps $STEPS --warmup 20 --no-cpu-baseline $args > $O/$label.json 2> $O/$label.err
  echo "== $label: flags[$flags] env[$envs] args[$args] $(python tools/bench_brief.py $O/$label.json | cut -c40-)" >> $O/sweep.log
  python - "$O/$label.json" >> $O/sweep.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    sp = d.get("spans") or {}
    print("   spans", sp.get("duration_us"), "busy", sp.get("stream_busy_us_per_step"), "step", sp.get("step_us"),
          "| eng", {k: v for k, v in d["host_engine"].items() if k != "threads"})
except Exception as e:
    print("   parse error", e)
PY
done
SP_NVCC_EXTRA="" python -c "
import importlib.util
s = importlib.util.spec_from_file_location('b', 'paper_2205_04702_b200/build.py'); m = importlib.util.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)" >> $O/build.log 2>&1
cat $O/sweep.log
