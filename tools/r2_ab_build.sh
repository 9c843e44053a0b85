#!/bin/bash
# A/B of compile-time kernel knobs: r2_ab_build.sh TAG STEPS "label|-DFLAGS|bench args" ...
TAG=$1; STEPS=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
python -c "import oracle; oracle.build()" > $O/build.log 2>&1
for spec in "$@"; do
  IFS='|' read -r label flags args <<< "$spec"
  SP_NVCC_EXTRA="$flags" python -c "
import importlib.util
s = importlib.util.spec_from_file_location('b', 'paper_2205_04702_b200/build.py'); m = importlib.util.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)" >> $O/build.log 2>&1
  echo "== $label: flags[$flags] args[$args]" >> $O/sweep.log
  timeout 900 python bench.py --steps $STEPS --warmup 20 --no-cpu-baseline $args > $O/$label.json 2> $O/$label.err
  python - "$O/$label.json" >> $O/sweep.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = d["kernels"]; o = d.get("overlap") or {}
    print("value %.0f e2e %.0f step %.1f | busy %s | fwd %.1f surr %.1f bwd %.1f xfer %.1f plan %.1f | %s | roof %.3f" % (
        d["value"], d["e2e"]["value"], d["ms_per_step"] * 1e3, o.get("stream_busy_us_per_step"),
        k["forward"]["avg_us"], k["surrogate"]["avg_us"], k["backward"]["avg_us"], k["transfer"]["avg_us"],
        k["plan"]["avg_us"], d["host_link"].get("transfer_mode"), d["roofline"]["frac"]))
except Exception as e:
    print("parse error", e)
PY
done
cat $O/sweep.log
