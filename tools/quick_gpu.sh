#!/bin/bash
# quick GPU pass: build, GPU tests, short benches over env settings
#   RUNS="name:ENV=V,ENV2=V ..."  (default one run with no env)
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
for R in ${RUNS:-base:}; do
  name=${R%%:*}; envs=${R#*:}
  env $(echo $envs | tr ',' ' ') SP_TIMELINE=$O/tl_$name.json timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline ${BENCH_ARGS} > $O/bench_$name.json 2> $O/bench_$name.err
  python tools/timeline_report.py $O/tl_$name.json > $O/tl_$name.txt 2>&1
  rm -f $O/tl_$name.json
done
