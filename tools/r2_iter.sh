#!/bin/bash
# One iteration on the GPU box: build, GPU tests (all | none | -k expr),
# isolated-stage (serial) + gpuonly + pipelined TB bench lines, one summary.
#   r2_iter.sh TAG [all|none|expr] [extra bench args...]
TAG=${1:-it}; SEL=${2:-all}; shift 2
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
python -c "import oracle; oracle.build()" >> $O/build.log 2>&1
if [ "$SEL" == "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
elif [ "$SEL" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$SEL" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
for v in serial gpuonly pipelined; do
  timeout 600 python bench.py --variant $v --steps 500 --warmup 20 --no-cpu-baseline "$@" > $O/$v.json 2> $O/$v.err
done
tail -3 $O/pytest_gpu.log 2>/dev/null; grep ^FAILED $O/pytest_gpu.log 2>/dev/null | head
python tools/bench_brief.py $O/serial.json $O/gpuonly.json $O/pipelined.json
