#!/bin/bash
# Quick GPU pass: build, GPU tests (optionally a -k filter), TB bench (1000
# steps), optional extra bench args.   r2_quick.sh TAG ["pytest -k expr"|all|none] [extra bench args...]
set -x
TAG=${1:-q}; SEL=${2:-all}; shift 2
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
python -c "import oracle; oracle.build()" >> $O/build.log 2>&1
if [ "$SEL" == "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
elif [ "$SEL" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$SEL" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 900 python bench.py --steps 1000 --warmup 50 --no-cpu-baseline "$@" > $O/bench.json 2> $O/bench.err
tail -2 $O/pytest_gpu.log 2>/dev/null
