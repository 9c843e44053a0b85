#!/bin/bash
# quick_gpu.sh plus a GPU-test pass under the env of $TESTENV
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
if [ -n "$TESTENV" ]; then
  env $(echo $TESTENV | tr ',' ' ') timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_env.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_env.log
fi
NOTEST=1 bash tools/quick_gpu.sh $TAG
