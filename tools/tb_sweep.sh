#!/bin/bash
O=gpurun_out/${1:-tb}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for X in 0 16 48; do
  if [ $X = 0 ]; then E=""; else E="SP_PULL_CTAS=$X"; fi
  env $E timeout 1200 python bench.py --config terabyte --steps 300 --warmup 20 --profile-steps 100 --no-cpu-baseline > $O/tb_$X.json 2> $O/tb_$X.err
done
timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > $O/kaggle.json 2> $O/kaggle.err
