#!/bin/bash
# PAPER.md Fig. 10 / Table 1 design points from the same kernels
O=gpurun_out/${1:-var}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
for V in pipelined serial resident; do
  timeout 900 python bench.py --variant $V --steps 1000 --warmup 20 --no-cpu-baseline > $O/kaggle_$V.json 2> $O/kaggle_$V.err
done
for V in pipelined serial resident; do
  timeout 1500 python bench.py --config terabyte --variant $V --steps 300 --warmup 20 --profile-steps 100 --no-cpu-baseline > $O/terabyte_$V.json 2> $O/terabyte_$V.err
done
ls -la $O
