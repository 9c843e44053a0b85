#!/bin/bash
# Bench lines for the non-headline BASELINE configs (evidence, not the driver's
# line): Terabyte-shaped and high-pooling on one B200.  Host RAM: ~96 / ~82 GB
# of pinned tables (run one at a time).
O=gpurun_out/${1:-cfg}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
free -g > $O/free.txt
timeout 1500 python bench.py --config terabyte --steps 300 --warmup 20 --profile-steps 100 --cpu-seconds 10 > $O/bench_terabyte.json 2> $O/bench_terabyte.err
free -g >> $O/free.txt
timeout 1500 python bench.py --config highpool --steps 40 --warmup 5 --profile-steps 20 --cpu-seconds 10 > $O/bench_highpool.json 2> $O/bench_highpool.err
ls -la $O
