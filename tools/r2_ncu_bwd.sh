#!/bin/bash
# ncu --set full of the Train kernels on one config + an isolated-stage bench:
#   r2_ncu_bwd.sh TAG "bench args"
TAG=$1; ARGS=$2
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 600 python bench.py $ARGS --variant serial --steps 300 --warmup 20 --no-cpu-baseline > $O/serial.json 2> $O/serial.err
timeout 600 python bench.py $ARGS --variant gpuonly --steps 300 --warmup 20 --no-cpu-baseline > $O/gpuonly.json 2> $O/gpuonly.err
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:^(k_fwd|k_bwd|k_surrogate)' -s 300 -c 6 \
  -o $O/full python bench.py $ARGS --variant gpuonly --preroll 200 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ls -la $O
