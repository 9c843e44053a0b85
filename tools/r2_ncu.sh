#!/bin/bash
# ncu --set full of the Train kernels (+ launch list) on one bench config:
#   r2_ncu.sh TAG "bench args" [kernel regex]
TAG=$1; ARGS=$2; KR=${3:-'regex:^(k_fwd|k_bwd|k_surrogate|k_push|k_pullfill)'}
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 2000 -c 500 --csv \
  --log-file $O/launches.csv python bench.py $ARGS --preroll 1000 --steps 200 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_list.log 2>&1
SP_CPU_GATHER=0 timeout 1500 ncu --set full --import-source on --clock-control none -k "$KR" -s 2000 -c 10 \
  -o $O/full python bench.py $ARGS --preroll 1000 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ls -la $O
