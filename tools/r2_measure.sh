#!/bin/bash
# One GPU-box measurement pass (run via gpurun from the repo root):
#   r2_measure.sh TAG [CONFIG] [tests]
# build, (GPU tests), the driver-shaped bench (--steps 20 --warmup 5), a
# 1000-step bench, the ncu launch list and one full ncu capture of the hot
# kernels on CONFIG (default terabyte).
set -x
TAG=${1:-m}; CFG=${2:-terabyte}; TESTS=${3:-}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt; free -g > $O/free.txt
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
python -c "import oracle; oracle.build()" >> $O/build.log 2>&1
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q $TESTS > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 900 python bench.py --config $CFG --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err
timeout 900 python bench.py --config $CFG --steps 1000 --warmup 50 --no-cpu-baseline > $O/bench1000.json 2> $O/bench1000.err
KR='regex:^(k_push|k_pullfill|k_fwd|k_bwd|k_surrogate)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 2000 -c 500 --csv \
  --log-file $O/launches.csv python bench.py --config $CFG --preroll 1000 --steps 200 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_list.log 2>&1
KF='regex:^(k_push|k_pullfill|k_fwd|k_bwd|k_surrogate)'
SP_CPU_GATHER=0 timeout 1200 ncu --set full --clock-control none --import-source on -k "$KF" -s 2000 -c 10 \
  -o $O/full python bench.py --config $CFG --preroll 1000 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ls -la $O
