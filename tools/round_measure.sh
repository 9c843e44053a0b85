#!/bin/bash
# One GPU-box measurement pass (run via gpurun from the repo root):
# build, GPU tests, default bench (with cpu_baseline), reference arm,
# ncu launch list and one full ncu capture of the hot kernels.
set -x
TAG=${1:-m}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.json 2> $O/ref.err
KR='regex:^(k_push|k_pullfill|k_fwd|k_bwd|k_surrogate)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 3000 -c 600 --csv \
  --log-file $O/launches.csv python bench.py --steps 200 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_list.log 2>&1
# The full capture runs with the GPU pull (SP_CPU_GATHER=0): ncu serialises
# every launch, which deadlocks the CPU gather handshake (a transfer waits for
# the gather thread, which waits for a Plan ncu has not let run yet).  The
# Train kernels it measures are the same; the launch list above is timed in
# the default configuration.
KF='regex:^(k_push|k_pullfill|k_fwd|k_bwd|k_surrogate)'
SP_CPU_GATHER=0 timeout 1200 ncu --set full --clock-control none --import-source on -k "$KF" -s 3000 -c 12 \
  -o $O/full python bench.py --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ls -la $O
