#!/bin/bash
# Round-2 closing measurement (after the two-phase backward and bf16 Storage):
#   r3_final.sh TAG
# box facts, build, the GPU suite, smoke(), the driver-shaped bench (--steps 20
# --warmup 5, with cpu_baseline), a 1000-step bench, bf16 / GPU-only / Kaggle /
# high-pooling lines, the reference arm, the ncu launch list and one ncu --set
# full capture of the stage kernels.
TAG=${1:-final3}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt; free -g > $O/free.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err
timeout 900 python bench.py --steps 1000 --warmup 50 --no-cpu-baseline > $O/bench1000.json 2> $O/bench1000.err
timeout 900 python bench.py --steps 1000 --warmup 50 --no-cpu-baseline --storage bf16 > $O/bench1000_bf16.json 2> $O/bench1000_bf16.err
timeout 900 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/gpuonly.json 2> $O/gpuonly.err
timeout 900 python bench.py --config kaggle --steps 1000 --warmup 50 --no-cpu-baseline > $O/kaggle.json 2> $O/kaggle.err
timeout 900 python bench.py --config highpool --steps 50 --warmup 5 --no-cpu-baseline > $O/highpool.json 2> $O/highpool.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/ref.json 2> $O/ref.err
KR='regex:^(k_push|k_pullfill|k_fwd|k_bwd|k_surrogate)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 2000 -c 600 --csv \
  --log-file $O/launches.csv python bench.py --preroll 1000 --steps 200 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_list.log 2>&1
SP_CPU_GATHER=0 timeout 1500 ncu --set full --import-source on --clock-control none -k "$KR" -s 2000 -c 12 \
  -o $O/full python bench.py --preroll 1000 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
python tools/bench_brief.py $O/bench20.json $O/bench1000.json $O/bench1000_bf16.json $O/gpuonly.json $O/kaggle.json $O/highpool.json
ls -la $O
