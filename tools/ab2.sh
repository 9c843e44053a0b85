#!/bin/bash
O=gpurun_out/${1:-ab2}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
for R in base: nowb:SP_DIAG=4 nopull:SP_DIAG=1 base2:; do
  name=${R%%:*}; envs=${R#*:}
  env $envs timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > $O/bench_$name.json 2> $O/bench_$name.err
done
SP_NVCC_EXTRA="-DSP_PUSH_MIN_BLOCKS=2" python paper_2205_04702_b200/build.py --force > $O/build2.log 2>&1
timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > $O/bench_mb2.json 2> $O/bench_mb2.err
