#!/bin/bash
# event-vs-span diagnostic under different hardware-queue counts
O=gpurun_out/${1:-conn}
mkdir -p $O
for c in 32 2 8; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c SP_BENCH_EVSPAN=1 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/tb_c$c.json 2> $O/tb_c$c.err
done
grep evspan $O/*.err
python tools/bench_brief.py $O/tb_c*.json
