#!/bin/bash
# bf16 Storage vs fp32 on the Terabyte and Kaggle shapes, plus the event-vs-span
# diagnostic (SP_BENCH_EVSPAN=1: in-kernel spans stamped inside the event pass)
O=gpurun_out/${1:-bf}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SP_BENCH_EVSPAN=1 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/tb_f32.json 2> $O/tb_f32.err
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --storage bf16 > $O/tb_bf16.json 2> $O/tb_bf16.err
timeout 600 python bench.py --config kaggle --steps 1000 --warmup 50 --no-cpu-baseline > $O/kg_f32.json 2> $O/kg_f32.err
timeout 600 python bench.py --config kaggle --steps 1000 --warmup 50 --no-cpu-baseline --storage bf16 > $O/kg_bf16.json 2> $O/kg_bf16.err
SP_CPU_GATHER=0 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly --storage bf16 > $O/tb_gpuonly_bf16.json 2> $O/tb_gpuonly_bf16.err
grep evspan $O/*.err
python tools/bench_brief.py $O/tb_f32.json $O/tb_bf16.json $O/kg_f32.json $O/kg_bf16.json $O/tb_gpuonly_bf16.json
