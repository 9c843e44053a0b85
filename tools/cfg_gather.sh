#!/bin/bash
# Terabyte / high-pool: CPU gather (default) vs GPU pull of random host rows
O=gpurun_out/${1:-cfgg}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 1200 python bench.py --config terabyte --steps 300 --warmup 20 --profile-steps 100 --no-cpu-baseline > $O/tb_cg.json 2> $O/tb_cg.err
SP_CPU_GATHER=0 timeout 1200 python bench.py --config terabyte --steps 300 --warmup 20 --profile-steps 100 --no-cpu-baseline > $O/tb_gp.json 2> $O/tb_gp.err
timeout 1500 python bench.py --config highpool --steps 40 --warmup 5 --profile-steps 20 --no-cpu-baseline > $O/hp_cg.json 2> $O/hp_cg.err
SP_CPU_GATHER=0 timeout 1500 python bench.py --config highpool --steps 40 --warmup 5 --profile-steps 20 --no-cpu-baseline > $O/hp_gp.json 2> $O/hp_gp.err
ls -la $O
