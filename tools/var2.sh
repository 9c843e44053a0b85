#!/bin/bash
O=gpurun_out/${1:-var2}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --variant gpuonly --preroll 200 --steps 1000 --warmup 20 --no-cpu-baseline > $O/kaggle_gpuonly.json 2> $O/kaggle_gpuonly.err
timeout 1500 python bench.py --config terabyte --variant gpuonly --preroll 200 --steps 300 --warmup 20 --profile-steps 100 --no-cpu-baseline > $O/terabyte_gpuonly.json 2> $O/terabyte_gpuonly.err
