#!/bin/bash
# ncu --set full of the Train kernels (k_fwd, k_surrogate, k_bwd*) on the TB bench:
#   r2_ncu_train.sh TAG ["bench args"]
TAG=$1; ARGS=${2:-}
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
SP_CPU_GATHER=0 timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:^(k_fwd|k_bwd|k_surrogate)' -s 60 -c 6 \
  -o $O/full python bench.py $ARGS --preroll 300 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ncu -i $O/full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__shared_mem_per_block_dynamic > $O/raw.csv 2>&1
ls -la $O
