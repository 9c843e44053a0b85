#!/bin/bash
# ncu --set full on k_bwd_tile + k_fwd + k_pullfill in the TB pipelined steady state, source-level
TAG=$1
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
cp paper_2205_04702_b200/lib/k_train.o $O/ 2>/dev/null
SP_CPU_GATHER=0 timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:^(k_fwd|k_bwd|k_pullfill)' -s 60 -c 6 \
  -o $O/full python bench.py --preroll 300 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ncu -i $O/full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum > $O/raw.csv 2>&1
ncu -i $O/full.ncu-rep --page source --csv --kernel-name regex:k_bwd_tile --launch-skip 0 --launch-count 1 > $O/bwd_source.csv 2>&1
ncu -i $O/full.ncu-rep --page details --csv --kernel-name regex:k_bwd_tile --launch-skip 0 --launch-count 1 > $O/bwd_details.csv 2>&1
ls -la $O
