#!/bin/bash
# ncu --set full (source-level) of k_bwd_tile / k_bwd_rows / k_fwd in the TB pipelined steady state (GPU-only holds 128 GB: too large for ncu replay)
O=gpurun_out/${1:-nb}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
cp paper_2205_04702_b200/lib/k_train.o $O/
SP_CPU_GATHER=0 timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:^(k_fwd|k_bwd)' -s 30 -c 6 \
  -o $O/full python bench.py --preroll 300 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ncu -i $O/full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum > $O/raw.csv 2>&1
ls -la $O
