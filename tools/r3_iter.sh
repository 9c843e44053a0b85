#!/bin/bash
# iteration pass: backward parity, TB pipelined + GPU-only benches, ncu of the Train kernels
O=gpurun_out/${1:-it}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_terabyte.py tests/test_gpu_bf16.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for v in gpuonly pipelined; do
  timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant $v > $O/tb_${v}.json 2> $O/tb_${v}.err
done
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f',d['value'],s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'), d['roofline'].get('frac'), d['roofline'].get('span_frac'))"; done
if [ "${NCU:-1}" = 1 ]; then
cp paper_2205_04702_b200/lib/k_train.o $O/
SP_CPU_GATHER=0 timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:^(k_fwd|k_bwd)' -s 30 -c 6 \
  -o $O/full python bench.py --preroll 300 --steps 40 --warmup 5 --no-cpu-baseline --profile-steps 5 > $O/ncu_full.log 2>&1
ncu -i $O/full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum > $O/raw.csv 2>&1
python3 -c "
import csv
r=list(csv.reader(open('$O/raw.csv')))
h=r[0]
for x in r[2:]:
    d=dict(zip(h,x)); print(d['Kernel Name'][:40], d['gpu__time_duration.sum'], 'us', d['dram__bytes_read.sum'], d['smsp__inst_executed.sum'], d['sm__warps_active.avg.pct_of_peak_sustained_active'])
"
fi
