#!/bin/bash
# backward tile size A/B (SP_BWD_TR) and the claims, TB GPU-only + pipelined
O=gpurun_out/${1:-tr}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_terabyte.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for tr in 16 32 8; do
  SP_BWD_TR=$tr timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/go_tr$tr.json 2> $O/go_tr$tr.err
done
SP_BWD_DYN=0 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/go_static.json 2> $O/go_static.err
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/tb.json 2> $O/tb.err
timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --storage bf16 > $O/tb_bf16.json 2> $O/tb_bf16.err
timeout 600 python bench.py --config kaggle --steps 1000 --warmup 50 --no-cpu-baseline > $O/kg.json 2> $O/kg.err
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f',d['value'],s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'), d['roofline'].get('frac'), d['roofline'].get('span_frac'))"; done
