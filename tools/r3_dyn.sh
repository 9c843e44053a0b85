#!/bin/bash
# k_bwd_tile dynamic tile claims: parity, then A/B against static round robin
O=gpurun_out/${1:-dyn}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_terabyte.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for d in 1 0 1 0; do
  SP_BWD_DYN=$d SP_BENCH_EVSPAN=1 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/tb_d$d.json 2> $O/tb_d$d.err
  grep evspan $O/tb_d$d.err
  python tools/bench_brief.py $O/tb_d$d.json
done
SP_BWD_DYN=1 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/go_d1.json 2> $O/go_d1.err
SP_BWD_DYN=0 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/go_d0.json 2> $O/go_d0.err
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f',d['value'],s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'), d['roofline'].get('span_frac'))"; done
