#!/bin/bash
# two-phase backward: parity, then A/B (SP_BWD_2P) in the TB pipeline and GPU-only
O=gpurun_out/${1:-tp}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_terabyte.py tests/test_gpu_variants.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for v in pipelined gpuonly; do
for p in 1 0; do
  SP_BWD_2P=$p timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant $v > $O/tb_${v}_p$p.json 2> $O/tb_${v}_p$p.err
done; done
SP_BWD_2P=1 timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --storage bf16 > $O/tb_bf16_p1.json 2> $O/tb_bf16_p1.err
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f',d['value'],s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'), d['roofline'].get('frac'), d['roofline'].get('span_frac'))"; done
