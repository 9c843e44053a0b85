#!/bin/bash
# transfer A/B after the dynamic forward: pull CTAs x CPU gather share, TB pipelined, interleaved x2
O=gpurun_out/${1:-xf}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_terabyte.py -x -q -k bf16 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for rep in 1 2; do
for cta in 16 24 32; do for gf in 0.5 0.35; do
  SP_PULL_CTAS=$cta timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --gather-frac $gf > $O/c${cta}_g${gf}_$rep.json 2> $O/c${cta}_g${gf}_$rep.err
done; done; done
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f'.split('/')[-1],round(d['value']),'e2e',round(d['e2e']['value']),s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'))"; done
