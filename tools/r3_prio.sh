#!/bin/bash
# plan stream at high (default) vs normal priority (SP_PLAN_PRIO=0), TB pipelined, interleaved x2
O=gpurun_out/${1:-pr}
mkdir -p $O
for rep in 1 2; do for p in 1 0; do
  SP_PLAN_PRIO=$p timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/prio${p}_$rep.json 2> $O/p${p}_$rep.err
done; done
for f in $O/*.json; do python3 -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f'.split('/')[-1],round(d['value']),'e2e',round(d['e2e']['value']),s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'),d['roofline']['frac'],d['roofline'].get('span_frac'))"; done
