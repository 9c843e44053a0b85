#!/bin/bash
# global radix dedup: every pass's histogram in one read; parity on the large-n paths + high-pooling plan timing
O=gpurun_out/${1:-hi}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_highpool.py tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 900 python bench.py --config highpool --steps 50 --warmup 5 --no-cpu-baseline > $O/hp.json 2> $O/hp.err
timeout 600 python bench.py --config kaggle --pooling 20 --steps 300 --warmup 10 --no-cpu-baseline > $O/kg_l20.json 2> $O/kg_l20.err
for f in $O/*.json; do python3 -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f'.split('/')[-1],round(d['value'],1),s.get('duration_us'),json.dumps(d.get('plan_ctas',{}))[:400])"; done
