#!/bin/bash
# high-pooling configuration: where the step goes (plan / transfer / train)
O=gpurun_out/${1:-hp}
mkdir -p $O
free -g > $O/free.txt
timeout 900 python bench.py --config highpool --steps 50 --warmup 5 --no-cpu-baseline > $O/hp.json 2> $O/hp.err
python tools/bench_brief.py $O/hp.json
python3 -c "
import json;d=json.loads(open('$O/hp.json').read().strip().splitlines()[-1]);s=d.get('spans') or {};print(d['value'],s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'), d['roofline'])"
tail -3 $O/hp.err
