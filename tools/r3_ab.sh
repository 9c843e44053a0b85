#!/bin/bash
# A/B of k_bwd_rows' one-warp threshold (SP_BWD2_SMALL) in the TB GPU-only variant, interleaved
O=gpurun_out/${1:-ab}
mkdir -p $O
for rep in 1 2 3; do for v in 8 32 16; do
  SP_BWD2_SMALL=$v timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --no-cpu-baseline --variant gpuonly > $O/go_s${v}_$rep.json 2> $O/go_s${v}_$rep.err
done; done
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f',d['value'],s.get('duration_us',{}).get('backward'),s.get('step_us'))"; done
