#!/bin/bash
# k_push CTA size A/B on Terabyte: 1024 threads (default; a CTA fills an SM's registers)
# vs 512 (two per SM, room for the Train kernels beside it), interleaved x2
O=gpurun_out/${1:-pu}
mkdir -p $O
for rep in 1 2; do
  python paper_2205_04702_b200/build.py --force > $O/b1024.log 2>&1
  timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/p1024_$rep.json 2> $O/p1024_$rep.err
  SP_NVCC_EXTRA="-DSP_PUSH_THREADS=512" python paper_2205_04702_b200/build.py --force > $O/b512.log 2>&1
  timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/p512_$rep.json 2> $O/p512_$rep.err
  timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/g512_$rep.json 2> $O/g512_$rep.err
done
SP_NVCC_EXTRA="-DSP_PUSH_THREADS=512" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_highpool.py -x -q > $O/pytest512.log 2>&1; echo "rc=$?" >> $O/pytest512.log
tail -2 $O/pytest512.log
python paper_2205_04702_b200/build.py --force > $O/b1024.log 2>&1
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f'.split('/')[-1],round(d['value']),'e2e',round(d['e2e']['value']),s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'),d['roofline']['frac'],d['roofline'].get('span_frac'))"; done
