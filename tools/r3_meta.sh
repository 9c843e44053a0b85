#!/bin/bash
# k_bwd_tile metadata two tiles ahead (168 regs, 12 warps/SM) vs one tile ahead (128 regs), TB GPU-only + pipelined, interleaved x2
O=gpurun_out/${1:-me}
mkdir -p $O
for rep in 1 2; do
  for v in "1 12" "0 16"; do set -- $v
    SP_NVCC_EXTRA="-DSP_META2=$1 -DSP_BWD_TILE_MINB=$2" python paper_2205_04702_b200/build.py --force > $O/b$1.log 2>&1
    timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/g_m$1_$rep.json 2> $O/g_m$1_$rep.err
    timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > $O/p_m$1_$rep.json 2> $O/p_m$1_$rep.err
  done
done
python paper_2205_04702_b200/build.py --force > $O/bdef.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bf16.py tests/test_gpu_terabyte.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f'.split('/')[-1],round(d['value']),'e2e',round(d['e2e']['value']),s.get('duration_us'),s.get('step_us'),d['roofline']['frac'],d['roofline'].get('span_frac'))"; done
