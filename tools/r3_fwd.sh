#!/bin/bash
# k_fwd dynamic bag chunks, k_bwd_rows 8-in-flight up to 32 pieces, k_pullfill bf16 conversion: parity + A/B
O=gpurun_out/${1:-fw}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_terabyte.py tests/test_gpu_bf16.py tests/test_gpu_variants.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for d in 1 0; do
  SP_FWD_DYN=$d timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > $O/tb_f$d.json 2> $O/tb_f$d.err
  SP_FWD_DYN=$d timeout 600 python bench.py --steps 300 --warmup 20 --no-cpu-baseline --variant gpuonly > $O/go_f$d.json 2> $O/go_f$d.err
done
timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --storage bf16 > $O/tb_bf16.json 2> $O/tb_bf16.err
timeout 600 python bench.py --config kaggle --steps 1000 --warmup 50 --no-cpu-baseline > $O/kg.json 2> $O/kg.err
for f in $O/*.json; do python3 -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);s=d.get('spans') or {};print('$f',d['value'],d['e2e']['value'],s.get('duration_us'),s.get('stream_busy_us_per_step'),s.get('step_us'), d['roofline'].get('frac'), d['roofline'].get('span_frac'))"; done
