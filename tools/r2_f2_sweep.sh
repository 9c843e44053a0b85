#!/bin/bash
# sensitivity sweeps on the Terabyte shape:
# replacement policy, D, L, batch, slot fraction.  r2_f2_sweep.sh TAG
TAG=${1:-f2}
O=gpurun_out/$TAG
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
run() {  # label args...
  local label=$1; shift
  timeout 900 python bench.py --steps 200 --warmup 10 --preroll 2000 --no-cpu-baseline "$@" > $O/$label.json 2> $O/$label.err
  echo "== $label [$*] $(python tools/bench_brief.py $O/$label.json | cut -c40-)" >> $O/sweep.log
}
run base
run random --policy random
run lfu --policy lfu
run static --variant static
run b2048 --batch 2048
run b8192 --batch 8192
run s02 --slot-frac 0.02
run s10 --slot-frac 0.10
# D and L on the Kaggle shape (Terabyte at D=256 needs 192 GB of host tables)
run kg_base --config kaggle
run kg_d128 --config kaggle --dim 128
run kg_d256 --config kaggle --dim 256
run kg_l20 --config kaggle --pooling 20 --steps 50
run kg_l50 --config kaggle --pooling 50 --steps 30 --preroll 300
run serial --variant serial
run bf16 --storage bf16
cat $O/sweep.log
