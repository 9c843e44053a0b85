#!/bin/bash
# five default bench runs back to back (run-to-run spread of the headline)
O=gpurun_out/${1:-rep}
mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_$i.json 2> $O/bench_$i.err
done
