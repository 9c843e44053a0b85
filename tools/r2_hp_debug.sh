O=gpurun_out/hp1; mkdir -p $O
python paper_2205_04702_b200/build.py > $O/build.log 2>&1; python -c "import oracle; oracle.build()" >> $O/build.log 2>&1
for cfg in "A:" "B:" "C:SP_DIAG=32" "D:SP_BWD=rec" "E:SP_CPU_GATHER=0" "F:SP_BWD_TR=16"; do
  tag=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python -m pytest tests/test_gpu_highpool.py -q -x -p no:cacheprovider > $O/$tag.log 2>&1
  echo "$cfg -> $(tail -1 $O/$tag.log)"
done
