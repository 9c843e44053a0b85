set -x
mkdir -p gpurun_out/q19
python paper_2205_04702_b200/build.py > gpurun_out/q19/build1024.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q19/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q19/pytest_gpu.log
SP_PULL_CTAS=8 timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/q19/bench_1024.json 2> gpurun_out/q19/bench_1024.err
SP_NVCC_EXTRA="-DSP_PUSH_THREADS=512" python paper_2205_04702_b200/build.py --force > gpurun_out/q19/build512.log 2>&1
SP_PULL_CTAS=8 timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/q19/bench_512.json 2> gpurun_out/q19/bench_512.err
SP_DIAG=3 SP_PULL_CTAS=8 timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/q19/bench_512n.json 2> gpurun_out/q19/bench_512n.err
