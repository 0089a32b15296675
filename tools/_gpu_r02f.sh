# session 3 baseline: full gpu tests, default bench (C4), launch list of a short bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err ) 2> gpurun_out/bench_c4.time
tail -c 400 gpurun_out/bench_c4.err
