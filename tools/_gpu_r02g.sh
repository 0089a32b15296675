# split engine + staged host tier: tests, then C3 / C4 host-tier engine timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_split_engine_gpu.py tests/test_adam_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/pytest_g.txt 2>&1
tail -15 gpurun_out/pytest_g.txt
timeout 900 python bench.py --n 18000000 --width 1920 --height 1080 --nongeo-tier host --no-cpu-baseline --no-probe --steps 8 --warmup 3 > gpurun_out/bench_c3_host.json 2> gpurun_out/bench_c3_host.err
tail -c 300 gpurun_out/bench_c3_host.err
timeout 900 python bench.py --nongeo-tier host --no-cpu-baseline --no-probe --steps 6 --warmup 3 > gpurun_out/bench_c4_host.json 2> gpurun_out/bench_c4_host.err
tail -c 300 gpurun_out/bench_c4_host.err
