# cp.async row staging (chain, colour), tail zero-fill instead of the partials memset, slot-sum ILP,
# optimizer launch shapes: tests + timings + bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_adam_gpu.py tests/test_fullsize_gpu.py -x -q > gpurun_out/pytest_o.txt 2>&1
tail -2 gpurun_out/pytest_o.txt
timeout 300 python tools/time_render.py 40000000 3840 2160 > gpurun_out/time_render_o.txt 2>&1; tail -1 gpurun_out/time_render_o.txt
timeout 300 python tools/adam_probe.py 40000000 0.1292 > gpurun_out/adam_probe_o.txt 2>&1; tail -1 gpurun_out/adam_probe_o.txt
( time timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_o.json 2> gpurun_out/bench_c4_o.err ) 2> gpurun_out/bench_c4_o.time
tail -c 300 gpurun_out/bench_c4_o.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_o.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_o.log 2>&1
