# packed depth-sort payload (binning reads sequentially): tests + timings + bench + launch list
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_fullsize_gpu.py tests/test_dropin_gpu.py tests/test_scale_parity_gpu.py -x -q > gpurun_out/pytest_p.txt 2>&1
tail -2 gpurun_out/pytest_p.txt
timeout 300 python tools/time_render.py 40000000 3840 2160 > gpurun_out/time_render_p.txt 2>&1; tail -1 gpurun_out/time_render_p.txt
( time timeout 1200 python bench.py --no-cpu-baseline --no-probe > gpurun_out/bench_c4_p.json 2> gpurun_out/bench_c4_p.err ) 2> gpurun_out/bench_c4_p.time
tail -c 300 gpurun_out/bench_c4_p.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_p.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_p.log 2>&1
