# drop-in (free functions + engine), host-tier tests, full bench at C4, ncu source capture
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dropin_gpu.py tests/test_adam_gpu.py -x -q > gpurun_out/pytest_j.txt 2>&1
tail -3 gpurun_out/pytest_j.txt
./oracle/_ref/dropin_test > gpurun_out/dropin_j.txt 2>&1; tail -8 gpurun_out/dropin_j.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4_j.json 2> gpurun_out/bench_c4_j.err ) 2> gpurun_out/bench_c4_j.time
tail -c 300 gpurun_out/bench_c4_j.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"forward_kernel|backward_kernel" -s 2 -c 2 -o gpurun_out/c4_raster_src python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_src.txt 2>&1
tail -3 gpurun_out/ncu_src.txt
