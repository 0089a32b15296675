# tests (incl. stage delays / timeline), default bench at C4, link probes, new-kernel profiles
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --ignore=tests/test_scale_parity_gpu.py > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
( time timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err ) 2> gpurun_out/bench_c4.time
tail -c 400 gpurun_out/bench_c4.err
timeout 300 tools/linkprobe > gpurun_out/linkprobe2.txt 2>&1
GSS_LIB=paper_2509_15645_b200/_build/var_stats/libgss_b200.so timeout 600 python tools/raster_work.py 40000000 3840 2160 gpurun_out/work_c4.json > gpurun_out/work_c4.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"forward_kernel|backward_kernel" -s 8 -c 2 -o gpurun_out/c4_raster_r02 python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_c4.txt 2>&1
tail -2 gpurun_out/ncu_c4.txt
