# rasterizer work accounting + timing + ncu source capture at C2 and C4
set -x
mkdir -p gpurun_out
V=paper_2509_15645_b200/_build/var_stats/libgss_b200.so
GSS_LIB=$V timeout 600 python tools/raster_work.py 4000000 1920 1080 gpurun_out/work_c2.json > gpurun_out/work_c2.txt 2>&1
GSS_LIB=$V timeout 600 python tools/raster_work.py 40000000 3840 2160 gpurun_out/work_c4.json > gpurun_out/work_c4.txt 2>&1
timeout 600 python tools/time_render.py 40000000 3840 2160 2 > gpurun_out/time_c4.txt 2>&1
timeout 600 python tools/time_render.py 4000000 1920 1080 3 > gpurun_out/time_c2.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"forward_kernel|backward_kernel" -s 8 -c 2 -o gpurun_out/c4_raster python tools/time_render.py 40000000 3840 2160 1 > gpurun_out/ncu_c4.txt 2>&1
ls -la gpurun_out
timeout 600 python -m pytest tests/test_ply.py -q -m gpu > gpurun_out/pytest_ply.txt 2>&1
export GSS_PARITY_OUT=$PWD/gpurun_out/parity.json
timeout 1500 python -m pytest tests/test_scale_parity_gpu.py -q -m gpu -k engine --durations=5 > gpurun_out/pytest_scale.txt 2>&1
