# backward sweep rework (9 sums, scalar suffix, clamp-free path) + staged host tier A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_adam_gpu.py -x -q > gpurun_out/pytest_h.txt 2>&1
tail -3 gpurun_out/pytest_h.txt
timeout 300 python tools/time_render.py 40000000 3840 2160 > gpurun_out/time_render_c4_h.txt 2>&1
tail -2 gpurun_out/time_render_c4_h.txt
timeout 300 python tools/host_tier_probe.py 40000000 0.13 > gpurun_out/htp_staged.txt 2>&1
GSS_HOST_STAGING=0 timeout 300 python tools/host_tier_probe.py 40000000 0.13 > gpurun_out/htp_inplace.txt 2>&1
cat gpurun_out/htp_staged.txt gpurun_out/htp_inplace.txt | tail -4
timeout 900 python bench.py --n 18000000 --width 1920 --height 1080 --nongeo-tier host --no-cpu-baseline --no-probe --steps 8 --warmup 3 > gpurun_out/bench_c3_host.json 2> gpurun_out/bench_c3_host.err
