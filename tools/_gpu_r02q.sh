# colour kernel templated on the SH degree, depth-order slot sums; dense geo update unroll variants
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_dropin_gpu.py tests/test_fullsize_gpu.py tests/test_evalsplit_gpu.py tests/test_densify_gpu.py -x -q > gpurun_out/pytest_q.txt 2>&1
tail -2 gpurun_out/pytest_q.txt
timeout 300 python tools/time_render.py 40000000 3840 2160 > gpurun_out/time_render_q.txt 2>&1; tail -1 gpurun_out/time_render_q.txt
for v in default dku1 dku3 dku4; do
  if [ $v = default ]; then L=""; else L="paper_2509_15645_b200/_build/var_$v/libgss_b200.so"; fi
  GSS_LIB=$L timeout 300 python tools/adam_probe.py 40000000 0.1292 >> gpurun_out/adam_probe_q.txt 2>&1
done
grep "{" gpurun_out/adam_probe_q.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4_q.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/launch_bench_q.log 2>&1
( time timeout 1200 python bench.py --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_c4_q.json 2> gpurun_out/bench_c4_q.err ) 2> gpurun_out/bench_c4_q.time
tail -c 200 gpurun_out/bench_c4_q.err
