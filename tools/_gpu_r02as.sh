# sweep with dx-factored moments (GSS_BWD_XFACT): raster parity + same-box A/B; row-walk access ceiling probe
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_adam_gpu.py "tests/test_scale_parity_gpu.py" -x -q > gpurun_out/pytest_as.txt 2>&1; tail -n 3 gpurun_out/pytest_as.txt
timeout 300 ./tools/rowprobe > gpurun_out/rowprobe_as.txt 2>&1; cat gpurun_out/rowprobe_as.txt
for i in 1 2; do
  for v in default xf0; do
    if [ $v = default ]; then L=; else L=paper_2509_15645_b200/_build/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 600 python tools/time_render.py 40000000 3840 2160 2 > gpurun_out/tr_as_$v$i.txt 2>&1; echo $v; tail -n 2 gpurun_out/tr_as_$v$i.txt
  done
done
for i in 1 2; do
  for v in default xf0; do
    if [ $v = default ]; then L=; else L=paper_2509_15645_b200/_build/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_as_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_as_$v$i.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_as.txt
  done
done
cat gpurun_out/ab_as.txt
