# certified composite path without max/clamp (records certified also carry alpha_base <= 0.999): parity + A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_engine_gpu.py "tests/test_scale_parity_gpu.py" -x -q > gpurun_out/pytest_ap.txt 2>&1; tail -n 2 gpurun_out/pytest_ap.txt
for i in 1 2; do
  for v in new prev; do
    if [ $v = prev ]; then L=paper_2509_15645_b200/_build/var_fprev/libgss_b200.so; else L=; fi
    GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_ap_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_ap_$v$i.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_ap.txt
  done
done
cat gpurun_out/ab_ap.txt
