# segmented slot sums with GSS_SUM_U chunks' loads in flight (long spans of big splats): parity + same-box A/B
set -x
mkdir -p gpurun_out
B=paper_2509_15645_b200/_build
timeout 1500 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py "tests/test_scale_parity_gpu.py::test_c4_strip_forward_backward_vs_reference" "tests/test_scale_parity_gpu.py::test_c2_view_forward_backward_vs_reference" -x -q > gpurun_out/pytest_ay.txt 2>&1; tail -n 3 gpurun_out/pytest_ay.txt
GSS_LIB=$B/var_su8/libgss_b200.so timeout 900 python -m pytest tests/test_raster_gpu.py -x -q > gpurun_out/pytest_ay_su8.txt 2>&1; tail -n 1 gpurun_out/pytest_ay_su8.txt
for i in 1 2; do
  for v in default su8 su1 seg0; do
    if [ $v = default ]; then L=; else L=$B/var_$v/libgss_b200.so; fi
    GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_ay_$v$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/bench_ay_$v$i.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_ay.txt
  done
done
cat gpurun_out/ab_ay.txt
