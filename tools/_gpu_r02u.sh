# composite with certified-range records (GSS_FWD_SAFE): bit-exactness + kernel timing A/B in the engine
set -x
mkdir -p gpurun_out
F=paper_2509_15645_b200/_build/var_fsafe/libgss_b200.so
GSS_LIB=$F timeout 1200 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_fullsize_gpu.py "tests/test_scale_parity_gpu.py::test_c2_view_forward_backward_vs_reference" -x -q > gpurun_out/pytest_u.txt 2>&1
tail -2 gpurun_out/pytest_u.txt
for v in default fsafe default fsafe; do
  if [ $v = default ]; then L=""; else L=$F; fi
  GSS_LIB=$L timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_u_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_u_$v.json').read().strip().splitlines()[-1]);print('$v',d['value'],d['render_kernels']['composite_ms_per_launch'],d['render_kernels']['sweep_ms_per_launch'])" >> gpurun_out/ab_u.txt
done
cat gpurun_out/ab_u.txt
