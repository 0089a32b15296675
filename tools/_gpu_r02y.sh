# sweep with neutral idle lanes (GSS_BWD_NEUTRAL): MUFU exactness facts, parity, kernel timing A/B
set -x
mkdir -p gpurun_out
./tools/mufucheck > gpurun_out/mufucheck.txt 2>&1; cat gpurun_out/mufucheck.txt
B=paper_2509_15645_b200/_build/var_bneutral/libgss_b200.so
GSS_LIB=$B timeout 900 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/pytest_y.txt 2>&1; tail -n 2 gpurun_out/pytest_y.txt
for v in default bneutral default bneutral; do
  if [ $v = default ]; then L=""; else L=$B; fi
  GSS_LIB=$L timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_y_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_y_$v.json').read().strip().splitlines()[-1]);print('$v',round(d['value'],3),d['render_kernels']['composite_ms_per_launch'],d['render_kernels']['sweep_ms_per_launch'])" >> gpurun_out/ab_y.txt
done
cat gpurun_out/ab_y.txt
