# lazy update released after the render's geometry phase (GSS_LAZY_AFTER_GEOM) A/B at C4
set -x
mkdir -p gpurun_out
for m in 0 1 0 1; do
  GSS_LAZY_AFTER_GEOM=$m timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_ad_$m.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_ad_$m.json').read().strip().splitlines()[-1]);print('lazy_after_geom $m',round(d['value'],3),{k:round(v,2) for k,v in d['stage_ms_per_step'].items()},{k:round(v,2) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_ad.txt
done
cat gpurun_out/ab_ad.txt
GSS_LAZY_AFTER_GEOM=1 timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_split_engine_gpu.py -x -q > gpurun_out/pytest_ad.txt 2>&1; tail -n 2 gpurun_out/pytest_ad.txt
