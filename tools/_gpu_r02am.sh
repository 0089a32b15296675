# sweep at 11 CTAs/SM + 16-byte slot-sum staging: parity + bench phases
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_raster_gpu.py tests/test_imgpar_gpu.py tests/test_engine_gpu.py tests/test_split_engine_gpu.py -x -q > gpurun_out/pytest_am.txt 2>&1; tail -n 2 gpurun_out/pytest_am.txt
for i in 1 2; do
  timeout 900 python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_am_$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_am_$i.json').read().strip().splitlines()[-1]);print('am',round(d['value'],3),{k:round(v,3) for k,v in d['render_kernels']['phases_ms_per_step'].items()})" >> gpurun_out/ab_am.txt
done
cat gpurun_out/ab_am.txt
