# engine prewarm (every stored camera rendered once at creation): tests, short-warm-up bench, default bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_split_engine_gpu.py tests/test_densify_gpu.py tests/test_dropin_gpu.py tests/test_imgpar_gpu.py -x -q > gpurun_out/pytest_aj.txt 2>&1; tail -n 2 gpurun_out/pytest_aj.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-probe --no-host-offload > gpurun_out/bench_aj_w3.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench_aj_w3.json').read().strip().splitlines()[-1]);print('w3',d['value'],d['e2e']['value'])"
( time timeout 1200 python bench.py > gpurun_out/bench_c4_aj.json 2> gpurun_out/bench_c4_aj.err ) 2> gpurun_out/bench_c4_aj.time
python -c "import json;d=json.loads(open('gpurun_out/bench_c4_aj.json').read().strip().splitlines()[-1]);print('default',d['value'],d['e2e']['value'],[(k['kernel'][:12],round(k['frac'],3)) for k in d['kernels']],d['host_offload']['value'])"
